"""Device time per evaluation at small n for each tile size (development aid)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1708_02835_b200 as ex
import synth_inputs as si

TH = (1.0, 0.1, 0.5)
for n in (256, 400, 700, 1000, 1600, 2500):
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
    row = [f"n={n:5d}"]
    for nb in (128, 256, 384, 512):
        with ex.Context(device=0, nb=nb) as c:
            for _ in range(5):
                c.loglik_dev(X, Y, Z, TH)
            d = [c.loglik_dev(X, Y, Z, TH).info["ms_total"] for _ in range(30)]
            row.append(f"nb={nb}: {1e3 * statistics.median(d):7.1f} us")
    print("  ".join(row), flush=True)
