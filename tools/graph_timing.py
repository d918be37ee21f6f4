"""Evaluation latency with and without CUDA-graph replay (development aid)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1708_02835_b200 as ex
import synth_inputs as si

TH = (1.0, 0.1, 0.5)
for n in [int(v) for v in sys.argv[1:]] or [400, 1600, 5000, 10000, 20000]:
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
    row = [f"n={n}"]
    for g in (-1, 1):
        with ex.Context(device=0, graphs=g) as c:
            reps = 50 if n <= 5000 else 10
            for _ in range(3):
                c.loglik_dev(X, Y, Z, TH)
            dev, wall = [], []
            for _ in range(reps):
                t0 = time.perf_counter()
                r = c.loglik_dev(X, Y, Z, TH)
                wall.append(time.perf_counter() - t0)
                dev.append(r.info["ms_total"])
            row.append(f"graphs={g}: device {1e3 * statistics.median(dev):8.1f} us wall {1e6 * statistics.median(wall):8.1f} us")
    print("  ".join(row), flush=True)
