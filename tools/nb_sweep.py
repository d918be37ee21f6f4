"""Tile-size sweep: Cholesky TFLOP/s of exageo_loglik_dev for n x nb (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

ns = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [10000, 20000, 40000]
nbs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 384, 512, 768]
for n in ns:
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
    for nb in nbs:
        with ex.Context(device=0, nb=nb) as c:
            c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
            best = min(c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5)).info["ms_total"] for _ in range(3))
        print(f"n={n} nb={nb} total={best:.2f} ms  TF={n**3 / 3 / best / 1e9:.2f}", flush=True)
