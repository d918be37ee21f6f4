"""Evaluation latency: tile-task executor (one persistent kernel) vs the stream-launched
schedule, both with CUDA-graph replay where eligible (development aid; prints device and
wall medians per n)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1708_02835_b200 as ex
import synth_inputs as si

TH = (1.0, 0.1, 0.5)
for n in [int(v) for v in sys.argv[1:]] or [400, 1600, 3000, 5000, 6144, 8000, 10000]:
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
    row = [f"n={n:6d}"]
    for tt in (1, -1):
        with ex.Context(device=0, tile_tasks=tt) as c:
            reps = 50 if n <= 5000 else 10
            for _ in range(3):
                c.loglik_dev(X, Y, Z, TH)
            dev, wall = [], []
            for _ in range(reps):
                t0 = time.perf_counter()
                r = c.loglik_dev(X, Y, Z, TH)
                wall.append(time.perf_counter() - t0)
                dev.append(r.info["ms_total"])
            row.append(f"tile_tasks={tt:2d}: device {1e3 * statistics.median(dev):9.1f} us "
                       f"wall {1e6 * statistics.median(wall):9.1f} us ({r.info['kernels']} kernels)")
    print("  ".join(row), flush=True)
