"""Quick per-phase timing of exageo_loglik_dev over n (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1708_02835_b200 as ex
import synth_inputs as si

ns = [int(v) for v in sys.argv[1:]] or [10000, 20000, 40000]
THETA = tuple(float(v) for v in os.environ.get("THETA", "1.0,0.1,0.5").split(","))
ctx = ex.Context(device=0)
for n in ns:
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
    r = ctx.loglik_dev(X, Y, Z, THETA)
    t0 = time.time()
    r = ctx.loglik_dev(X, Y, Z, THETA)
    wall = time.time() - t0
    i = r.info
    tf = i["flops"] / (i["ms_chol"] * 1e-3) / 1e12
    print(f"n={n} nb={i['nb']} ll={r.loglik:.10e} total={i['ms_total']:.1f}ms gen={i['ms_gen']:.2f} "
          f"chol={i['ms_chol']:.1f} red={i['ms_reduce']:.2f} chol_TF={tf:.2f} wall={wall:.2f}s kernels={i['kernels']}",
          flush=True)
