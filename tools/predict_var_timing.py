"""Timing of exageo_predict_var (kriging mean + variance) vs exageo_predict (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_1708_02835_b200 as ex
import synth_inputs as si

TH = (1.0, 0.1, 0.5)
for n, m in [(20000, 2000), (60000, 4000)]:
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    rng = np.random.default_rng(0)
    xn, yn = rng.random(m), rng.random(m)
    with ex.Context(device=0) as c:
        c.predict_var(x, y, z, xn[:10], yn[:10], TH)  # warm-up (module loading, allocations)
        for rep in range(2):
            t0 = time.perf_counter()
            mean = c.predict(x, y, z, xn, yn, TH)
            t1 = time.perf_counter()
            mean2, var = c.predict_var(x, y, z, xn, yn, TH)
            t2 = time.perf_counter()
            extra = (t2 - t1) - (t1 - t0)
            print(f"n={n} m={m}: predict {t1 - t0:.3f} s, predict_var {t2 - t1:.3f} s (variance part {extra:.3f} s"
                  f" = {n * n * m / extra / 1e12:.1f} TF of n^2 m); var range [{var.min():.3e}, {var.max():.3e}]",
                  flush=True)
