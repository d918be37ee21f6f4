import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1708_02835_b200 as ex
import synth_inputs as si
TH = (1.0, 0.1, 0.5)
n, m = 20000, 2000
x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
rng = np.random.default_rng(0)
xn, yn = rng.random(m), rng.random(m)
with ex.Context(device=0) as c:
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        t1 = time.perf_counter()
        mean2, var = c.predict_var(x, y, z, xn, yn, TH)
        t2 = time.perf_counter()
        print(f"predict_var {t2-t1:.3f}s", flush=True)
