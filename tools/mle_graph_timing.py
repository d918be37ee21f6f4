import sys, time, math, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1708_02835_b200 as ex
import synth_inputs as si
n = 1600
x, y = ex.gen_locations(n, 1)
lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
start = tuple(math.sqrt(a * b) for a, b in zip(lo, hi))
for g in (-1, 1, -1, 1):
    with ex.Context(device=0, graphs=g) as c:
        z = c.simulate(x, y, si.normals(n, 1), (1.0, 0.1, 0.5))
        t0 = time.perf_counter()
        th, ll, ne, tr = c.mle(x, y, z, lo, hi, start, xtol_rel=1e-6, max_evals=2000)
        dt = time.perf_counter() - t0
        t1 = time.perf_counter()
        for _ in range(50):
            r = c.loglik(x, y, z, (1.0, 0.1, 0.5))
        dt2 = (time.perf_counter() - t1) / 50
        print(f"graphs={g}: mle {ne} evals {dt:.3f}s = {1e3*dt/ne:.3f} ms/eval; loglik(host) {1e3*dt2:.3f} ms, device {r.info['ms_total']:.3f} ms; nonPD evals {int(np.sum(~np.isfinite(tr[:,3])))}")
