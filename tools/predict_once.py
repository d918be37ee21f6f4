"""One exageo_predict at n (default 100k) with m new sites (profiling target for K5^T / K8)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_1708_02835_b200 as ex
import synth_inputs as si

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
rng = np.random.default_rng(0)
with ex.Context(device=0) as c:
    t0 = time.perf_counter()
    out = c.predict(x, y, z, rng.random(m), rng.random(m), (1.0, 0.1, 0.5))
    print(f"predict n={n} m={m}: {time.perf_counter() - t0:.3f} s", flush=True)
