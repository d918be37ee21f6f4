"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once at n ~ 1000 (loglik single + virtual ranks, simulate, predict, mle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

n = 1000
x, y = ex.gen_locations(n, 1)
e = si.normals(n, 2)
with ex.Context(device=0, nb=128) as c:
    z = c.simulate(x, y, e, (1.0, 0.1, 0.5))
    r = c.loglik(x, y, z, (1.0, 0.1, 0.8))
    p = c.predict(x, y, z, np.array([0.3, 0.7]), np.array([0.2, 0.9]), (1.0, 0.1, 0.8))
    th, ll, ne, _ = c.mle(x[:200], y[:200], z[:200], (0.1, 0.01, 0.2), (5.0, 1.0, 2.0), (1.0, 0.1, 0.5),
                          xtol_rel=1e-3, max_evals=30)
with ex.Context(device=0, nb=128, virtual_ranks=3) as c:
    r3 = c.loglik(x, y, z, (1.0, 0.1, 0.8))
with ex.Context(device=0, nb=256) as c:
    r4 = c.loglik(x, y, z, (1.0, 0.1, 1.7))
print("ok", r.loglik, r3.loglik, r4.loglik, p, th, ne)
