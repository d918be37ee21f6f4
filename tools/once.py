"""Two evaluations at (n, nb) through the stream schedule, graphs off (profiling target).
Usage: once.py n [nb] [tile_tasks]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

n = int(sys.argv[1])
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tt = int(sys.argv[3]) if len(sys.argv) > 3 else -1
x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
with ex.Context(device=0, nb=nb, graphs=-1, tile_tasks=tt) as c:
    for _ in range(int(__import__("os").environ.get("EVALS", "2"))):
        c.loglik_dev(X, Y, Z, tuple(float(v) for v in __import__("os").environ.get("THETA", "1.0,0.1,0.5").split(",")))
