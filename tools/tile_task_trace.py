"""Run one executor evaluation with EXAGEO_TILE_TASK_TRACE set and summarise the trace:
critical chain timing per step (POTRF k ready/done, TRSM(k+1,k), SYRK(k+1,k+1,k)), mean
durations per task type, and the idle (waiting) share. Usage: tile_task_trace.py n [nb]"""
import os
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
path = os.path.join(tempfile.gettempdir(), f"tt_trace_{n}.txt")
os.environ["EXAGEO_TILE_TASK_TRACE"] = path

import torch  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
with ex.Context(device=0, tile_tasks=1, graphs=-1) as c:
    for _ in range(3):
        r = c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
    print(f"n={n} device {1e3 * r.info['ms_total']:.1f} us (chol {1e3 * r.info['ms_chol']:.1f} us)")
rows = [list(map(int, l.split())) for l in open(path) if not l.startswith("#")]
rows = [r for r in rows if r[8] > 0]
names = {0: "POTRF", 1: "TRSM", 2: "GEMM", 3: "ZTRSM", 4: "ZGEMM", 5: "GEN"}
nt = (n + 63) // 64
ntasks = len([r for r in rows if r[0] < len(rows)]) if False else None
chain_first = max(r[0] for r in rows) + 1 - 3 * nt  # chain records follow the ticket list
dur = defaultdict(list)
wait = defaultdict(list)
chain = {}
end = 0
for t, ty, i, j, k, cta, g, rd, d in rows:
    end = max(end, d)
    if t >= chain_first:
        chain[(ty, k)] = (g, rd, d)
        continue
    dur[ty].append(d - rd)
    wait[ty].append(rd - g)
print(f"kernel span {end / 1e3:.1f} us, {len(rows)} records")
for ty in sorted(dur):
    v = dur[ty]
    print(f"  pool {names[ty]:6s} n={len(v):6d} exec mean {sum(v) / len(v) / 1e3:7.2f} us  max {max(v) / 1e3:7.2f}  "
          f"wait mean {sum(wait[ty]) / len(v) / 1e3:7.2f} us")
print("chain step: [start, after wait/prefetch issue, done] in us for POTRF | TRSM (wait..mma start..done) | SYRK")
for k in range(min(nt, 40)):
    cells = []
    for ty in (0, 1, 2):
        e = chain.get((ty, k))
        cells.append(f"{e[0] / 1e3:8.2f} {e[1] / 1e3:8.2f} {e[2] / 1e3:8.2f}" if e else " " * 26)
    print(f"{k:4d}  " + " | ".join(cells))
# the pool tasks that feed chain step k: TRSM(k+1, k-1) and the last updates of A_{k+1,k}, A_{k+1,k+1}
print("feeders of step k: ticket [grab, ready, done] us for TRSM(k+1,k-1) | GEMM(k+1,k,k-1) | GEMM(k+1,k+1,k-1)")
pool = {(ty, i, j, k): (t, g, rd, d) for t, ty, i, j, k, cta, g, rd, d in rows if t < chain_first}
for k in range(1, min(nt - 1, 16)):
    cells = []
    for key in ((1, k + 1, k - 1, k - 1), (2, k + 1, k, k - 1), (2, k + 1, k + 1, k - 1)):
        e = pool.get(key)
        cells.append(f"#{e[0]:5d} {e[1] / 1e3:7.2f} {e[2] / 1e3:7.2f} {e[3] / 1e3:7.2f}" if e else " " * 30)
    print(f"{k:4d}  " + " | ".join(cells))
