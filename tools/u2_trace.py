"""Per-step timeline of the stream schedule at one n (env EXAGEO_U2_TRACE): each bulk trailing
update U2(k)'s duration and the gap before it (time the trailing update waited for the panel
chain F(k+1) / U1(k)). Usage: u2_trace.py n [nb] [tile_tasks] (default -1: no executor tail; 0: the
automatic tail hand-off, whose time is then part of "after last U2")"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1])
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tt = int(sys.argv[3]) if len(sys.argv) > 3 else -1
path = os.path.join(tempfile.gettempdir(), f"u2_{n}_{nb}.txt")
if os.path.exists(path):
    os.remove(path)
os.environ["EXAGEO_U2_TRACE"] = path
import torch  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
with ex.Context(device=0, nb=nb, graphs=-1, tile_tasks=tt) as c:
    for _ in range(3):
        r = c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
blocks = open(path).read().split("# ")[1:]
last = blocks[-1].strip().splitlines()
rows = [tuple(map(float, l.split()[1:])) for l in last[1:] if not l.startswith("end")]
end = float(last[-1].split()[1])
print(last[0], f"chol {end:.3f} ms, TF {n ** 3 / 3 / end / 1e9:.2f}")
prev = 0.0
gap_sum = 0.0
busy = 0.0
for k, (b, e) in enumerate(rows):
    gap = b - prev
    gap_sum += gap
    busy += e - b
    m = n - (k + 2) * r.info["nb"]
    fl = r.info["nb"] * max(m, 0) ** 2
    print(f"k={k:3d} m={m:6d} gap {1e3 * gap:8.1f} us  U2 {1e3 * (e - b):9.1f} us  {fl / max(e - b, 1e-9) / 1e9:6.1f} TF")
    prev = e
print(f"U2 busy {busy:.3f} ms, gaps {gap_sum:.3f} ms, after last U2 {end - prev:.3f} ms")
