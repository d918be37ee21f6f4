import sys; sys.path.insert(0, ".")
import torch, paper_1708_02835_b200 as ex, synth_inputs as si
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x, y = ex.gen_locations(n, 1); z = si.normals(n, 2)
X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
with ex.Context(device=0, graphs=-1) as c:
    for _ in range(2): c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
