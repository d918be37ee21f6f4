"""Tail hand-off sweep (development aid): evaluation time at n for EXAGEO_TAIL_N values; one
process per value (the threshold is read once). Usage: tail_sweep.py n nb v1,v2,..."""
import os
import subprocess
import sys

n, nb = sys.argv[1], sys.argv[2]
for v in sys.argv[3].split(","):
    env = dict(os.environ, EXAGEO_TAIL_N=v)
    code = ("import sys; sys.path.insert(0, '.'); import torch, paper_1708_02835_b200 as ex, synth_inputs as si\n"
            f"n, nb = {n}, {nb}\nx, y = ex.gen_locations(n, 1); z = si.normals(n, 2)\n"
            "X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))\n"
            "with ex.Context(device=0, nb=nb) as c:\n"
            "    c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))\n"
            "    t = sorted(c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5)).info['ms_total'] for _ in range(5))[2]\n"
            "print(f'n={n} nb={nb} tail_n=" + v + " {t:.3f} ms {n**3/3/t/1e9:.2f} TF', flush=True)\n")
    subprocess.run([sys.executable, "-c", code], env=env, check=False)
