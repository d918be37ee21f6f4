#!/usr/bin/env python3
"""Cholesky time of exageo_loglik_dev (info.ms_chol: the tiled factorization with the fused
forward solve, generation excluded) against cuSOLVER potrf (torch.linalg.cholesky, float64)
at the same n on the same box. Context for DESIGN §6 / VERDICT item 4; vendor code is a
yardstick here and never part of the product path.

    python tools/chol_vs_vendor.py [n ...]     (default 8192 10000 16384 20000 32768 40000)
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402


def ours(n, reps=5):
    x, y = ex.gen_locations(n, 1)
    d = torch.device("cuda")
    xd, yd = torch.from_numpy(x).to(d), torch.from_numpy(y).to(d)
    zd = torch.from_numpy(si.normals(n, 1)).to(d)
    with ex.Context(device=0) as c:
        r = None
        for _ in range(2):
            r = c.loglik_dev(xd, yd, zd, (1.0, 0.1, 0.5))
        chol, tot = [], []
        for _ in range(reps):
            r = c.loglik_dev(xd, yd, zd, (1.0, 0.1, 0.5))
            chol.append(r.info["ms_chol"])
            tot.append(r.info["ms_total"])
        return statistics.median(chol), statistics.median(tot), int(r.info["nb"])


def cusolver(n, reps=3):
    d = torch.device("cuda")
    m = torch.randn(n, n, dtype=torch.float64, device=d)
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device=d)
    del m
    torch.linalg.cholesky(a)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.linalg.cholesky(a)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del a
    torch.cuda.empty_cache()
    return statistics.median(ts)


def main():
    ns = [int(v) for v in sys.argv[1:]] or [8192, 10000, 16384, 20000, 32768, 40000]
    for n in ns:
        f = n ** 3 / 3
        mc, mt, nb = ours(n)
        mv = cusolver(n)
        print(json.dumps({"n": n, "nb": nb, "exageo_ms_chol": round(mc, 3), "exageo_tf_chol": round(f / mc / 1e9, 2),
                          "exageo_ms_eval": round(mt, 3), "exageo_tf_eval": round(f / mt / 1e9, 2),
                          "cusolver_ms": round(mv, 3), "cusolver_tf": round(f / mv / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
