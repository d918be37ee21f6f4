"""Monte-Carlo replicas of the configs[1] MLE (n = 1600 jittered grid, theta = (1, 0.1, nu)):
R independent fields z = L e (seeds 1..R), theta_hat by the profiled trust-region MLE; the
paper's statistical check (boxplots of theta_hat around the truth).

    python tools/mc_replicas.py [--reps 50] [--nu 0.5] > profiles/r01_mc_replicas_nu0.5.json
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_1708_02835_b200 as ex
import synth_inputs as si


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--n", type=int, default=1600)
    ap.add_argument("--nu", type=float, default=0.5)
    a = ap.parse_args()
    truth = (1.0, 0.1, a.nu)
    lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
    start = tuple(math.sqrt(p * q) for p, q in zip(lo, hi))
    x, y = ex.gen_locations(a.n, 1)
    est, evals = [], []
    t0 = time.perf_counter()
    with ex.Context(device=0) as c:
        for r in range(1, a.reps + 1):
            z = c.simulate(x, y, si.normals(a.n, 1000 + r), truth)
            th, ll, ne, _ = c.mle(x, y, z, lo, hi, start, xtol_rel=1e-6, max_evals=500, profile=True,
                                  method="trust-region")
            est.append(th)
            evals.append(ne)
    est = np.array(est)
    q = {name: np.percentile(est[:, i], [5, 25, 50, 75, 95]).tolist() for i, name in enumerate(("sigma2", "beta", "nu"))}
    print(json.dumps({"n": a.n, "truth": truth, "reps": a.reps, "seconds": time.perf_counter() - t0,
                      "evals_median": float(np.median(evals)), "quantiles_5_25_50_75_95": q,
                      "theta_hat": est.tolist()}))


if __name__ == "__main__":
    main()
