"""BASELINE configs[4] on one GPU: MLE on 90% of an n-site synthetic field, kriging of the
held-out 10%, MSE against the truth.

    python tools/config5.py --n 160000 [--max-evals 60] [--xtol 1e-3] [--full] > out.json

Field: jittered grid (R1-R3), z = L(theta_true) e by exageo_simulate (Alg. 1); the hold-out
set is the m = n/10 sites with the smallest keys of the SplitMix64 hold-out substream
(synth_inputs.holdout_mask). The MLE profiles theta1 out (--full: 3-D search) and uses the
quadratic-model trust region (--method nelder-mead for the simplex search) from the geometric
midpoint of the bounds; prediction is exageo_predict_var at
theta_hat (mean and kriging variance; the mean variance is the expected MSE
(1/m) tr(Sigma11 - Sigma12 Sigma22^-1 Sigma21)) and exageo_predict at theta_true. Configs[4] names 8 GPUs; at n = 160k the
observed 144k x 144k lower triangle (83 GB) fits one B200, so this runs on one.
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
    ap.add_argument("--n", type=int, default=160_000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-evals", type=int, default=60)
    ap.add_argument("--xtol", type=float, default=1e-3)
    ap.add_argument("--full", action="store_true", help="3-D search instead of the profiled one")
    ap.add_argument("--method", default="trust-region", choices=["trust-region", "nelder-mead"])
    a = ap.parse_args()
    theta_true = (1.0, 0.1, 0.5)
    lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
    start = tuple(math.sqrt(p * q) for p, q in zip(lo, hi))
    n, m = a.n, a.n // 10
    out = {"config": "BASELINE configs[4] (1 GPU)", "n": n, "m_holdout": m, "theta_true": theta_true,
           "bounds": [lo, hi], "start": start, "xtol_rel": a.xtol, "max_evals": a.max_evals,
           "search": ("3-D" if a.full else "theta1 profiled") + " / " + a.method}
    x, y = ex.gen_locations(n, a.seed)
    with ex.Context(device=0) as c:
        t0 = time.perf_counter()
        z = c.simulate(x, y, si.normals(n, a.seed), theta_true)
        out["simulate_s"] = time.perf_counter() - t0
        hold = si.holdout_mask(n, m, a.seed)
        xo, yo, zo = x[~hold], y[~hold], z[~hold]
        t0 = time.perf_counter()
        th, ll, ne, trace = c.mle(xo, yo, zo, lo, hi, start, xtol_rel=a.xtol, max_evals=a.max_evals,
                                  profile=not a.full, method=a.method)
        sec = time.perf_counter() - t0
        out.update({"theta_hat": th, "loglik": ll, "evals": ne, "mle_s": sec, "s_per_eval": sec / max(ne, 1),
                    "budget_exhausted": ne >= a.max_evals, "trace": trace.tolist()})
        for tag, t in (("theta_hat", th), ("theta_true", theta_true)):
            t0 = time.perf_counter()
            if tag == "theta_hat":  # mean and kriging variance: expected MSE = mean variance
                pred, var = c.predict_var(xo, yo, zo, x[hold], y[hold], t)
                out["expected_mse_theta_hat"] = float(np.mean(var))
            else:
                pred = c.predict(xo, yo, zo, x[hold], y[hold], t)
            out[f"predict_s_{tag}"] = time.perf_counter() - t0
            out[f"mse_{tag}"] = float(np.mean((pred - z[hold]) ** 2))
        out["var_z_holdout"] = float(np.var(z[hold]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
