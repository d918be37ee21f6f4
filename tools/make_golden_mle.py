#!/usr/bin/env python3
"""Write tests/golden/mle_n400.json: the ORACLE's maximum-likelihood estimate on
BASELINE configs[0]'s field (n = 400 jittered grid, z = L(theta_true) e, seed 1),
bounds of DESIGN R16, start = geometric midpoint. Calls only oracle/ (whose MLE uses
scipy optimisers as steps) and the shared input generator."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth_inputs as si  # noqa: E402

N, SEED, THETA = 400, 1, (1.0, 0.1, 0.5)
LO, HI = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)


def main():
    x, y = oracle.gen_locations(N, SEED)
    z = oracle.simulate(x, y, THETA, si.normals(N, SEED))
    start = tuple(math.sqrt(a * b) for a, b in zip(LO, HI))
    t = time.time()
    th, ll, ne = oracle.mle(x, y, z, LO, HI, start)
    out = {"n": N, "seed": SEED, "theta_true": THETA, "lo": LO, "hi": HI, "start": start,
           "theta_hat": th, "loglik": ll, "oracle_evals": ne, "seconds": time.time() - t,
           "source": "tools/make_golden_mle.py (oracle.mle: scipy Nelder-Mead + L-BFGS-B on oracle.loglik)"}
    path = os.path.join(ROOT, "tests", "golden", "mle_n400.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
