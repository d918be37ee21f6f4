#!/usr/bin/env python3
"""Write tests/golden/loglik_n{N}.json (+ z_n{N}.npy): the ORACLE's exact log-likelihood
on the paper's 2-D jittered grid at sizes the GPU parity tests cannot afford to recompute.

Workload (P:842-847 the jittered grid, Alg. 1 P:604-648 the field, Alg. 2
P:674-689 the evaluation): locations oracle.gen_locations(N, seed=1), e = synth normals
(seed 1), z = L(theta_true) e by oracle.simulate at theta_true = (1, 0.1, 0.5); then
l(theta) = oracle.loglik for theta in {(1, 0.1, 0.5), (1, 0.1, 0.8)} (the paper's
Monte-Carlo theta and a general-nu case that exercises the K_nu series path).

Calls only oracle/ and the shared input generator; every stored number is the oracle's.
The measured oracle seconds, thread count and CPU model are stored with each value so
bench.py can quote a measured (not extrapolated) oracle time."""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth_inputs as si  # noqa: E402

SEED = 1
THETA_TRUE = (1.0, 0.1, 0.5)
THETAS = [(1.0, 0.1, 0.5), (1.0, 0.1, 0.8)]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[20000, 40000])
    args = ap.parse_args()
    for n in args.n:
        x, y = oracle.gen_locations(n, SEED)
        e = si.normals(n, SEED)
        t0 = time.time()
        z = oracle.simulate(x, y, THETA_TRUE, e)
        t_sim = time.time() - t0
        np.save(os.path.join(ROOT, "tests", "golden", f"z_n{n}.npy"), z)
        cases = []
        for th in THETAS:
            t0 = time.time()
            ll, ld, q = oracle.loglik(x, y, z, th)
            dt = time.time() - t0
            cases.append({"theta": list(th), "loglik": ll, "logdet": ld, "quad": q, "oracle_seconds": dt})
            print(f"n={n} theta={th} l={ll!r} ({dt:.0f} s)", flush=True)
            write(n, t_sim, cases)  # after every case: a long run keeps what it finished


def write(n, t_sim, cases):
    out = {
        "n": n, "seed": SEED, "theta_true": list(THETA_TRUE),
        "locations": "oracle.gen_locations(n, seed) (jittered grid, DESIGN R1-R3)",
        "z": f"z_n{n}.npy = oracle.simulate(x, y, theta_true, synth_inputs.normals(n, seed))",
        "simulate_seconds": t_sim, "cases": cases,
        "oracle_threads": oracle.num_threads(), "cpu_model": cpu_model(), "host": platform.node(),
        "source": "tools/make_golden_large.py (oracle.simulate + oracle.loglik only)",
    }
    path = os.path.join(ROOT, "tests", "golden", f"loglik_n{n}.json")
    with open(path + ".tmp", "w") as f:
        json.dump(out, f, indent=1)
    os.replace(path + ".tmp", path)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
