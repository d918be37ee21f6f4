"""Oracle MLE pins: the estimate maximises l -- profile identity
theta1_hat = z^T R(theta2_hat, theta3_hat)^{-1} z / n (closed-form stationarity in theta1
from Eq. (1)), coordinate-wise local maximum, bounds respected -- at a small n and for
the stored golden estimate of tests/golden/mle_n400.json (tools/make_golden_mle.py)."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth_inputs as si

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mle_n400.json")


def _is_local_max(x, y, z, th, ll, rel=2e-3):
    for p in range(3):
        for s in (1 - rel, 1 + rel):
            t = list(th)
            t[p] *= s
            if oracle.loglik(x, y, z, t)[0] > ll + 1e-9 * abs(ll):
                return False
    return True


def test_oracle_mle_small():
    n = 120
    x, y = oracle.gen_locations(n, 3)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.7), si.normals(n, 3))
    lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
    th, ll, ne = oracle.mle(x, y, z, lo, hi, (0.3, 0.2, 0.6))
    assert all(a <= t <= b for a, t, b in zip(lo, th, hi))
    assert ll == pytest.approx(oracle.loglik(x, y, z, th)[0], rel=1e-14)
    assert th[0] == pytest.approx(oracle.profile_sigma2(x, y, z, th[1], th[2]), rel=1e-5)
    assert _is_local_max(x, y, z, th, ll)


def test_golden_mle_is_the_maximum():
    g = json.load(open(GOLDEN))
    x, y = oracle.gen_locations(g["n"], g["seed"])
    z = oracle.simulate(x, y, tuple(g["theta_true"]), si.normals(g["n"], g["seed"]))
    th = tuple(g["theta_hat"])
    ll = oracle.loglik(x, y, z, th)[0]
    assert ll == pytest.approx(g["loglik"], rel=1e-13)
    assert th[0] == pytest.approx(oracle.profile_sigma2(x, y, z, th[1], th[2]), rel=1e-6)
    assert _is_local_max(x, y, z, th, ll, rel=1e-3)
