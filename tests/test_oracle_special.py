"""Oracle pins: Gamma, K_nu and the Matern function (Eq. 2) -- CPU only.

Pinned against closed forms, the three-term recurrence, the
golden SPEC/PAPER examples and an independent library (mpmath besselk/gamma).
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
from tests._golden import load

G = load()


def test_gamma_special_values():
    assert oracle.gamma(0.5) == pytest.approx(math.sqrt(math.pi), rel=1e-15)
    assert oracle.gamma(1.5) == pytest.approx(math.sqrt(math.pi) / 2, rel=1e-15)
    for k in range(1, 12):
        assert oracle.gamma(float(k)) == pytest.approx(math.factorial(k - 1), rel=1e-15)


@pytest.mark.parametrize("z", [0.1, 0.23, 0.5, 0.77, 1.3, 1.7, 2.0, 2.5, 3.9, 4.9])
def test_gamma_vs_mpmath(z):
    ref = float(mpmath.gamma(mpmath.mpf(z)))
    assert oracle.gamma(z) == pytest.approx(ref, rel=2e-15)


def test_bessel_golden():
    assert oracle.bessel_k(0.5, 1.0) == pytest.approx(G["bessel_k_0.5_at_1"], abs=5e-8)
    assert oracle.bessel_k(1.0, 1.0) == pytest.approx(G["bessel_k_1_at_1"], abs=5e-8)


@pytest.mark.parametrize("x", [1e-6, 1e-3, 0.1, 0.7, 1.0, 2.0, 5.0, 20.0, 100.0, 600.0])
def test_bessel_half_integer_closed_forms(x):
    pre = math.sqrt(math.pi / (2 * x)) * math.exp(-x)
    if pre == 0.0:
        pytest.skip("underflow")
    assert oracle.bessel_k(0.5, x) == pytest.approx(pre, rel=1e-14)
    assert oracle.bessel_k(1.5, x) == pytest.approx(pre * (1 + 1 / x), rel=1e-14)
    assert oracle.bessel_k(2.5, x) == pytest.approx(pre * (1 + 3 / x + 3 / x**2), rel=1e-14)


@pytest.mark.parametrize("nu", [0.3, 0.9, 1.2, 1.7, 2.2, 3.6])
@pytest.mark.parametrize("x", [1e-4, 0.05, 0.8, 1.9, 2.1, 7.5, 40.0])
def test_bessel_recurrence(nu, x):
    # K_{nu+1}(x) = K_{nu-1}(x) + (2 nu / x) K_nu(x)
    lhs = oracle.bessel_k(nu + 1, x)
    rhs = oracle.bessel_k(abs(nu - 1), x) + 2 * nu / x * oracle.bessel_k(nu, x)
    assert lhs == pytest.approx(rhs, rel=1e-13)


NUS = [0.1, 0.25, 0.5, 0.73, 1.0, 1.27, 1.5, 1.999, 2.5, 3.3, 4.9]
XS = [1e-6, 1e-3, 0.02, 0.3, 0.99, 1.5, 2.0, 2.01, 3.7, 10.0, 35.0, 120.0, 690.0]


@pytest.mark.parametrize("nu", NUS)
def test_bessel_vs_mpmath(nu):
    mpmath.mp.dps = 30
    for x in XS:
        ref = float(mpmath.besselk(mpmath.mpf(nu), mpmath.mpf(x)))
        if ref == 0.0 or ref < 1e-300:
            continue
        assert oracle.bessel_k(nu, x) == pytest.approx(ref, rel=5e-14), (nu, x)


def test_matern_golden():
    assert oracle.matern(0.1, (1.0, 0.1, 0.5)) == pytest.approx(G["matern_exp_r0.1"], abs=5e-8)
    assert oracle.matern(0.1, (1.0, 0.1, 1.0)) == pytest.approx(G["matern_whittle_r0.1"], abs=5e-8)


@pytest.mark.parametrize("theta", [(1.0, 0.1), (2.5, 0.03), (0.7, 1.3)])
def test_matern_reductions(theta):
    t1, t2 = theta
    for r in np.geomspace(1e-5, 3.0, 60):
        x = r / t2
        # nu = 1/2 -> exponential model
        assert oracle.matern(r, (t1, t2, 0.5)) == pytest.approx(t1 * math.exp(-x), rel=1e-14, abs=1e-300)
        # nu = 3/2, 5/2 closed forms in Eq. (2)'s parameterization (DESIGN R10)
        assert oracle.matern(r, (t1, t2, 1.5)) == pytest.approx(t1 * (1 + x) * math.exp(-x), rel=1e-14, abs=1e-300)
        assert oracle.matern(r, (t1, t2, 2.5)) == pytest.approx(
            t1 * (1 + x + x * x / 3) * math.exp(-x), rel=1e-14, abs=1e-300)
        # nu = 1 -> Whittle model theta1 (r/theta2) K_1(r/theta2)
        if x < 600:
            k1 = float(mpmath.besselk(1, x))
            assert oracle.matern(r, (t1, t2, 1.0)) == pytest.approx(t1 * x * k1, rel=1e-13)


def test_matern_limit_linearity_monotone():
    for nu in NUS:
        assert oracle.matern(0.0, (1.7, 0.1, nu)) == 1.7  # C(0) = theta1 (R9)
        # continuity at r -> 0
        # 1 - C(r)/theta1 = O(x^(2 min(nu,1))) (up to a log at nu = 1)
        x = 1e-8
        assert oracle.matern(x * 0.1, (1.0, 0.1, nu)) == pytest.approx(1.0, rel=20 * x ** (2 * min(nu, 0.95)))
        rs = np.linspace(1e-4, 2.0, 300)
        c = np.array([oracle.matern(r, (1.0, 0.1, nu)) for r in rs])
        assert np.all(np.diff(c) <= 0)
        c3 = np.array([oracle.matern(r, (3.0, 0.1, nu)) for r in rs])
        np.testing.assert_allclose(c3, 3.0 * c, rtol=1e-15)


def test_matern_vs_mpmath_general_nu():
    mpmath.mp.dps = 30
    for nu in [0.3, 0.8, 1.7, 2.2]:
        for r in [0.003, 0.05, 0.1, 0.29, 0.8]:
            x = mpmath.mpf(r) / mpmath.mpf(0.1)
            ref = x**nu * mpmath.besselk(nu, x) / (2 ** (nu - 1) * mpmath.gamma(nu))
            assert oracle.matern(r, (1.0, 0.1, nu)) == pytest.approx(float(ref), rel=5e-14)
