"""Oracle pins: unblocked Cholesky, substitutions, Alg. 1-3 -- CPU only.

Pinned against hand cases, the identity L L^T = Sigma,
exact rational determinants, closed-form likelihoods (n=1, n=2, AR(1)/KMS,
Sigma = theta1 I), permutation invariance, and independent library routines
(numpy.linalg / scipy.stats.multivariate_normal).
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg
import scipy.stats

import oracle
import synth_inputs as si
from tests._golden import load

G = load()
LOG2PI = math.log(2 * math.pi)


def test_cholesky_hand_case():
    L = oracle.cholesky([[4.0, 2.0], [2.0, 3.0]])
    np.testing.assert_allclose(L, [[2.0, 0.0], [1.0, math.sqrt(2.0)]], rtol=1e-15)
    assert 2 * np.log(np.diag(L)).sum() == pytest.approx(G["logdet_4_2_2_3"], abs=5e-8)


def test_cholesky_not_pd():
    with pytest.raises(oracle.NotPositiveDefinite) as ei:
        oracle.cholesky([[1.0, 2.0], [2.0, 1.0]])
    assert ei.value.pivot == 1


def test_cholesky_identity_and_scaled_identity():
    n = 37
    L = oracle.cholesky(np.eye(n) * 2.5)
    np.testing.assert_allclose(L, np.eye(n) * math.sqrt(2.5), rtol=1e-15)
    assert 2 * np.log(np.diag(L)).sum() == pytest.approx(n * math.log(2.5), rel=1e-14)


@pytest.mark.parametrize("nu", [0.5, 1.0, 1.7])
def test_cholesky_reconstructs_matern(nu):
    x, y = oracle.gen_locations(300, 3)
    S = oracle.cov(x, y, x, y, (1.3, 0.1, nu))
    L = oracle.cholesky(S)
    rel = np.linalg.norm(L @ L.T - S) / np.linalg.norm(S)
    assert rel < 1e-14
    assert np.all(np.diag(L) > 0)


def _exact_det(A):
    """Determinant by fraction-exact Gaussian elimination (no rounding at all)."""
    M = [[Fraction(float(v)) for v in row] for row in A]
    n = len(M)
    det = Fraction(1)
    for j in range(n):
        p = next(i for i in range(j, n) if M[i][j] != 0)
        if p != j:
            M[j], M[p] = M[p], M[j]
            det = -det
        det *= M[j][j]
        for i in range(j + 1, n):
            f = M[i][j] / M[j][j]
            for k in range(j, n):
                M[i][k] -= f * M[j][k]
    return det


@pytest.mark.parametrize("n,nu", [(3, 0.5), (5, 1.0), (6, 2.5), (7, 0.8)])
def test_logdet_vs_exact_rational_determinant(n, nu):
    x, y = oracle.gen_locations(n, 11 + n)
    theta = (1.4, 0.3, nu)
    S = oracle.cov(x, y, x, y, theta)
    det = _exact_det(S)
    assert det > 0
    logdet_exact = math.log(det.numerator) - math.log(det.denominator)
    z = si.normals(n, 5)
    ll, logdet, quad = oracle.loglik(x, y, z, theta)
    assert logdet == pytest.approx(logdet_exact, rel=1e-12, abs=1e-12)


def test_forward_backward_vs_library():
    x, y = oracle.gen_locations(200, 9)
    S = oracle.cov(x, y, x, y, (1.0, 0.1, 1.0))
    L = oracle.cholesky(S)
    z = si.normals(200, 1)
    np.testing.assert_allclose(oracle.forward(L, z), scipy.linalg.solve_triangular(L, z, lower=True), rtol=1e-10)
    np.testing.assert_allclose(oracle.backward(L, z), scipy.linalg.solve_triangular(L.T, z, lower=False), rtol=1e-10)


def test_loglik_golden_and_n1():
    ll, logdet, quad = oracle.loglik([0.3], [0.4], [0.0], (1.0, 0.1, 0.5))
    assert ll == pytest.approx(G["loglik_n1_z0_s1"], abs=5e-8)
    for t1, z in [(2.0, 1.0), (0.37, -2.2)]:
        ll, _, _ = oracle.loglik([0.3], [0.4], [z], (t1, 0.1, 1.3))
        assert ll == pytest.approx(-0.5 * LOG2PI - 0.5 * math.log(t1) - z * z / (2 * t1), rel=1e-15)


@pytest.mark.parametrize("nu", [0.5, 1.0, 2.5])
def test_loglik_n2_closed_form(nu):
    x, y = [0.1, 0.16], [0.2, 0.28]  # r = 0.1
    t1, t2 = 1.7, 0.1
    rho = oracle.matern(0.1, (1.0, t2, nu))
    z1, z2 = 1.0, -0.5
    logdet = 2 * math.log(t1) + math.log(1 - rho * rho)
    quad = (z1 * z1 - 2 * rho * z1 * z2 + z2 * z2) / (t1 * (1 - rho * rho))
    ll, ld, qd = oracle.loglik(x, y, [z1, z2], (t1, t2, nu))
    assert ld == pytest.approx(logdet, rel=1e-14)
    assert qd == pytest.approx(quad, rel=1e-14)
    assert ll == pytest.approx(-LOG2PI - 0.5 * logdet - 0.5 * quad, rel=1e-14)


def kms_loglik(z, t1, rho):
    """AR(1) / Kac-Murdock-Szego closed form: Sigma_ij = t1 rho^|i-j|."""
    n = z.size
    logdet = n * math.log(t1) + (n - 1) * math.log1p(-rho * rho)
    y = np.empty(n)
    y[0] = z[0] / math.sqrt(t1)
    y[1:] = (z[1:] - rho * z[:-1]) / math.sqrt(t1 * (1 - rho * rho))
    quad = float(np.dot(y, y))
    return -0.5 * quad - 0.5 * logdet - 0.5 * n * LOG2PI, logdet, quad


def test_loglik_ar1_kms_closed_form():
    n, h, t1, t2 = 700, 2.0**-12, 1.7, 0.05
    x, y = si.collinear_sites(n, h)
    z = si.normals(n, 21)
    rho = math.exp(-h / t2)
    ref = kms_loglik(z, t1, rho)
    got = oracle.loglik(x, y, z, (t1, t2, 0.5))
    for a, b in zip(got, ref):
        assert a == pytest.approx(b, rel=1e-11)


def test_loglik_identity_covariance():
    n, t1 = 257, 2.3
    x, y = si.spread_sites(n, 100.0)  # r/theta2 >= 1000: exp underflows exactly to 0
    z = si.normals(n, 4)
    ll, logdet, quad = oracle.loglik(x, y, z, (t1, 0.1, 1.5))
    assert logdet == pytest.approx(n * math.log(t1), rel=1e-15)
    assert quad == pytest.approx(float(np.dot(z, z)) / t1, rel=1e-14)


def test_loglik_permutation_invariance_and_library():
    n = 400
    x, y = oracle.gen_locations(n, 1)
    theta = (1.0, 0.1, 1.0)
    z = si.normals(n, 2)
    ll = oracle.loglik(x, y, z, theta)[0]
    p = np.random.default_rng(0).permutation(n)
    llp = oracle.loglik(x[p], y[p], z[p], theta)[0]
    assert llp == pytest.approx(ll, rel=1e-12)
    S = oracle.cov(x, y, x, y, theta)
    ref = scipy.stats.multivariate_normal(mean=np.zeros(n), cov=S).logpdf(z)
    assert ll == pytest.approx(ref, rel=1e-10)


def test_loglik_scaling_identity():
    # l(c theta1; sqrt(c) z) = l(theta1; z) - (n/2) log c
    n, c = 150, 3.7
    x, y = oracle.gen_locations(n, 8)
    z = si.normals(n, 8)
    a = oracle.loglik(x, y, z, (1.0, 0.2, 0.9))[0]
    b = oracle.loglik(x, y, z * math.sqrt(c), (c, 0.2, 0.9))[0]
    assert b == pytest.approx(a - 0.5 * n * math.log(c), rel=1e-12)


def test_simulate_solve_recovers_e():
    n = 300
    x, y = oracle.gen_locations(n, 5)
    theta = (1.0, 0.1, 0.5)
    e = si.normals(n, 6)
    z = oracle.simulate(x, y, theta, e)
    S = oracle.cov(x, y, x, y, theta)
    L = np.linalg.cholesky(S)
    np.testing.assert_allclose(z, L @ e, rtol=1e-10, atol=1e-12)
    _, _, quad = oracle.loglik(x, y, z, theta)
    assert quad == pytest.approx(float(e @ e), rel=1e-10)


def test_predict_kriging():
    n = 200
    x, y = oracle.gen_locations(n, 12)
    theta = (1.0, 0.1, 1.0)
    z = si.normals(n, 13)
    # Eq. (5) is an interpolator: predicting at an observed site returns its value
    idx = [3, 77, 150]
    got = oracle.predict(x, y, z, x[idx], y[idx], theta)
    np.testing.assert_allclose(got, z[idx], rtol=1e-8, atol=1e-8)
    # vs. numpy explicit solve Z1 = S12 S22^{-1} Z2
    xn, yn = np.array([0.5, 0.123, 0.9]), np.array([0.5, 0.77, 0.05])
    S22 = oracle.cov(x, y, x, y, theta)
    S12 = oracle.cov(xn, yn, x, y, theta)
    ref = S12 @ np.linalg.solve(S22, z)
    np.testing.assert_allclose(oracle.predict(x, y, z, xn, yn, theta), ref, rtol=1e-9, atol=1e-12)
    # far away -> prior mean 0
    far = oracle.predict(x, y, z, [1e4], [1e4], theta)
    assert far[0] == 0.0


def test_predict_var_pins():
    # oracle.predict_var: simple-kriging variance C(0) - sigma^T Sigma^{-1} sigma
    theta = (1.3, 0.1, 0.8)
    # n = 1: closed form theta1 - C(r)^2 / theta1
    x, y = np.array([0.2]), np.array([0.3])
    xn, yn = np.array([0.25, 0.9]), np.array([0.31, 0.1])
    got = oracle.predict_var(x, y, xn, yn, theta)
    for i in range(2):
        c = oracle.matern(math.hypot(xn[i] - 0.2, yn[i] - 0.3), theta)
        assert got[i] == pytest.approx(theta[0] - c * c / theta[0], rel=1e-13)
    # brute force with numpy's dense solve (independent of the oracle's Cholesky)
    xs, ys = oracle.gen_locations(30, 3)
    xn, yn = np.array([0.5, 0.01, 0.77]), np.array([0.5, 0.99, 0.2])
    S22 = oracle.cov(xs, ys, xs, ys, theta)
    s = oracle.cov(xs, ys, xn, yn, theta)
    ref = theta[0] - np.einsum("ij,ij->j", s, np.linalg.solve(S22, s))
    np.testing.assert_allclose(oracle.predict_var(xs, ys, xn, yn, theta), ref, rtol=1e-9, atol=1e-12)
    # an observed site has zero variance; a far site has the prior variance theta1
    v = oracle.predict_var(xs, ys, [xs[4], 1e4], [ys[4], 1e4], theta)
    assert abs(v[0]) < 1e-10 and v[1] == theta[0]
