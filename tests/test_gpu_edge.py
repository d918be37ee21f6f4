"""GPU edge cases: tile-boundary sizes, extreme smoothness, near-singular covariances
(GPU and oracle must agree on failure or on the value), caller-owned workspace,
argument validation."""
import math

import numpy as np
import pytest

import oracle
import synth_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402

from tests._tol import assert_ll, r13_tol  # noqa: E402


@pytest.mark.parametrize("n,nb", [(128, 128), (256, 128), (257, 128), (383, 384), (385, 384), (511, 256),
                                  (513, 512), (64, 128), (1, 512)])
def test_tile_boundaries(n, nb):
    x, y = ex.gen_locations(n, n)
    z = si.normals(n, n + 1)
    theta = (1.1, 0.1, 0.9)
    with ex.Context(device=0, nb=nb) as c:
        r = c.loglik(x, y, z, theta)
    ll, ld, qd = oracle.loglik(x, y, z, theta)
    assert_ll(r.loglik, (ll, ld, qd), n, what=(n, nb))


@pytest.mark.parametrize("nu", [0.05, 0.12, 3.9, 4.9])
def test_extreme_smoothness(nu):
    n = 300
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    theta = (1.0, 0.02, nu)  # short range keeps smooth fields well conditioned
    with ex.Context(device=0) as c:
        try:
            r = c.loglik(x, y, z, theta)
        except ex.NotPositiveDefinite:
            with pytest.raises(oracle.NotPositiveDefinite):
                oracle.loglik(x, y, z, theta)
            return
    ll, ld, qd = oracle.loglik(x, y, z, theta)
    assert_ll(r.loglik, (ll, ld, qd), n, what=nu)


# ---- ill-conditioned Sigma over the MLE box (DESIGN §7 "conditioning") -------------------
# theta grid beta in {0.3, 1, 2}, nu in {1.5, 2}, n in {400, 1600}: cond(Sigma) from 1e6 to
# 1.6e13, every case numerically PD (lambda_min > 0 for the oracle's Cholesky). z is a
# field of the same theta (Alg. 1), as the MLE sees it. First-order perturbation of Eq. (1):
#   l(Sigma + E) - l(Sigma) = -1/2 tr(Sigma^-1 E) + 1/2 w^T E w,  w = Sigma^-1 z,
# and |tr(Sigma^-1 E)| <= ||E||_2 tr(Sigma^-1), |w^T E w| <= ||E||_2 ||w||^2. Each side carries
# a backward error ||E||_2 <= eta ||Sigma||_2 with eta = 5e-14 (entrywise generation budget,
# Sigma > 0 entrywise so || |E| ||_2 <= 5e-14 ||Sigma||_2) + 2 n u (Cholesky, u = 2^-53), so
#   |dlogdet| <= 2 eta ||Sigma|| tr(Sigma^-1),  |dquad| <= 2 eta ||Sigma|| ||w||^2,
#   |dl| <= eta ||Sigma|| (tr(Sigma^-1) + ||w||^2)    (GPU and oracle errors added).
U = 2.0**-53


def cond_bounds(x, y, z, theta):
    S = oracle.cov(x, y, x, y, theta)
    lam = np.linalg.eigvalsh(S)  # library eigen-solver: condition estimate only
    L = oracle.cholesky(S)
    w = oracle.backward(L, oracle.forward(L, z))
    n = len(z)
    eta = 5e-14 + 2 * n * U
    snorm, trinv, w2 = lam[-1], float(np.sum(1.0 / lam)), float(w @ w)
    return {"cond": lam[-1] / lam[0], "ld": 2 * eta * snorm * trinv, "qd": 2 * eta * snorm * w2,
            "ll": eta * snorm * (trinv + w2)}


@pytest.mark.parametrize("n", [400, 1600])
@pytest.mark.parametrize("beta", [0.3, 1.0, 2.0])
@pytest.mark.parametrize("nu", [1.5, 2.0])
def test_ill_conditioned_theta_grid(n, beta, nu):
    theta = (1.0, beta, nu)
    x, y = ex.gen_locations(n, 5)
    z = oracle.simulate(x, y, theta, si.normals(n, 6))
    b = cond_bounds(x, y, z, theta)
    ll, ld, qd = oracle.loglik(x, y, z, theta)
    with ex.Context(device=0) as c:
        r = c.loglik(x, y, z, theta)  # must succeed: the matrix is numerically PD
    dll, dld, dqd = abs(r.loglik - ll), abs(r.logdet - ld), abs(r.quad - qd)
    print(f"n={n} theta={theta} cond={b['cond']:.2e} |dl|={dll:.2e} (bound {b['ll']:.2e}) "
          f"|dlogdet|={dld:.2e} ({b['ld']:.2e}) |dquad|={dqd:.2e} ({b['qd']:.2e})")
    assert dll <= max(b["ll"], r13_tol(ll, ld, qd, n))
    assert dld <= max(b["ld"], 1e-10 * abs(ld))
    assert dqd <= max(b["qd"], 1e-10 * abs(qd))


@pytest.mark.parametrize("n,theta", [(400, (1.0, 3.0, 3.5)), (1600, (1.0, 2.0, 4.0))])
def test_numerically_singular_both_fail(n, theta):
    # cond(Sigma) far beyond 1/u: no fp64 Cholesky exists; both sides must report ENOTPD
    # with a pivot inside [0, n) (where exactly is decided by rounding in either order)
    x, y = ex.gen_locations(n, 5)
    z = si.normals(n, 6)
    with pytest.raises(oracle.NotPositiveDefinite) as eo:
        oracle.loglik(x, y, z, theta)
    with ex.Context(device=0) as c:
        with pytest.raises(ex.NotPositiveDefinite) as eg:
            c.loglik(x, y, z, theta)
        # the context recovers for the next evaluation
        r = c.loglik(x, y, z, (1.0, 0.1, 0.5))
        assert np.isfinite(r.loglik)
    print(f"n={n} theta={theta} pivots gpu={eg.value.pivot} oracle={eo.value.pivot}")
    assert 0 < eg.value.pivot < n and 0 < eo.value.pivot < n


def test_caller_owned_workspace():
    n = 3000
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    theta = (1.0, 0.1, 0.7)
    with ex.Context(device=0) as c:
        ref = c.loglik(x, y, z, theta).loglik
    buf = torch.empty(ex.workspace_bytes(n) // 8 + 1, dtype=torch.float64, device="cuda")
    with ex.Context(device=0) as c:
        c.set_workspace(buf)
        assert c.loglik(x, y, z, theta).loglik == ref
        small = torch.empty(1000, dtype=torch.float64, device="cuda")
        c.set_workspace(small)
        with pytest.raises(ex.ExageoError) as ei:
            c.loglik(x, y, z, theta)
        assert ei.value.status == ex.ENOMEM
        c.set_workspace(None)
        assert c.loglik(x, y, z, theta).loglik == ref


def test_argument_validation():
    with ex.Context(device=0) as c:
        with pytest.raises(ex.ExageoError):
            c.loglik([], [], [], (1.0, 0.1, 0.5))
        c.stage_generate_dev(torch.zeros(10, dtype=torch.float64, device="cuda") + torch.arange(10, device="cuda"),
                             torch.zeros(10, dtype=torch.float64, device="cuda"), None, (1.0, 0.1, 0.5))
        with pytest.raises(ex.ExageoError) as ei:
            c.read_entries([1], [2])  # upper triangle
        assert ei.value.status == ex.EINVAL
    with pytest.raises(ex.ExageoError):
        ex.Context(device=0, nb=100)
    with pytest.raises(ex.ExageoError):
        ex.Context(device=0, world=2, rank=0)  # no NCCL id
