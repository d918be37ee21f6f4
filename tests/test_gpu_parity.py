"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances:
  * covariance entries: max relative error <= 5e-14 (K_nu evaluator vs the
    oracle's quadrature; R-budget in DESIGN.md);
  * factor: ||L_gpu - L_oracle||_max / ||L||_max <= 1e-12;
  * l(theta): |dl| <= 1e-10 * max(|l|, |logdet|/2, quad/2, (n/2) log 2 pi)
    (BASELINE.json north_star 1e-10 relative, guarded against cancellation, R13).
"""
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

from tests._tol import LOG2PI, assert_ll  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = ex.Context(device=0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx128():
    c = ex.Context(device=0, nb=128)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


THETAS = [(1.0, 0.1, 0.5), (1.0, 0.1, 1.0), (2.0, 0.05, 1.5), (0.7, 0.2, 2.5), (1.3, 0.08, 0.3),
          (1.0, 0.1, 0.77), (0.9, 0.03, 1.7), (1.0, 0.1, 2.2), (1.0, 0.3, 3.6)]


@pytest.mark.parametrize("theta", THETAS)
def test_matern_cov_entrywise(ctx, theta):
    x, y = oracle.gen_locations(300, 2)
    xn, yn = oracle.gen_locations(90, 5)
    got = ctx.matern_cov(xn, yn, x, y, theta)
    ref = oracle.cov(xn, yn, x, y, theta)
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    mask = np.abs(ref) > 1e-290
    assert rel[mask].max() <= 5e-14, (theta, rel[mask].max())


def test_matern_cov_distance_sweep(ctx):
    # distances r/theta2 from 1e-4 to 700 across the Temme / CF2 switch (x = 2)
    r = np.concatenate([np.geomspace(1e-5, 70.0, 400), [0.2 - 1e-12, 0.2, 0.2 + 1e-12]])
    x2, y2 = np.zeros(1), np.zeros(1)
    for nu in [0.1, 0.35, 0.5, 0.99, 1.0, 1.01, 1.5, 1.49999, 2.0, 2.5, 3.3, 4.9]:
        theta = (1.0, 0.1, nu)
        got = ctx.matern_cov(r, np.zeros_like(r), x2, y2, theta)[:, 0]
        ref = np.array([oracle.matern(v, theta) for v in r])
        mask = ref > 1e-290
        rel = np.abs(got[mask] - ref[mask]) / ref[mask]
        # exp(nu ln x - x) has relative condition number ~x: allow 4e-16 x on top
        bound = 5e-14 + 4e-16 * r[mask] / 0.1
        assert np.all(rel <= bound), (nu, rel.max(), r[mask][(rel / bound).argmax()])


# general nu runs through the per-theta Chebyshev table (K1T): theta2 = 0.01 puts most
# x = r/theta2 beyond the table (direct continued fraction), theta2 = 2 most below 2^-6 +
# the quarter-octave intervals, 0.1 the linear intervals
@pytest.mark.parametrize("n,nb,nu,beta", [(700, 128, 0.5, 0.1), (1000, 256, 1.3, 0.1), (131, 128, 2.5, 0.1),
                                          (900, 128, 0.37, 0.01), (600, 128, 1.73, 2.0), (800, 256, 1.0, 0.1),
                                          (500, 128, 0.83, 0.5), (400, 128, 0.1, 0.3), (400, 128, 4.9, 0.05)])
def test_generated_panels_match_oracle(n, nb, nu, beta):
    c = ex.Context(device=0, nb=nb)
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    theta = (1.2, beta, nu)
    c.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    S = c.read_lower(n)
    ref = np.tril(oracle.cov(x, y, x, y, theta))
    rel = np.abs(S - ref) / np.maximum(np.abs(ref), 1e-300)
    xr = np.hypot(x[:, None] - x[None, :], y[:, None] - y[None, :]) / beta
    mask = np.tril(np.abs(ref) > 1e-290)
    assert np.all(rel[mask] <= 5e-14 + 4e-16 * xr[mask]), rel[mask].max()
    np.testing.assert_array_equal(c.read_zrow(n), z)
    c.close()


@pytest.mark.parametrize("n,nb,theta", [(700, 128, (1.0, 0.1, 0.5)), (1000, 256, (1.0, 0.1, 1.0)),
                                        (1100, 128, (1.5, 0.05, 1.5)), (257, 128, (1.0, 0.2, 0.9)),
                                        (1300, 384, (1.0, 0.1, 0.7)), (2000, 384, (1.2, 0.08, 0.5)),
                                        (2500, 1024, (1.0, 0.1, 0.5)), (4500, 2048, (1.0, 0.1, 0.6))])
def test_factor_and_solve_match_oracle(n, nb, theta):
    c = ex.Context(device=0, nb=nb)
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    c.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    c.stage_factor()
    L = c.read_lower(n)
    yv = c.read_zrow(n)
    Lo = oracle.cholesky(oracle.cov(x, y, x, y, theta))
    err = np.abs(L - Lo).max() / np.abs(Lo).max()
    assert err <= 1e-12, err
    yo = oracle.forward(Lo, z)
    assert np.abs(yv - yo).max() / np.abs(yo).max() <= 1e-10
    ll, logdet, quad = c.stage_finish()
    llo, ldo, qo = oracle.loglik(x, y, z, theta)
    assert_ll(ll, (llo, ldo, qo), n, what=(n, nb, theta))
    c.close()


@pytest.mark.parametrize("n", [1, 2, 3, 17, 128, 129, 400, 1000, 1600])
@pytest.mark.parametrize("theta", [(1.0, 0.1, 0.5), (1.0, 0.1, 1.0), (2.0, 0.07, 0.6)])
def test_loglik_matches_oracle(ctx, n, theta):
    x, y = ex.gen_locations(n, 1)
    e = si.normals(n, 2)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), e)
    r = ctx.loglik(x, y, z, theta)
    llo, ldo, qo = oracle.loglik(x, y, z, theta)
    assert_ll(r.loglik, (llo, ldo, qo), n, what=(n, theta))
    assert r.logdet == pytest.approx(ldo, rel=1e-10, abs=1e-10)
    assert r.quad == pytest.approx(qo, rel=1e-10)


def test_loglik_config1_n400(ctx):
    # BASELINE.json configs[0]: n = 400 (20 x 20 grid), theta = (1, 0.1, 0.5), z from a fixed seed
    n, theta = 400, (1.0, 0.1, 0.5)
    x, y = ex.gen_locations(n, 1)
    z = oracle.simulate(x, y, theta, si.normals(n, 1))
    for nb in (128, 256, 512):
        c = ex.Context(device=0, nb=nb)
        r = c.loglik(x, y, z, theta)
        llo, ldo, qo = oracle.loglik(x, y, z, theta)
        assert_ll(r.loglik, (llo, ldo, qo), n, what=nb)
        c.close()


def test_loglik_closed_forms(ctx):
    # n = 1 and n = 2
    r = ctx.loglik([0.3], [0.4], [0.0], (1.0, 0.1, 0.5))
    assert r.loglik == pytest.approx(-0.5 * LOG2PI, rel=1e-15)
    t1, t2, nu = 1.7, 0.1, 0.5
    rho = math.exp(-1.0)
    z1, z2 = 1.0, -0.5
    logdet = 2 * math.log(t1) + math.log(1 - rho * rho)
    quad = (z1 * z1 - 2 * rho * z1 * z2 + z2 * z2) / (t1 * (1 - rho * rho))
    r = ctx.loglik([0.1, 0.16], [0.2, 0.28], [z1, z2], (t1, t2, nu))
    assert r.loglik == pytest.approx(-LOG2PI - 0.5 * logdet - 0.5 * quad, rel=1e-14)


def kms(z, t1, rho):
    n = z.size
    logdet = n * math.log(t1) + (n - 1) * math.log1p(-rho * rho)
    w = np.empty(n)
    w[0] = z[0] / math.sqrt(t1)
    w[1:] = (z[1:] - rho * z[:-1]) / math.sqrt(t1 * (1 - rho * rho))
    quad = float(np.dot(w, w))
    return -0.5 * quad - 0.5 * logdet - 0.5 * n * LOG2PI, logdet, quad


@pytest.mark.parametrize("n", [5000, 23456])
def test_loglik_ar1_closed_form(ctx, n):
    h, t1, t2 = 2.0**-12, 1.3, 0.05
    x, y = si.collinear_sites(n, h)
    z = si.normals(n, 31)
    r = ctx.loglik(x, y, z, (t1, t2, 0.5))
    ll, ld, qd = kms(z, t1, math.exp(-h / t2))
    assert_ll(r.loglik, (ll, ld, qd), n, what=n)
    assert r.logdet == pytest.approx(ld, rel=1e-11)


def test_loglik_identity_covariance(ctx):
    n, t1 = 3000, 2.3
    x, y = si.spread_sites(n, 100.0)
    z = si.normals(n, 4)
    r = ctx.loglik(x, y, z, (t1, 0.1, 1.5))
    assert r.logdet == pytest.approx(n * math.log(t1), rel=1e-13)
    assert r.quad == pytest.approx(float(z @ z) / t1, rel=1e-13)


def test_not_positive_definite_pivot(ctx):
    x = np.array([0.1, 0.5, 0.5, 0.9])
    y = np.array([0.1, 0.5, 0.5, 0.2])
    with pytest.raises(ex.NotPositiveDefinite) as ei:
        ctx.loglik(x, y, [1.0, 2.0, 3.0, 4.0], (1.0, 0.1, 0.5))
    assert ei.value.pivot == 2
    # the context stays usable afterwards
    r = ctx.loglik([0.3], [0.4], [0.0], (1.0, 0.1, 0.5))
    assert r.loglik == pytest.approx(-0.5 * LOG2PI, rel=1e-15)


def test_invalid_theta(ctx):
    for bad in [(0.0, 0.1, 0.5), (1.0, -0.1, 0.5), (1.0, 0.1, float("nan"))]:
        with pytest.raises(ex.ExageoError) as ei:
            ctx.loglik([0.1], [0.2], [0.3], bad)
        assert ei.value.status == ex.EINVAL


def test_deterministic(ctx):
    n = 3000
    x, y = ex.gen_locations(n, 1)
    z = si.normals(n, 2)
    a = ctx.loglik(x, y, z, (1.0, 0.1, 0.8))
    b = ctx.loglik(x, y, z, (1.0, 0.1, 0.8))
    assert a.loglik == b.loglik and a.logdet == b.logdet and a.quad == b.quad


def test_loglik_dev_matches_host(ctx):
    n = 2000
    x, y = ex.gen_locations(n, 4)
    z = si.normals(n, 5)
    a = ctx.loglik(x, y, z, (1.0, 0.1, 0.5))
    b = ctx.loglik_dev(dev(x), dev(y), dev(z), (1.0, 0.1, 0.5))
    assert a.loglik == b.loglik


def test_nb_independence():
    n = 2100
    x, y = ex.gen_locations(n, 6)
    z = si.normals(n, 7)
    vals = []
    for nb in (128, 256, 384, 512):
        c = ex.Context(device=0, nb=nb)
        vals.append(c.loglik(x, y, z, (1.0, 0.1, 1.0)).loglik)
        c.close()
    assert max(vals) - min(vals) <= 1e-12 * abs(vals[0])


def test_simulate_matches_oracle_and_roundtrip(ctx):
    n = 900
    theta = (1.0, 0.1, 1.0)
    x, y = ex.gen_locations(n, 9)
    e = si.normals(n, 10)
    z = ctx.simulate(x, y, e, theta)
    zo = oracle.simulate(x, y, theta, e)
    assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()
    # Alg. 1 then Alg. 2 at the same theta: y = L^{-1} z = e, so quad = e^T e
    r = ctx.loglik(x, y, z, theta)
    assert r.quad == pytest.approx(float(e @ e), rel=1e-10)


# ---- distributed schedule on one GPU (virtual ranks) ----------------
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("n,nb", [(1000, 128), (2600, 256), (700, 128)])
def test_virtual_ranks_match_single_and_oracle(world, n, nb):
    x, y = ex.gen_locations(n, 21)
    theta = (1.0, 0.1, 0.8)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 22))
    single = ex.Context(device=0, nb=nb, tile_tasks=-1)  # the distributed schedule's kernels
    r1 = single.loglik(x, y, z, theta)
    single.close()
    c = ex.Context(device=0, nb=nb, virtual_ranks=world)
    r = c.loglik(x, y, z, theta)
    llo, ldo, qo = oracle.loglik(x, y, z, theta)
    assert_ll(r.loglik, (llo, ldo, qo), n, what=(world, n, nb))
    # same kernels and order per panel; only the final partial sums are grouped by rank
    assert r.loglik == pytest.approx(r1.loglik, rel=1e-13)
    # factor read back from the distributed panels equals the single-GPU factor bitwise
    c.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    c.stage_factor()
    Lv = c.read_lower(n)
    s2 = ex.Context(device=0, nb=nb, tile_tasks=-1)
    s2.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    s2.stage_factor()
    assert np.array_equal(Lv, s2.read_lower(n))
    assert np.array_equal(c.read_zrow(n), s2.read_zrow(n))
    s2.close()
    c.close()


def test_virtual_ranks_not_pd_and_simulate():
    c = ex.Context(device=0, nb=128, virtual_ranks=3)
    x = np.concatenate([ex.gen_locations(300, 1)[0], [0.5, 0.5]])
    y = np.concatenate([ex.gen_locations(300, 1)[1], [0.5, 0.5]])
    with pytest.raises(ex.NotPositiveDefinite) as ei:
        c.loglik(x, y, np.ones(302), (1.0, 0.1, 0.5))
    assert ei.value.pivot == 301
    n = 800
    x, y = ex.gen_locations(n, 2)
    e = si.normals(n, 3)
    z = c.simulate(x, y, e, (1.0, 0.1, 1.0))
    zo = oracle.simulate(x, y, (1.0, 0.1, 1.0), e)
    assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()
    c.close()


# ---- 2-D block-cyclic P x Q process grids on one GPU (virtual ranks) --------
GRIDS = [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (3, 2)]  # (P, Q)


@pytest.mark.parametrize("P,Q", GRIDS, ids=[f"{p}x{q}" for p, q in GRIDS])
@pytest.mark.parametrize("n,nb", [(1000, 128), (2600, 256), (700, 128)])
def test_grid_virtual_ranks_match_single_and_oracle(P, Q, n, nb):
    x, y = ex.gen_locations(n, 21)
    theta = (1.0, 0.1, 0.8)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 22))
    single = ex.Context(device=0, nb=nb, tile_tasks=-1)  # the distributed schedule's kernels
    r1 = single.loglik(x, y, z, theta)
    single.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    single.stage_factor()
    L1, y1 = single.read_lower(n), single.read_zrow(n)
    single.close()
    c = ex.Context(device=0, nb=nb, virtual_ranks=P * Q, grid_rows=P)
    r = c.loglik(x, y, z, theta)
    assert_ll(r.loglik, oracle.loglik(x, y, z, theta), n, what=(P, Q, n, nb))
    # same tile kernels in the same order per tile: only the final partial sums are grouped
    # by rank
    assert r.loglik == pytest.approx(r1.loglik, rel=1e-13)
    assert r.logdet == pytest.approx(r1.logdet, rel=1e-13) and r.quad == pytest.approx(r1.quad, rel=1e-13)
    # the factor and y read back from the block-cyclic tiles equal the single-GPU ones bitwise
    c.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    c.stage_factor()
    assert np.array_equal(c.read_lower(n), L1)
    assert np.array_equal(c.read_zrow(n), y1)
    c.close()


@pytest.mark.parametrize("P,Q", [(2, 2), (2, 1), (4, 2)], ids=["2x2", "2x1", "4x2"])
def test_grid_simulate_predict_not_pd(P, Q):
    n, nb, theta = 900, 128, (1.0, 0.1, 1.0)
    x, y = ex.gen_locations(n, 9)
    e = si.normals(n, 10)
    c = ex.Context(device=0, nb=nb, virtual_ranks=P * Q, grid_rows=P)
    z = c.simulate(x, y, e, theta)
    zo = oracle.simulate(x, y, theta, e)
    assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()
    xn, yn = ex.gen_locations(37, 11)
    xn, yn = xn * 0.97 + 0.011, yn * 0.97 + 0.013
    got = c.predict(x, y, z, xn, yn, theta)
    ref = oracle.predict(x, y, z, xn, yn, theta)
    assert np.abs(got - ref).max() <= 1e-9 * np.abs(ref).max()
    xd = np.concatenate([x[:300], x[:1]])
    yd = np.concatenate([y[:300], y[:1]])
    with pytest.raises(ex.NotPositiveDefinite) as ei:
        c.loglik(xd, yd, np.ones(301), theta)
    assert ei.value.pivot == 300
    c.close()


def test_grid_ind_matches_single():
    n, nb = 1500, 128
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    a = ex.Context(device=0, nb=nb, ind_tiles=3).loglik(x, y, z, (1.0, 0.1, 1.0))
    b = ex.Context(device=0, nb=nb, ind_tiles=3, virtual_ranks=4, grid_rows=2).loglik(x, y, z, (1.0, 0.1, 1.0))
    assert b.loglik == pytest.approx(a.loglik, rel=1e-13)


def test_grid_rows_validation():
    with pytest.raises(ex.ExageoError) as ei:
        ex.Context(device=0, virtual_ranks=6, grid_rows=4)
    assert ei.value.status == ex.EINVAL
