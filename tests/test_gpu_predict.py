"""GPU exageo_predict (NEXT-2; Eq. (5), Alg. 3): kriging through the factor, against the
oracle's Alg. 3 (explicit dposv by substitution + dense Sigma12 product), plus the
properties Eq. (5) fixes: interpolation at observed sites, zero prior mean far away,
linearity in Z2; distributed schedule (virtual ranks) equal to the single GPU; a small
BASELINE configs[4] analogue (10% hold-out, MLE on the rest, MSE vs truth)."""
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


@pytest.fixture(scope="module")
def ctx():
    c = ex.Context(device=0)
    yield c
    c.close()


@pytest.mark.parametrize("n,m,theta", [(400, 38, (1.0, 0.1, 0.5)), (1000, 200, (1.0, 0.1, 1.0)),
                                       (1600, 1, (1.5, 0.05, 1.5)), (2100, 64, (0.8, 0.2, 0.7))])
def test_predict_matches_oracle(ctx, n, m, theta):
    x, y = ex.gen_locations(n, 5)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 6))
    rng = np.random.default_rng(n)
    xn, yn = rng.random(m), rng.random(m)
    got = ctx.predict(x, y, z, xn, yn, theta)
    ref = oracle.predict(x, y, z, xn, yn, theta)
    assert np.abs(got - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


def test_predict_properties(ctx):
    n = 900
    theta = (1.0, 0.1, 1.0)
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    idx = np.array([0, 17, 450, 899])
    got = ctx.predict(x, y, z, x[idx], y[idx], theta)
    np.testing.assert_allclose(got, z[idx], rtol=1e-8, atol=1e-8)  # interpolation
    far = ctx.predict(x, y, z, [1e4, -1e4], [1e4, 3.0], theta)
    assert np.all(far == 0.0)  # prior mean
    xn, yn = np.array([0.31, 0.77]), np.array([0.52, 0.05])
    a = ctx.predict(x, y, z, xn, yn, theta)
    b = ctx.predict(x, y, 2.5 * z, xn, yn, theta)
    np.testing.assert_allclose(b, 2.5 * a, rtol=1e-12)


@pytest.mark.parametrize("world", [2, 3])
def test_predict_virtual_ranks(ctx, world):
    n, m = 1300, 50
    theta = (1.0, 0.1, 0.8)
    x, y = ex.gen_locations(n, 9)
    z = si.normals(n, 10)
    rng = np.random.default_rng(1)
    xn, yn = rng.random(m), rng.random(m)
    c1 = ex.Context(device=0, nb=128, tile_tasks=-1)  # the distributed schedule's kernels
    a = c1.predict(x, y, z, xn, yn, theta)
    c1.close()
    cv = ex.Context(device=0, nb=128, virtual_ranks=world)
    b = cv.predict(x, y, z, xn, yn, theta)
    cv.close()
    assert np.array_equal(a, b)


def test_holdout_mle_and_kriging(ctx):
    # BASELINE configs[4] analogue at n = 1600: 10% hold-out, MLE on the rest, kriging
    n, theta_true = 1600, (1.0, 0.1, 0.5)
    x, y = ex.gen_locations(n, 11)
    z = ctx.simulate(x, y, si.normals(n, 11), theta_true)
    hold = si.holdout_mask(n, n // 10, 11)
    lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
    start = tuple(math.sqrt(a * b) for a, b in zip(lo, hi))
    th, ll, ne, _ = ctx.mle(x[~hold], y[~hold], z[~hold], lo, hi, start, xtol_rel=1e-7)
    pred = ctx.predict(x[~hold], y[~hold], z[~hold], x[hold], y[hold], th)
    mse = float(np.mean((pred - z[hold]) ** 2))
    ref = oracle.predict(x[~hold], y[~hold], z[~hold], x[hold], y[hold], th)
    assert np.abs(pred - ref).max() <= 1e-9
    assert mse < 0.5 * float(np.var(z))  # kriging beats the prior mean by a wide margin
    # the expected MSE (1/m) tr(Sigma11 - Sigma12 Sigma22^-1 Sigma21) = mean kriging variance
    # agrees with the realised MSE to sampling accuracy (m = 160 correlated sites)
    _, var = ctx.predict_var(x[~hold], y[~hold], z[~hold], x[hold], y[hold], th)
    assert 0.5 < mse / float(np.mean(var)) < 2.0


@pytest.mark.parametrize("n,m,nb,theta", [(800, 100, 128, (1.0, 0.1, 0.5)), (1500, 37, 256, (1.4, 0.07, 1.2)),
                                          (333, 5, 128, (0.8, 0.2, 2.5))])
def test_predict_var_matches_oracle(n, m, nb, theta):
    x, y = ex.gen_locations(n, 21)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 22))
    rng = np.random.default_rng(n)
    xn = np.concatenate([rng.random(m - 2), [x[3], 50.0]])  # includes an observed and a far site
    yn = np.concatenate([rng.random(m - 2), [y[3], 50.0]])
    with ex.Context(device=0, nb=nb) as c:
        mean, var = c.predict_var(x, y, z, xn, yn, theta)
        np.testing.assert_array_equal(mean, c.predict(x, y, z, xn, yn, theta))
    ref = oracle.predict_var(x, y, xn, yn, theta)
    assert np.abs(var - ref).max() <= 1e-9 * theta[0]
    assert abs(var[-2]) <= 1e-9 * theta[0] and var[-1] == theta[0]
    assert np.all(var >= -1e-9) and np.all(var <= theta[0])


@pytest.mark.parametrize("world,P,n,nb", [(2, 1, 1100, 128), (2, 2, 1100, 128), (4, 2, 1500, 128), (3, 1, 900, 256),
                                          (6, 2, 2000, 128), (8, 2, 1700, 128)])
def test_predict_var_distributed_virtual_ranks(world, P, n, nb):
    """The distributed kriging variance (process-row reduce of the partial updates onto the
    diagonal rank, broadcast of V_I down the process column) on virtual ranks of a P x Q grid:
    equal to the single-rank variance to rounding and to the oracle's."""
    m = 45
    x, y = ex.gen_locations(n, 31)
    z = si.normals(n, 32)
    theta = (1.2, 0.08, 0.9)
    rng = np.random.default_rng(world)
    xn = np.concatenate([rng.random(m - 2), [x[7], 40.0]])
    yn = np.concatenate([rng.random(m - 2), [y[7], 40.0]])
    with ex.Context(device=0, nb=nb, virtual_ranks=world, grid_rows=P) as c:
        mean, var = c.predict_var(x, y, z, xn, yn, theta)
    with ex.Context(device=0, nb=nb) as c1:
        mean1, var1 = c1.predict_var(x, y, z, xn, yn, theta)
    np.testing.assert_allclose(mean, mean1, rtol=1e-10, atol=1e-11)
    assert np.abs(var - var1).max() <= 1e-11 * theta[0]
    ref = oracle.predict_var(x, y, xn, yn, theta)
    assert np.abs(var - ref).max() <= 1e-9 * theta[0]
    assert abs(var[-2]) <= 1e-9 * theta[0] and var[-1] == theta[0]


@pytest.mark.parametrize("nb", [1024, 2048])
def test_predict_wide_tiles(nb):
    """The automatic tile size of large single-GPU problems (nb = 2048 from n = 56k): the backward
    solve's diagonal-tile kernel needs more than 48 KB of shared memory there (regression: an
    n = 144k predict failed with 'invalid argument' before the opt-in)."""
    n, m = 2500, 20
    x, y = ex.gen_locations(n, 41)
    z = si.normals(n, 42)
    theta = (1.0, 0.1, 0.5)
    rng = np.random.default_rng(nb)
    xn, yn = rng.random(m), rng.random(m)
    with ex.Context(device=0, nb=nb) as c:
        got = c.predict(x, y, z, xn, yn, theta)
    ref = oracle.predict(x, y, z, xn, yn, theta)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-10)
