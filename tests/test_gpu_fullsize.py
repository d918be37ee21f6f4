"""Full-size GPU parity at BASELINE's headline size (n = 100k, nb = 2048, the launch
configuration bench.py times: stream schedule, then the tile-task executor for the last
panel -- the tail hand-off), where the O(n^3) oracle cannot run:

  * AR(1) / Kac-Murdock-Szego closed form of l (exact in O(n), nu = 1/2, collinear sites);
  * sampled generated entries vs the oracle's Matern function;
  * L L^T vs the oracle's Sigma_rc on >= 200 pairs of sampled rows covering every panel-edge
    class and the ragged last panel (O(n) per pair, from read-back rows of L);
  * Alg. 1 -> Alg. 2 round trip at theta_true: y = L^{-1} (L e) = e, so quad = e^T e.
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

N = 100_000
THETA = (1.0, 0.1, 0.5)


@pytest.fixture(scope="module")
def ctx():
    c = ex.Context(device=0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def test_ar1_closed_form_full_size(ctx):
    h, t1, t2 = 2.0**-12, 1.0, 0.05
    x, y = si.collinear_sites(N, h)
    z = si.normals(N, 5)
    r = ctx.loglik(x, y, z, (t1, t2, 0.5))
    assert r.info["nb"] == 2048 and r.info["ntiles"] == 49  # the bench's launch configuration
    rho = math.exp(-h / t2)
    logdet = N * math.log(t1) + (N - 1) * math.log1p(-rho * rho)
    w = np.empty(N)
    w[0] = z[0] / math.sqrt(t1)
    w[1:] = (z[1:] - rho * z[:-1]) / math.sqrt(t1 * (1 - rho * rho))
    quad = float(w @ w)
    ll = -0.5 * quad - 0.5 * logdet - 0.5 * N * LOG2PI
    assert_ll(r.loglik, (ll, logdet, quad), N, what="AR(1) 100k")
    assert r.logdet == pytest.approx(logdet, rel=1e-11)
    assert r.quad == pytest.approx(quad, rel=1e-10)


def test_sampled_entries_and_factor_residual_full_size(ctx):
    x, y = ex.gen_locations(N, 1)
    z = si.normals(N, 1)
    ctx.stage_generate_dev(dev(x), dev(y), dev(z), THETA)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, N, 3000)
    cols = (rng.random(3000) * (rows + 1)).astype(np.int64)
    got = ctx.read_entries(rows, cols)
    ref = np.array([oracle.matern(math.hypot(x[r] - x[c], y[r] - y[c]) if r != c else 0.0, THETA)
                    for r, c in zip(rows, cols)])
    mask = ref > 1e-290
    assert np.all(np.abs(got[mask] - ref[mask]) <= 5e-14 * ref[mask] + 1e-300)
    ctx.stage_factor()
    check_llt_sample(ctx, x, y)
    ll, logdet, quad = ctx.stage_finish()
    assert np.isfinite(ll)


# rows of L read back for the L L^T check: every panel-edge class of the bench layout
# (nb = 2048, 64-column POTRF blocks, T = 49, N = 100352): first/last row of a panel and of a
# 64-block, the rows either side of them, and the ragged last panel (panel 48 starts at 98304;
# rows 98304..99999 are real, 100000..100351 identity padding; it is factored by the tile-task
# executor after the stream schedule's hand-off), plus random rows
EDGE_ROWS = [0, 1, 63, 64, 127, 128, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 49151, 49152, 49215,
             49216, 98303, 98304, 98305, 98367, 98368, 99327, 99328, 99967, 99968, 99998, 99999]


def check_llt_sample(ctx, x, y, theta=THETA, extra=15):
    """(L L^T)_rc = sum_{t <= c} L_rt L_ct must reproduce Sigma_rc = C(||s_r - s_c||; theta), the
    oracle's Matern value, for every pair c <= r of the sampled rows (>= 200 pairs)."""
    rng = np.random.default_rng(3)
    rows = sorted(set(EDGE_ROWS) | set(int(v) for v in rng.integers(0, N, extra)))
    Lrow = {}
    for r in rows:
        t = np.arange(r + 1, dtype=np.int64)
        Lrow[r] = ctx.read_entries(np.full(r + 1, r, np.int64), t)
    pairs = [(r, c) for i, r in enumerate(rows) for c in rows[: i + 1]]
    assert len(pairs) >= 200
    worst = 0.0
    for r, c in pairs:
        s = math.fsum(Lrow[r][: c + 1] * Lrow[c])
        d = math.hypot(x[r] - x[c], y[r] - y[c]) if r != c else 0.0
        sig = oracle.matern(d, theta)
        worst = max(worst, abs(s - sig))
        assert abs(s - sig) <= 1e-12 * theta[0], (r, c, s, sig)
    print(f"L L^T sample: {len(pairs)} pairs over {len(rows)} rows, max |(LL^T - Sigma)_rc| = {worst:.2e}")


def test_simulate_roundtrip_full_size(ctx):
    x, y = ex.gen_locations(N, 1)
    e = si.normals(N, 3)
    z = ctx.simulate(x, y, e, THETA)
    r = ctx.loglik(x, y, z, THETA)
    assert r.quad == pytest.approx(float(e @ e), rel=1e-9)


@pytest.mark.parametrize("theta", [(1.3, 0.1, 1.27), (0.8, 0.03, 0.61)])
def test_sampled_entries_general_nu_full_size(ctx, theta):
    # general nu at full size: the generator reads the per-theta Chebyshev table (K1T)
    x, y = ex.gen_locations(N, 2)
    z = si.normals(N, 2)
    ctx.stage_generate_dev(dev(x), dev(y), dev(z), theta)
    rng = np.random.default_rng(1)
    rows = rng.integers(0, N, 2000)
    cols = (rng.random(2000) * (rows + 1)).astype(np.int64)
    got = ctx.read_entries(rows, cols)
    d = np.array([math.hypot(x[r] - x[c], y[r] - y[c]) if r != c else 0.0 for r, c in zip(rows, cols)])
    ref = np.array([oracle.matern(v, theta) for v in d])
    mask = ref > 1e-290
    bound = 5e-14 * ref[mask] + 4e-16 * (d[mask] / theta[1]) * ref[mask]
    assert np.all(np.abs(got[mask] - ref[mask]) <= bound)
