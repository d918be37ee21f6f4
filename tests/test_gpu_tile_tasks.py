"""The tile-task executor (dag.cu): the whole factorization as one persistent kernel running
the 64 x 64 tile DAG of Fig. 2 on the device, with the z row (Alg. 2 l.4) fused.

Checked against the oracle (Alg. 2) on the paper's jittered grid at
sizes spanning one tile, several tiles and a ragged last tile, against the stream-launched
schedule on the same inputs (the same operations in another order: agreement to rounding),
and on the degenerate cases: n = 1, a non-PD covariance (ENOTPD with the oracle's pivot),
predict / simulate through the executor's factor, CUDA-graph replay."""
import numpy as np
import pytest

import oracle
import synth_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402
from tests._tol import assert_ll  # noqa: E402


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 127, 128, 200, 400, 777, 1600])
@pytest.mark.parametrize("theta", [(1.0, 0.1, 0.5), (1.3, 0.07, 1.2)])
def test_tile_tasks_match_oracle(n, theta):
    x, y = ex.gen_locations(n, 11)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 12))
    with ex.Context(device=0, tile_tasks=1, graphs=-1) as c:
        r = c.loglik(x, y, z, theta)
    ref = oracle.loglik(x, y, z, theta)
    assert_ll(r.loglik, ref, n, what=(n, theta))
    assert r.logdet == pytest.approx(ref[1], rel=1e-10, abs=1e-12)
    assert r.quad == pytest.approx(ref[2], rel=1e-10)
    assert r.info["kernels"] <= 8, r.info["kernels"]  # one factorization kernel, not ~4 per 64 columns


@pytest.mark.parametrize("n,nb", [(3000, 128), (5000, 256), (6500, 128), (9000, 384)])
def test_tile_tasks_match_stream_schedule(n, nb):
    """Larger n (many CTAs racing on the ticket and the version counters): the executor and
    the stream schedule agree to rounding, and the factor itself agrees entry by entry."""
    x, y = ex.gen_locations(n, 5)
    z = si.normals(n, 6)
    theta = (1.0, 0.1, 0.5)
    out = {}
    for tt in (1, -1):
        with ex.Context(device=0, nb=nb, tile_tasks=tt, graphs=-1) as c:
            r = c.loglik(x, y, z, theta)
            rows = np.random.default_rng(n).integers(0, n, 400)
            cols = np.minimum(rows, np.random.default_rng(n + 1).integers(0, n, 400))
            out[tt] = (r, c.read_entries(rows, cols), c.read_zrow(n))
    (a, la, ya), (b, lb, yb) = out[1], out[-1]
    assert abs(a.loglik - b.loglik) <= 1e-11 * abs(b.loglik)
    np.testing.assert_allclose(la, lb, rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(ya, yb, rtol=1e-9, atol=1e-11)


def test_tile_tasks_deterministic():
    n = 2500
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    with ex.Context(device=0, tile_tasks=1) as c:
        vals = [c.loglik(x, y, z, (1.0, 0.1, 0.5)).loglik for _ in range(5)]
    assert len(set(vals)) == 1, vals


def test_tile_tasks_not_pd_exact_pivot():
    """A duplicated site makes pivot 2 exactly zero (identical rows): ENOTPD at pivot 2."""
    x = np.array([0.1, 0.5, 0.5, 0.9])
    y = np.array([0.1, 0.5, 0.5, 0.2])
    with ex.Context(device=0, tile_tasks=1) as c:
        with pytest.raises(ex.NotPositiveDefinite) as e:
            c.loglik(x, y, [1.0, 2.0, 3.0, 4.0], (1.0, 0.1, 0.5))
        assert e.value.pivot == 2
        r = c.loglik([0.3], [0.4], [0.0], (1.0, 0.1, 0.5))  # the context stays usable
        assert np.isfinite(r.loglik)


@pytest.mark.parametrize("n,theta", [(400, (1.0, 3.0, 3.5)), (1600, (1.0, 2.0, 4.0))])
def test_tile_tasks_numerically_singular(n, theta):
    """cond(Sigma) far beyond 1/u: both the oracle and the executor report ENOTPD with a pivot
    inside (0, n) (where exactly is decided by rounding), and every CTA leaves the kernel."""
    x, y = ex.gen_locations(n, 5)
    z = si.normals(n, 6)
    with pytest.raises(oracle.NotPositiveDefinite) as eo:
        oracle.loglik(x, y, z, theta)
    with ex.Context(device=0, tile_tasks=1) as c:
        with pytest.raises(ex.NotPositiveDefinite) as eg:
            c.loglik(x, y, z, theta)
        r = c.loglik(x, y, z, (1.0, 0.1, 0.5))
    assert 0 < eg.value.pivot < n and 0 < eo.value.pivot < n
    assert_ll(r.loglik, oracle.loglik(x, y, z, (1.0, 0.1, 0.5)), n)


def test_tile_tasks_graph_replay_matches_launch():
    n = 1600
    x, y = ex.gen_locations(n, 9)
    z = si.normals(n, 10)
    thetas = [(1.0, 0.1, 0.5), (0.8, 0.2, 0.9), (1.2, 0.05, 1.5)]
    with ex.Context(device=0, tile_tasks=1, graphs=1) as cg, ex.Context(device=0, tile_tasks=1, graphs=-1) as cl:
        for th in thetas:
            assert cg.loglik(x, y, z, th).loglik == cl.loglik(x, y, z, th).loglik


def test_tile_tasks_predict_and_simulate():
    n, m = 900, 50
    x, y = ex.gen_locations(n + m, 13)
    theta = (1.0, 0.1, 0.5)
    e = si.normals(n, 14)
    with ex.Context(device=0, tile_tasks=1) as c:
        z = c.simulate(x[:n], y[:n], e, theta)
        zp = c.predict(x[:n], y[:n], z, x[n:], y[n:], theta)
    z_ref = oracle.simulate(x[:n], y[:n], theta, e)
    np.testing.assert_allclose(z, z_ref, rtol=1e-10, atol=1e-11)
    zp_ref = oracle.predict(x[:n], y[:n], z, x[n:], y[n:], theta)
    np.testing.assert_allclose(zp, zp_ref, rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("n,nb", [(3300, 128), (4100, 256), (7000, 256), (12500, 384)])
def test_tail_handoff_matches_stream_schedule(n, nb):
    """Above the executor's own range the stream schedule hands the last panels (trailing size
    <= 2560) to the executor (t0 > 0, no generation): same l, factor and y as the pure stream
    schedule (tile_tasks=-1) to rounding."""
    x, y = ex.gen_locations(n, 15)
    z = si.normals(n, 16)
    theta = (1.0, 0.1, 0.5)
    rows = np.random.default_rng(n).integers(0, n, 500)
    rows[:100] = n - 1 - np.arange(100)  # the handed-over trailing corner
    cols = np.minimum(rows, np.random.default_rng(n + 1).integers(0, n, 500))
    out = {}
    for tt in (0, -1):
        with ex.Context(device=0, nb=nb, tile_tasks=tt, graphs=-1) as c:
            r = c.loglik(x, y, z, theta)
            out[tt] = (r, c.read_entries(rows, cols), c.read_zrow(n))
    (a, la, ya), (b, lb, yb) = out[0], out[-1]
    assert a.info["kernels"] < b.info["kernels"]  # the tail ran as one launch
    assert abs(a.loglik - b.loglik) <= 1e-11 * abs(b.loglik)
    assert a.logdet == pytest.approx(b.logdet, rel=1e-12) and a.quad == pytest.approx(b.quad, rel=1e-11)
    np.testing.assert_allclose(la, lb, rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(ya, yb, rtol=1e-9, atol=1e-11)


def test_tail_handoff_matches_oracle():
    n = 3600
    x, y = ex.gen_locations(n, 17)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 18))
    theta = (1.0, 0.1, 0.9)
    with ex.Context(device=0, nb=128) as c:  # graphs and the hand-off: the default path at this n
        r = c.loglik(x, y, z, theta)
        r2 = c.loglik(x, y, z, theta)
    assert r.loglik == r2.loglik
    assert_ll(r.loglik, oracle.loglik(x, y, z, theta), n)


def test_tile_tasks_fuzz_against_stream_schedule():
    """Randomised n (1 .. 3200, ragged and tile-aligned) and theta: the
    executor (one persistent kernel, device-side list schedule, per-tile version counters)
    against the stream schedule on the same inputs, and bitwise against itself on a repeat --
    a scheduling race (a task reading a tile before its inputs are final) would show as a
    mismatch in some draw."""
    rng = np.random.default_rng(2024)
    ns = sorted(set([1, 63, 64, 65, 129, 1024, 3200] + [int(v) for v in rng.integers(2, 3201, 14)]))
    with ex.Context(device=0, tile_tasks=1) as ce, ex.Context(device=0, tile_tasks=-1) as cs:
        for n in ns:
            x, y = ex.gen_locations(n, n + 7)
            z = si.normals(n, n + 8)
            # well conditioned part of the MLE box (the ill-conditioned part: test_gpu_edge.py)
            theta = (float(rng.uniform(0.3, 3.0)), float(rng.uniform(0.02, 0.15)), float(rng.uniform(0.3, 1.0)))
            try:
                a = ce.loglik(x, y, z, theta)
            except ex.NotPositiveDefinite:
                with pytest.raises(ex.NotPositiveDefinite):
                    cs.loglik(x, y, z, theta)
                continue
            b = cs.loglik(x, y, z, theta)
            again = ce.loglik(x, y, z, theta)
            assert again.loglik == a.loglik, (n, theta)
            scale = max(abs(b.loglik), 0.5 * abs(b.logdet), 0.5 * b.quad, 0.5 * n * 1.8378770664093453)
            assert abs(a.loglik - b.loglik) <= 1e-10 * scale, (n, theta, a.loglik, b.loglik)


@pytest.mark.parametrize("n,reps", [(1000, 40), (3200, 12)])
def test_tile_tasks_repeat_bitwise(n, reps):
    """Many executor runs with two alternating theta (racing CTAs; tiles published by a barrier
    plus st.release and acquired by relaxed polls plus fence.acq_rel; the pool's early ticket and
    operand prefetch; the chain's prefetch hook): every run reproduces its theta's first result
    bit for bit -- l, logdet, quad and a sample of factor entries -- so no task ever read a tile
    before its producer published it, nor a stale version from the other theta's run."""
    x, y = ex.gen_locations(n, 21)
    z = si.normals(n, 22)
    thetas = [(1.0, 0.1, 0.5), (1.4, 0.05, 1.1)]
    rows = np.random.default_rng(n).integers(0, n, 300)
    cols = np.minimum(rows, np.random.default_rng(n + 7).integers(0, n, 300))
    with ex.Context(device=0, tile_tasks=1, graphs=-1) as c:
        ref = {}
        for th in thetas:
            r = c.loglik(x, y, z, th)
            ref[th] = ((r.loglik, r.logdet, r.quad), c.read_entries(rows, cols))
        for it in range(reps):
            th = thetas[it % 2]
            r = c.loglik(x, y, z, th)
            assert (r.loglik, r.logdet, r.quad) == ref[th][0], (it, th)
            if it % 4 < 2:
                np.testing.assert_array_equal(c.read_entries(rows, cols), ref[th][1])
