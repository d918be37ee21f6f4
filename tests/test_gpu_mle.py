"""GPU exageo_mle (NEXT-1): theta_hat of the product's derivative-free search
against the ORACLE's estimate (tests/golden/mle_n400.json, written by
tools/make_golden_mle.py from oracle.mle) within 1e-4 relative (BASELINE north_star), and
the stationarity pins evaluated with the oracle: profile identity in theta1 and
coordinate-wise local maximum; BASELINE configs[1] (n = 1600, nu in {0.5, 1.0})."""
import ctypes
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mle_n400.json")
LO, HI = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)


@pytest.fixture(scope="module")
def ctx():
    c = ex.Context(device=0)
    yield c
    c.close()


def test_mle_matches_oracle_estimate(ctx):
    g = json.load(open(GOLDEN))
    n = g["n"]
    x, y = ex.gen_locations(n, g["seed"])
    z = oracle.simulate(x, y, tuple(g["theta_true"]), si.normals(n, g["seed"]))
    th, ll, ne, trace = ctx.mle(x, y, z, tuple(g["lo"]), tuple(g["hi"]), tuple(g["start"]), xtol_rel=1e-10,
                                max_evals=3000)
    ref = g["theta_hat"]
    for a, b in zip(th, ref):
        assert a == pytest.approx(b, rel=1e-4), (th, ref)
    assert ll == pytest.approx(g["loglik"], rel=1e-10)
    assert ne == len(trace) and ne <= 3000
    assert np.max(trace[:, 3]) == pytest.approx(ll, rel=1e-15)
    # the oracle agrees that theta_hat is stationary in theta1 (profile identity)
    assert th[0] == pytest.approx(oracle.profile_sigma2(x, y, z, th[1], th[2]), rel=1e-4)


@pytest.mark.parametrize("nu_true", [0.5, 1.0])
def test_mle_config2_n1600(ctx, nu_true):
    n = 1600
    theta_true = (1.0, 0.1, nu_true)
    x, y = ex.gen_locations(n, 2)
    z = ctx.simulate(x, y, si.normals(n, 2), theta_true)
    start = tuple(math.sqrt(a * b) for a, b in zip(LO, HI))
    th, ll, ne, trace = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-9, max_evals=3000)
    assert all(a <= t <= b for a, t, b in zip(LO, th, HI))
    assert ll >= ctx.loglik(x, y, z, theta_true).loglik
    # profile identity with the oracle at the product's (theta2, theta3)
    assert th[0] == pytest.approx(oracle.profile_sigma2(x, y, z, th[1], th[2]), rel=1e-4)
    # coordinate-wise local maximum on the GPU likelihood
    for p in range(3):
        for s in (1 - 1e-3, 1 + 1e-3):
            t = list(th)
            t[p] *= s
            t[p] = min(max(t[p], LO[p]), HI[p])
            assert ctx.loglik(x, y, z, t).loglik <= ll + 1e-9 * abs(ll)
    # estimates near the truth (statistical sanity)
    assert abs(th[2] - nu_true) < 0.25


def test_mle_fixed_parameters(ctx):
    n = 400
    x, y = ex.gen_locations(n, 4)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 4))
    lo, hi = (0.01, 0.1, 0.5), (5.0, 0.1, 0.5)  # only theta1 free
    th, ll, ne, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.1, 0.5), xtol_rel=1e-11)
    assert th[1] == 0.1 and th[2] == 0.5
    # l is flat to ~1e-13 relative within ~5e-7 of the maximiser (curvature ~n/2 in log theta1)
    assert th[0] == pytest.approx(oracle.profile_sigma2(x, y, z, 0.1, 0.5), rel=2e-6)


def test_mle_invalid_bounds(ctx):
    with pytest.raises(ex.ExageoError) as ei:
        ctx.mle([0.1, 0.2], [0.1, 0.3], [1.0, 2.0], (1, 1, 1), (0.5, 2, 2), (1, 1, 1))
    assert ei.value.status == ex.EINVAL
    with pytest.raises(ex.ExageoError) as ei:
        ctx.mle([0.1, 0.2], [0.1, 0.3], [1.0, 2.0], (1, 1, 1), (2, 2, 2), (1, 1, 1), method="trust-region",
                max_evals=0)
    assert ei.value.status == ex.EINVAL
    o = ex.MleOpts(1e-6, 10, 0, 7)  # unknown method
    th, ll, ne = ex.Theta(), ctypes.c_double(), ctypes.c_int()
    lo, hi, st = ex.Theta(1, 1, 1), ex.Theta(2, 2, 2), ex.Theta(1, 1, 1)
    xs = np.array([0.1, 0.2])
    rc = ctx._lib.exageo_mle_ex(ctx._ctx, 2, ex._p(xs), ex._p(xs), ex._p(xs), ctypes.byref(lo), ctypes.byref(hi),
                                ctypes.byref(st), ctypes.byref(o), ctypes.byref(th), ctypes.byref(ll),
                                ctypes.byref(ne), None)
    assert rc == ex.EINVAL


def test_mle_profile_matches_oracle_estimate(ctx):
    # exageo_mle_profile: theta1 in closed form, search over (theta2, theta3); same maximiser
    g = json.load(open(GOLDEN))
    n = g["n"]
    x, y = ex.gen_locations(n, g["seed"])
    z = oracle.simulate(x, y, tuple(g["theta_true"]), si.normals(n, g["seed"]))
    th, ll, ne, trace = ctx.mle(x, y, z, tuple(g["lo"]), tuple(g["hi"]), tuple(g["start"]), xtol_rel=1e-10,
                                max_evals=3000, profile=True)
    for a, b in zip(th, g["theta_hat"]):
        assert a == pytest.approx(b, rel=1e-4), (th, g["theta_hat"])
    assert ll == pytest.approx(g["loglik"], rel=1e-10)
    # the closed-form l(s, theta2, theta3) equals a direct evaluation at theta_hat
    assert ll == pytest.approx(ctx.loglik(x, y, z, th).loglik, rel=1e-12)
    assert np.max(trace[:, 3]) == ll
    # theta1 of every trace row is the profile maximiser q/n of its (theta2, theta3) (oracle)
    for row in trace[:: max(1, len(trace) // 5)]:
        assert row[0] == pytest.approx(oracle.profile_sigma2(x, y, z, row[1], row[2]), rel=1e-10)


@pytest.mark.parametrize("nu_true", [0.5, 1.0])
def test_mle_profile_config2_fewer_evals(ctx, nu_true):
    n = 1600
    x, y = ex.gen_locations(n, 2)
    z = ctx.simulate(x, y, si.normals(n, 2), (1.0, 0.1, nu_true))
    start = tuple(math.sqrt(a * b) for a, b in zip(LO, HI))
    th3, ll3, ne3, _ = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-9, max_evals=3000)
    th2, ll2, ne2, _ = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-9, max_evals=3000, profile=True)
    assert ll2 >= ll3 - 1e-9 * abs(ll3)
    for a, b in zip(th2, th3):
        assert a == pytest.approx(b, rel=1e-4)
    assert ne2 < ne3


def test_mle_profile_sigma2_bound_active(ctx):
    n = 400
    x, y = ex.gen_locations(n, 4)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 4))
    lo, hi = (0.01, 0.01, 0.1), (0.3, 2.0, 2.0)  # q/n ~ 1 lies above hi.sigma2
    th, ll, _, _ = ctx.mle(x, y, z, lo, hi, (0.1, 0.1, 0.5), xtol_rel=1e-9, profile=True)
    assert th[0] == 0.3
    assert ll == pytest.approx(ctx.loglik(x, y, z, th).loglik, rel=1e-12)
    thf, llf, _, _ = ctx.mle(x, y, z, lo, hi, (0.1, 0.1, 0.5), xtol_rel=1e-9)
    assert ll >= llf - 1e-9 * abs(llf)


@pytest.mark.parametrize("profile", [False, True])
def test_mle_trust_region_matches_oracle_estimate(ctx, profile):
    # the quadratic-model trust region (BOBYQA class) reaches the oracle's estimate too
    g = json.load(open(GOLDEN))
    n = g["n"]
    x, y = ex.gen_locations(n, g["seed"])
    z = oracle.simulate(x, y, tuple(g["theta_true"]), si.normals(n, g["seed"]))
    th, ll, ne, trace = ctx.mle(x, y, z, tuple(g["lo"]), tuple(g["hi"]), tuple(g["start"]), xtol_rel=1e-10,
                                max_evals=3000, profile=profile, method="trust-region")
    for a, b in zip(th, g["theta_hat"]):
        assert a == pytest.approx(b, rel=1e-4), (th, g["theta_hat"])
    assert ll == pytest.approx(g["loglik"], rel=1e-10)
    assert ne == len(trace) and np.max(trace[:, 3]) == ll


@pytest.mark.parametrize("nu_true", [0.5, 1.0])
def test_mle_trust_region_config2_fewer_evals(ctx, nu_true):
    n = 1600
    x, y = ex.gen_locations(n, 2)
    z = ctx.simulate(x, y, si.normals(n, 2), (1.0, 0.1, nu_true))
    start = tuple(math.sqrt(a * b) for a, b in zip(LO, HI))
    for profile in (False, True):
        thn, lln, nen, _ = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-9, max_evals=3000, profile=profile)
        tht, llt, net, _ = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-9, max_evals=3000, profile=profile,
                                   method="trust-region")
        assert llt >= lln - 1e-9 * abs(lln)
        for a, b in zip(tht, thn):
            assert a == pytest.approx(b, rel=1e-4)
        assert net < nen, (profile, net, nen)


def test_mle_trust_region_bound_active(ctx):
    n = 400
    x, y = ex.gen_locations(n, 4)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 4))
    lo, hi = (0.01, 0.01, 0.1), (5.0, 0.05, 2.0)  # the range bound binds (truth 0.1)
    th, ll, _, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.02, 0.5), xtol_rel=1e-9, method="trust-region")
    assert th[1] == pytest.approx(0.05, rel=1e-12)
    thn, lln, _, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.02, 0.5), xtol_rel=1e-9)
    assert ll >= lln - 1e-9 * abs(lln)


def test_mle_monte_carlo_median_near_truth(ctx):
    # statistical sanity: over independent fields the estimates centre on the
    # truth (not exact; 12 replicas at n = 900)
    n, truth = 900, (1.0, 0.1, 0.7)
    x, y = ex.gen_locations(n, 1)
    start = tuple(math.sqrt(a * b) for a, b in zip(LO, HI))
    est = []
    for r in range(12):
        z = ctx.simulate(x, y, si.normals(n, 500 + r), truth)
        th, _, _, _ = ctx.mle(x, y, z, LO, HI, start, xtol_rel=1e-6, profile=True, method="trust-region")
        est.append(th)
    med = np.median(np.array(est), axis=0)
    assert abs(med[0] - 1.0) < 0.25 and abs(med[1] - 0.1) < 0.025 and abs(med[2] - 0.7) < 0.07, med


def test_mle_trust_region_one_and_zero_free_parameters(ctx):
    n = 600
    x, y = ex.gen_locations(n, 6)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.8), si.normals(n, 6))
    # profiled, beta fixed: a 1-D trust-region search over nu
    lo, hi = (0.01, 0.1, 0.1), (5.0, 0.1, 2.0)
    t1, l1, _, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.1, 0.5), xtol_rel=1e-8, profile=True, method="trust-region")
    t2, l2, _, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.1, 0.5), xtol_rel=1e-8, profile=True)
    assert t1[1] == 0.1 and t2[1] == 0.1
    assert t1[2] == pytest.approx(t2[2], rel=1e-5) and l1 >= l2 - 1e-9 * abs(l2)
    # profiled with beta and nu fixed: no search at all, theta1 = clamp(q / n) in closed form
    lo, hi = (0.01, 0.1, 0.8), (5.0, 0.1, 0.8)
    t3, l3, ne, _ = ctx.mle(x, y, z, lo, hi, (1.0, 0.1, 0.8), profile=True, method="trust-region")
    assert ne == 1 and t3[1:] == (0.1, 0.8)
    assert t3[0] == pytest.approx(oracle.profile_sigma2(x, y, z, 0.1, 0.8), rel=1e-10)
    assert l3 == pytest.approx(ctx.loglik(x, y, z, t3).loglik, rel=1e-12)
