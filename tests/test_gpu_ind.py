"""GPU IND approximation (NEXT-3): annihilating the tiles outside the diagonal
super tiles makes Sigma block diagonal over consecutive groups of s * nb locations, so
l_IND must equal the sum of the ORACLE's exact log-likelihoods of those groups (the
(n_b/2) log 2 pi terms add up); s >= T must reproduce the exact path bit for bit; the
distributed schedule must agree; and skipping the zero tiles must make it cheaper."""
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

from tests._tol import LOG2PI, assert_ll  # noqa: E402,F401


def block_sum_oracle(x, y, z, theta, width):
    tot = [0.0, 0.0, 0.0]
    for b0 in range(0, len(z), width):
        ll, ld, qd = oracle.loglik(x[b0:b0 + width], y[b0:b0 + width], z[b0:b0 + width], theta)
        tot = [tot[0] + ll, tot[1] + ld, tot[2] + qd]
    return tot


@pytest.mark.parametrize("n,nb,s,theta", [(1000, 128, 2, (1.0, 0.1, 0.5)), (1500, 128, 3, (1.0, 0.1, 1.0)),
                                          (2300, 256, 1, (1.2, 0.07, 0.8))])
def test_ind_equals_sum_of_block_logliks(n, nb, s, theta):
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    c = ex.Context(device=0, nb=nb, ind_tiles=s)
    r = c.loglik(x, y, z, theta)
    c.close()
    ll, ld, qd = block_sum_oracle(x, y, z, theta, s * nb)
    assert_ll(r.loglik, (ll, ld, qd), n, what=(n, nb, s))
    assert r.logdet == pytest.approx(ld, rel=1e-10)


def test_ind_large_super_tile_is_exact():
    n, nb = 1700, 128
    x, y = ex.gen_locations(n, 5)
    z = si.normals(n, 6)
    a = ex.Context(device=0, nb=nb, tile_tasks=-1).loglik(x, y, z, (1.0, 0.1, 0.7))  # same (stream) schedule
    b = ex.Context(device=0, nb=nb, ind_tiles=100).loglik(x, y, z, (1.0, 0.1, 0.7))
    assert a.loglik == b.loglik


def test_ind_virtual_ranks_and_predict():
    n, nb, s = 1600, 128, 3
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    theta = (1.0, 0.1, 0.9)
    c1 = ex.Context(device=0, nb=nb, ind_tiles=s)
    cv = ex.Context(device=0, nb=nb, ind_tiles=s, virtual_ranks=3)
    assert c1.loglik(x, y, z, theta).loglik == pytest.approx(cv.loglik(x, y, z, theta).loglik, rel=1e-13)
    # prediction with the IND Sigma22 (block diagonal) and a dense Sigma12
    xn, yn = np.array([0.2, 0.55, 0.9]), np.array([0.3, 0.5, 0.95])
    got = c1.predict(x, y, z, xn, yn, theta)
    S22 = oracle.cov(x, y, x, y, theta)
    w = s * nb
    blk = np.arange(n) // w
    S22[blk[:, None] != blk[None, :]] = 0.0
    ref = oracle.cov(xn, yn, x, y, theta) @ np.linalg.solve(S22, z)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-10)
    assert np.array_equal(got, cv.predict(x, y, z, xn, yn, theta))
    c1.close()
    cv.close()


def test_ind_is_cheaper():
    n = 20000
    x, y = ex.gen_locations(n, 9)
    z = si.normals(n, 10)
    exact = ex.Context(device=0)
    ind = ex.Context(device=0, ind_tiles=4)
    for c in (exact, ind):
        c.loglik(x, y, z, (1.0, 0.1, 0.5))  # warm-up
    te = exact.loglik(x, y, z, (1.0, 0.1, 0.5)).info["ms_chol"]
    ti = ind.loglik(x, y, z, (1.0, 0.1, 0.5)).info["ms_chol"]
    assert ti < 0.6 * te, (ti, te)
