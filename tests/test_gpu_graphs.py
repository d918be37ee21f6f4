"""CUDA-graph replay of whole evaluations (exageo_opts.graphs): the captured graph, with
theta patched into the generator nodes on every replay, reproduces the stream-launched
evaluation bit for bit (same kernels, same fixed-order reductions), across theta changes,
non-PD evaluations, shape changes (recapture) and virtual ranks; and the oracle agrees."""
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
from tests._tol import assert_ll  # noqa: E402

THETAS = [(1.0, 0.1, 0.5), (0.7, 0.05, 1.3), (2.0, 0.2, 0.8), (1.0, 0.1, 2.5), (0.3, 0.02, 0.6)]


def _dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


@pytest.mark.parametrize("n", [400, 1600, 5000])
def test_graph_replay_bitwise_equal_to_stream_path(n):
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    X, Y, Z = _dev(x, y, z)
    with ex.Context(device=0, graphs=1) as g, ex.Context(device=0, graphs=-1) as s:
        for th in THETAS:
            a, b = g.loglik_dev(X, Y, Z, th), s.loglik_dev(X, Y, Z, th)
            assert (a.loglik, a.logdet, a.quad) == (b.loglik, b.logdet, b.quad), th
            assert a.info["kernels"] == b.info["kernels"]
            assert a.info["ms_total"] > 0 and a.info["ms_chol"] > 0
            assert a.info["trailing_launches"] == b.info["trailing_launches"]


def test_graph_matches_oracle_and_recaptures_on_shape_change():
    with ex.Context(device=0, graphs=1) as g:
        for n in (700, 300, 700):
            x, y = ex.gen_locations(n, 5)
            z = si.normals(n, 6)
            X, Y, Z = _dev(x, y, z)
            for th in THETAS[:3]:
                r = g.loglik_dev(X, Y, Z, th)
                ll, ld, qd = oracle.loglik(x, y, z, th)
                assert_ll(r.loglik, (ll, ld, qd), n, what=(n, th))


def test_graph_not_pd_then_valid():
    x = np.concatenate([ex.gen_locations(300, 1)[0], [0.5, 0.5]])
    y = np.concatenate([ex.gen_locations(300, 1)[1], [0.5, 0.5]])
    z = np.ones(302)
    X, Y, Z = _dev(x, y, z)
    with ex.Context(device=0, graphs=1) as g, ex.Context(device=0, graphs=-1) as s:
        for _ in range(2):
            with pytest.raises(ex.NotPositiveDefinite) as ei:
                g.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
            assert ei.value.pivot == 301
        xs, ys = ex.gen_locations(302, 2)
        Xs, Ys = _dev(xs, ys)
        a, b = g.loglik_dev(Xs, Ys, Z, (1.0, 0.1, 0.5)), s.loglik_dev(Xs, Ys, Z, (1.0, 0.1, 0.5))
        assert a.loglik == b.loglik


def test_graph_virtual_ranks():
    n = 1300
    x, y = ex.gen_locations(n, 7)
    z = si.normals(n, 8)
    X, Y, Z = _dev(x, y, z)
    with ex.Context(device=0, nb=128, virtual_ranks=3, graphs=1) as g, \
            ex.Context(device=0, nb=128, virtual_ranks=3, graphs=-1) as s:
        for th in THETAS[:3]:
            assert g.loglik_dev(X, Y, Z, th).loglik == s.loglik_dev(X, Y, Z, th).loglik


def test_graph_mle_identical_to_stream_mle():
    n = 900
    x, y = ex.gen_locations(n, 9)
    z = oracle.simulate(x, y, (1.0, 0.1, 0.5), si.normals(n, 9))
    lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
    start = tuple(math.sqrt(a * b) for a, b in zip(lo, hi))
    with ex.Context(device=0, graphs=1) as g, ex.Context(device=0, graphs=-1) as s:
        a = g.mle(x, y, z, lo, hi, start, xtol_rel=1e-6, profile=True)
        b = s.mle(x, y, z, lo, hi, start, xtol_rel=1e-6, profile=True)
    assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]
    assert np.array_equal(a[3], b[3])


def test_graph_ind_and_great_circle():
    # the IND mask and the haversine distance are baked into the captured kernels' arguments
    n = 1500
    x, y = ex.gen_locations(n, 11)
    z = si.normals(n, 12)
    X, Y, Z = _dev(x, y, z)
    for kw in ({"ind_tiles": 3, "nb": 128}, {"distance": "great_circle", "radius": 1.0}):
        with ex.Context(device=0, graphs=1, **kw) as g, ex.Context(device=0, graphs=-1, **kw) as s:
            for th in THETAS[:3]:
                a, b = g.loglik_dev(X, Y, Z, th), s.loglik_dev(X, Y, Z, th)
                assert (a.loglik, a.logdet, a.quad) == (b.loglik, b.logdet, b.quad), (kw, th)


def test_graph_closed_form_to_general_nu_recapture():
    # nu = 1/2 needs no table kernel, general nu does: switching recaptures, results stay exact
    n = 800
    x, y = ex.gen_locations(n, 13)
    z = si.normals(n, 14)
    X, Y, Z = _dev(x, y, z)
    seq = [(1.0, 0.1, 0.5), (1.0, 0.1, 0.9), (1.0, 0.1, 1.5), (1.0, 0.1, 0.9), (1.0, 0.1, 0.5), (1.0, 0.1, 0.61)]
    with ex.Context(device=0, graphs=1) as g, ex.Context(device=0, graphs=-1) as s:
        for th in seq:
            assert g.loglik_dev(X, Y, Z, th).loglik == s.loglik_dev(X, Y, Z, th).loglik, th
