"""The NCCL code path on one GPU: a single-rank NCCL communicator (world = 1 with an
NCCL id) drives every collective of the distributed schedule -- panel broadcasts,
the {logdet, quad} and pivot all-reduces, simulate's z all-reduce and predict's w_j
broadcasts -- through the run-time-loaded NCCL. Results must equal the plain
single-GPU path bit for bit (a one-rank sum is exact)."""
import numpy as np
import pytest

import oracle
import synth_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402


def test_single_rank_nccl_equals_plain():
    n = 1500
    x, y = ex.gen_locations(n, 1)
    e = si.normals(n, 2)
    theta = (1.0, 0.1, 0.8)
    plain = ex.Context(device=0, nb=128, tile_tasks=-1)  # the NCCL context's schedule
    nc = ex.Context(device=0, nb=128, world=1, rank=0, nccl_id=ex.nccl_unique_id())
    z1 = plain.simulate(x, y, e, theta)
    z2 = nc.simulate(x, y, e, theta)
    assert np.array_equal(z1, z2)
    a = plain.loglik(x, y, z1, theta)
    b = nc.loglik(x, y, z1, theta)
    assert a.loglik == b.loglik and a.logdet == b.logdet and a.quad == b.quad
    xn, yn = np.array([0.25, 0.8]), np.array([0.6, 0.1])
    assert np.array_equal(plain.predict(x, y, z1, xn, yn, theta), nc.predict(x, y, z1, xn, yn, theta))
    # non-PD through the NCCL pivot all-reduce
    xd = np.concatenate([x[:100], x[:1]])
    yd = np.concatenate([y[:100], y[:1]])
    with pytest.raises(ex.NotPositiveDefinite) as ei:
        nc.loglik(xd, yd, np.ones(101), theta)
    assert ei.value.pivot == 100
    plain.close()
    nc.close()


def test_nccl_graph_replay_equals_stream_launch():
    """CUDA-graph replay with NCCL collectives captured in the graph (the {logdet, quad} and the
    pivot all-reduces): bitwise equal to stream launches, over several theta (patched per
    replay), and ENOTPD with the all-reduced pivot through the graph."""
    n = 1300
    x, y = ex.gen_locations(n, 3)
    z = si.normals(n, 4)
    uid = ex.nccl_unique_id()
    g = ex.Context(device=0, nb=128, world=1, rank=0, nccl_id=uid, graphs=1)
    s = ex.Context(device=0, nb=128, world=1, rank=0, nccl_id=ex.nccl_unique_id(), graphs=-1)
    for th in [(1.0, 0.1, 0.5), (0.7, 0.2, 1.3), (1.5, 0.05, 0.9)]:
        a, b = g.loglik(x, y, z, th), s.loglik(x, y, z, th)
        assert a.loglik == b.loglik and a.logdet == b.logdet and a.quad == b.quad, th
    xd = np.concatenate([x[:200], x[:1]])
    yd = np.concatenate([y[:200], y[:1]])
    for c in (g, s):
        with pytest.raises(ex.NotPositiveDefinite) as ei:
            c.loglik(xd, yd, np.ones(201), (1.0, 0.1, 0.5))
        assert ei.value.pivot == 200
    assert np.isfinite(g.loglik(x, y, z, (1.0, 0.1, 0.5)).loglik)  # recovers after the failure
    g.close()
    s.close()
