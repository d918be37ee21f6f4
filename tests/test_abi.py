"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/exageo.h declares, the host-side location generator is
bit-exact against the independent oracle generator, and the product refuses
to run without a CUDA device (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_1708_02835_b200 as ex

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "exageo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(exageo_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported_and_bound():
    lib = ex.load_library()
    names = declared_symbols()
    assert len(names) >= 15
    bound = {n for n, _, _ in ex.SIGNATURES}
    for n in names:
        assert hasattr(lib, n), f"{n} declared in exageo.h but not exported"
        assert n in bound, f"{n} has no Python binding"


def test_strerror_and_workspace_size():
    assert ex.strerror(ex.ENOTPD).startswith("covariance")
    # n = 100k, nb = 512: T = 196 panels, 8 * 512 * sum_j (N - 512 j + 128) bytes
    T, nb = 196, 512
    N = T * nb
    expect = 8 * nb * sum(N - nb * j + 128 for j in range(T)) + 256 * 8
    assert ex.workspace_bytes(100_000, 512) == expect
    T2, nb2 = 49, 2048  # auto nb = 2048 at n >= 56k (single GPU)
    N2 = T2 * nb2
    assert ex.workspace_bytes(100_000) == 8 * nb2 * sum(N2 - nb2 * j + 128 for j in range(T2)) + 256 * 8


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 9), (400, 1), (401, 3), (1600, 1), (9999, 77), (100_000, 1)])
def test_locations_bit_exact_vs_oracle(n, seed):
    x, y = ex.gen_locations(n, seed)
    xo, yo = oracle.gen_locations(n, seed)
    assert x.tobytes() == xo.tobytes()
    assert y.tobytes() == yo.tobytes()


def test_locations_invalid():
    with pytest.raises(ex.ExageoError):
        ex.gen_locations(0, 1)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ex.ExageoError) as ei:
        ex.Context()
    assert ei.value.status == ex.ECUDA
