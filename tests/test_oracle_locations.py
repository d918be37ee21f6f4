"""Oracle pins: jittered-grid location generator (DESIGN R1-R3)."""
import math

import numpy as np
import pytest

import oracle


def test_splitmix64_published_vector():
    # SplitMix64 reference sequence for state 1234567 (Vigna's test vector):
    # output_k = mix(1234567 + k * gamma), gamma = 0x9E3779B97F4A7C15.
    gamma = 0x9E3779B97F4A7C15
    got = [oracle.splitmix64((1234567 + k * gamma) % 2**64) for k in range(5)]
    assert got == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                   4593380528125082431, 16408922859458223821]


@pytest.mark.parametrize("n", [1, 2, 3, 17, 400, 1000, 1600, 10007])
def test_locations_structure(n):
    x, y = oracle.gen_locations(n, 1)
    g = math.isqrt(n - 1) + 1 if n > 1 else 1
    assert g * g >= n and (g - 1) * (g - 1) < n
    assert np.all((x > 0) & (x < 1) & (y > 0) & (y < 1))
    # one point per grid cell, emitted in increasing row-major cell order
    r = np.floor(x * g).astype(np.int64)
    l = np.floor(y * g).astype(np.int64)
    q = r * g + l
    assert np.all(np.diff(q) > 0)
    # jitter bound: |g x - (r + 0.5)| <= 0.4 (+ rounding)
    assert np.all(np.abs(g * x - (r + 0.5)) <= 0.4 + 1e-12)
    assert np.all(np.abs(g * y - (l + 0.5)) <= 0.4 + 1e-12)
    if n <= 1600:
        d = np.hypot(x[:, None] - x[None, :], y[:, None] - y[None, :])
        d[np.diag_indices(n)] = np.inf
        assert d.min() >= 0.2 / g - 1e-15  # SPEC.md:80 separation


def test_locations_square_uses_every_cell_and_is_deterministic():
    x, y = oracle.gen_locations(400, 7)
    q = np.floor(x * 20).astype(int) * 20 + np.floor(y * 20).astype(int)
    assert np.array_equal(q, np.arange(400))
    x2, y2 = oracle.gen_locations(400, 7)
    assert np.array_equal(x, x2) and np.array_equal(y, y2)
    x3, _ = oracle.gen_locations(400, 8)
    assert not np.array_equal(x, x3)


def test_jitter_formula_bits():
    # x for cell q is ((r - 0.5) + (0.8 u - 0.4)) / g with u from the jitter stream
    n, seed = 16, 5
    x, y = oracle.gen_locations(n, seed)
    JIT = 0x4C4F434A49545452
    for q in range(16):
        u = (oracle.draw(seed, JIT, 2 * q) >> 11) * 2.0**-53
        v = (oracle.draw(seed, JIT, 2 * q + 1) >> 11) * 2.0**-53
        r, l = q // 4 + 1, q % 4 + 1
        assert x[q] == ((r - 0.5) + (0.8 * u - 0.4)) / 4
        assert y[q] == ((l - 0.5) + (0.8 * v - 0.4)) / 4


@pytest.mark.parametrize("n,seed", [(2, 3), (17, 1), (401, 3), (1000, 1), (10007, 5), (100_000, 1)])
def test_subset_rule_r2_independent_selection(n, seed):
    """DESIGN R2, written out independently in numpy (keys from the shared counter-based
    draw of synth_inputs, selection by a stable lexicographic sort): of the g*g cells,
    the n with the smallest (key, q) are kept and emitted in increasing q. An oracle that
    kept the first n cells, the largest keys, or emitted in key order fails here."""
    import synth_inputs as si

    g = math.isqrt(n - 1) + 1
    SUBSET = 0x4C4F43535542534B
    keys = si.draws(seed, SUBSET, g * g)
    q_all = np.arange(g * g, dtype=np.int64)
    order = np.lexsort((q_all, keys))  # primary key: draw, ties by q
    q_sel = np.sort(order[:n])
    x, y = oracle.gen_locations(n, seed)
    q = np.floor(x * g).astype(np.int64) * g + np.floor(y * g).astype(np.int64)
    assert np.array_equal(q, q_sel)
    if n < g * g:  # the rule is not "first n cells" for these sizes
        assert not np.array_equal(q_sel, np.arange(n))
    # jitter (R3) of the kept cells from the same shared draw, IEEE double, no contraction
    JIT = 0x4C4F434A49545452
    jb = si.draws(seed, JIT, 2 * g * g)
    u = (jb[2 * q_sel] >> np.uint64(11)).astype(np.float64) * 2.0**-53
    v = (jb[2 * q_sel + 1] >> np.uint64(11)).astype(np.float64) * 2.0**-53
    r = (q_sel // g + 1).astype(np.float64)
    l = (q_sel % g + 1).astype(np.float64)
    assert np.array_equal(((r - 0.5) + (0.8 * u - 0.4)) / g, x)
    assert np.array_equal(((l - 0.5) + (0.8 * v - 0.4)) / g, y)
