"""Parity gates for l(theta) shared by the GPU tests.

Two gates, both asserted for every l comparison against the oracle:
  * plain relative:  |dl| / |l| <= 1e-10 (BASELINE.json north_star, fp64);
  * R13 guard:       |dl| <= 1e-10 * max(|l|, |logdet|/2, quad/2, (n/2) log 2 pi),
    which only matters when l itself is small through cancellation between the terms
    of Eq. (1); it is never looser than the plain gate when |l| dominates.
Where the plain gate cannot hold for a mathematical reason (cancellation, an
ill-conditioned Sigma), the caller passes plain=False or its own bound and says why.
"""
import math

LOG2PI = math.log(2.0 * math.pi)
REL = 1e-10


def r13_tol(ll, logdet, quad, n, rel=REL):
    return rel * max(abs(ll), 0.5 * abs(logdet), 0.5 * abs(quad), 0.5 * n * LOG2PI)


def assert_ll(got, ref, n, plain=True, rel=REL, what=""):
    """got: GPU l; ref: the oracle's (l, logdet, quad). Returns |dl| / |l|."""
    ll, logdet, quad = ref
    d = abs(got - ll)
    assert d <= r13_tol(ll, logdet, quad, n, rel), (what, got, ll, d)
    r = d / abs(ll) if ll != 0 else (0.0 if d == 0 else math.inf)
    if plain:
        assert r <= rel, (what, "plain |dl|/|l|", got, ll, r)
    return r
