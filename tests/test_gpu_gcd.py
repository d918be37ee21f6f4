"""GPU great-circle distance (NEXT-4): lon/lat inputs, haversine distance in
the covariance generator, the dense covariance block and kriging, against the oracle
(which computes the haversine formula in long double)."""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402

from tests._tol import LOG2PI, assert_ll  # noqa: E402,F401


@pytest.fixture
def gcd():
    oracle.set_distance("great_circle", 6371.0)
    yield
    oracle.set_distance("euclidean")


def lonlat(n, seed):
    # an irregular lon/lat field over the Mississippi basin box
    rng = np.random.default_rng(seed)
    return rng.uniform(-100.0, -85.0, n), rng.uniform(30.0, 45.0, n)


def test_gcd_covariance(gcd):
    lon, lat = lonlat(300, 1)
    with ex.Context(device=0, distance="great_circle") as c:
        for theta in [(1.0, 300.0, 0.5), (1.3, 150.0, 1.2), (0.8, 500.0, 2.5)]:
            got = c.matern_cov(lon[:80], lat[:80], lon, lat, theta)
            ref = oracle.cov(lon[:80], lat[:80], lon, lat, theta)
            # distances carry ~1e-16 relative error from sin/asin in double: allow 5e-14 + conditioning
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_gcd_loglik_and_predict(gcd):
    n = 900
    lon, lat = lonlat(n, 2)
    z = np.random.default_rng(3).standard_normal(n)
    theta = (1.0, 250.0, 0.9)
    with ex.Context(device=0, nb=128, distance="great_circle") as c:
        r = c.loglik(lon, lat, z, theta)
        ll, ld, qd = oracle.loglik(lon, lat, z, theta)
        assert_ll(r.loglik, (ll, ld, qd), n, what=theta)
        lon2, lat2 = lonlat(20, 4)
        got = c.predict(lon, lat, z, lon2, lat2, theta)
        ref = oracle.predict(lon, lat, z, lon2, lat2, theta)
        assert np.abs(got - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())
