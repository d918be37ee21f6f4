"""Oracle pins for the distance metrics: Euclidean hand cases and the
great-circle (haversine) distance against hand cases (antipodes, quarter
circumference) and an independent formula (chord length of unit vectors:
d = 2 R asin(|u1 - u2| / 2))."""
import math

import numpy as np
import pytest

import oracle


@pytest.fixture
def gcd():
    oracle.set_distance("great_circle", 6371.0)
    yield
    oracle.set_distance("euclidean")


def test_euclidean_hand_cases():
    oracle.set_distance("euclidean")
    assert oracle.distance(0, 0, 0, 0) == 0.0
    assert oracle.distance(0, 0, 3, 4) == 5.0
    assert oracle.distance(0.1, 0.2, 0.4, 0.6) == pytest.approx(0.5, rel=1e-15)


def test_great_circle_hand_cases(gcd):
    assert oracle.distance(12.5, -33.0, 12.5, -33.0) == 0.0
    assert oracle.distance(0, 0, 90, 0) == pytest.approx(math.pi * 6371.0 / 2, rel=1e-15)
    oracle.set_distance("great_circle", 1.0)
    assert oracle.distance(0, 0, 180, 0) == pytest.approx(math.pi, rel=1e-15)
    assert oracle.distance(0, -90, 0, 90) == pytest.approx(math.pi, rel=1e-15)


def test_great_circle_vs_chord_formula(gcd):
    rng = np.random.default_rng(0)
    for _ in range(200):
        lon1, lon2 = rng.uniform(-180, 180, 2)
        lat1, lat2 = rng.uniform(-89, 89, 2)
        u = [np.array([math.cos(math.radians(la)) * math.cos(math.radians(lo)),
                       math.cos(math.radians(la)) * math.sin(math.radians(lo)), math.sin(math.radians(la))])
             for lo, la in ((lon1, lat1), (lon2, lat2))]
        ref = 2 * 6371.0 * math.asin(min(1.0, np.linalg.norm(u[0] - u[1]) / 2))
        got = oracle.distance(lon1, lat1, lon2, lat2)
        assert got == pytest.approx(ref, rel=1e-12, abs=1e-9)
        assert got == oracle.distance(lon2, lat2, lon1, lat1)


def test_great_circle_loglik_is_permutation_invariant(gcd):
    rng = np.random.default_rng(1)
    n = 150
    lon, lat = rng.uniform(-100, -85, n), rng.uniform(30, 45, n)
    z = rng.standard_normal(n)
    theta = (1.0, 300.0, 0.7)  # range in km
    a = oracle.loglik(lon, lat, z, theta)[0]
    p = rng.permutation(n)
    assert oracle.loglik(lon[p], lat[p], z[p], theta)[0] == pytest.approx(a, rel=1e-12)
