"""CPU oracle for the exact Gaussian log-likelihood -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct implementation of arXiv 1708.02835's hot path
(Eq. 1, Eq. 2, Alg. 1-3) in C (``oracle.c``), loaded with ctypes. Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package. It shares no code with the
product package ``paper_1708_02835_b200`` and neither imports the other.

Parity pins (what the oracle is checked against, ``tests/test_oracle_*.py``):
  * K_nu: half-integer closed forms, the three-term recurrence, mpmath besselk.
  * Gamma: Gamma(1/2) = sqrt(pi), factorials, mpmath gamma.
  * Matern: nu=1/2 exponential reduction and nu=1 Whittle form,
    nu=3/2, 5/2 closed forms, C(0)=theta1, linearity in theta1.
  * Cholesky: L L^T = Sigma, 2x2 hand case, log|cI| = n log c, exact rational
    determinant (fractions) for n <= 7.
  * loglik: n=1 and n=2 closed forms, AR(1)/Kac-Murdock-Szego closed form,
    Sigma = theta1 I at widely spaced sites, permutation invariance,
    scipy.stats.multivariate_normal.logpdf.
  * locations: SplitMix64 published test vector, bounds, separation, one point
    per grid cell.
No oracle function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_splitmix64.restype = ctypes.c_uint64
        L.oracle_splitmix64.argtypes = [ctypes.c_uint64]
        L.oracle_draw.restype = ctypes.c_uint64
        L.oracle_draw.argtypes = [ctypes.c_uint64] * 3
        L.oracle_gen_locations.restype = ctypes.c_int
        L.oracle_gen_locations.argtypes = [ctypes.c_int64, ctypes.c_uint64, _f64p, _f64p]
        L.oracle_gamma.restype = ctypes.c_double
        L.oracle_gamma.argtypes = [ctypes.c_double]
        L.oracle_bessel_k.restype = ctypes.c_double
        L.oracle_bessel_k.argtypes = [ctypes.c_double, ctypes.c_double]
        L.oracle_matern.restype = ctypes.c_double
        L.oracle_matern.argtypes = [ctypes.c_double] * 4
        L.oracle_cov.restype = None
        L.oracle_cov.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.c_int64, _f64p, _f64p,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double, _f64p, ctypes.c_int64]
        L.oracle_cholesky.restype = ctypes.c_int64
        L.oracle_cholesky.argtypes = [ctypes.c_int64, _f64p]
        L.oracle_forward.restype = None
        L.oracle_forward.argtypes = [ctypes.c_int64, _f64p, _f64p, _f64p]
        L.oracle_backward.restype = None
        L.oracle_backward.argtypes = [ctypes.c_int64, _f64p, _f64p, _f64p]
        L.oracle_loglik.restype = ctypes.c_int
        L.oracle_loglik.argtypes = [ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, _f64p, _i64p]
        L.oracle_simulate.restype = ctypes.c_int
        L.oracle_simulate.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, _f64p, _f64p, _i64p]
        L.oracle_predict.restype = ctypes.c_int
        L.oracle_predict.argtypes = [ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.c_int64, _f64p, _f64p,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _f64p, _i64p]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_distance.restype = None
        L.oracle_set_distance.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oracle_distance.restype = ctypes.c_double
        L.oracle_distance.argtypes = [ctypes.c_double] * 4
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_f64p)


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class NotPositiveDefinite(RuntimeError):
    def __init__(self, pivot: int):
        super().__init__(f"covariance not positive definite at pivot {pivot}")
        self.pivot = pivot


def splitmix64(v: int) -> int:
    return int(lib().oracle_splitmix64(ctypes.c_uint64(v & (2**64 - 1))))


def draw(seed: int, stream: int, i: int) -> int:
    return int(lib().oracle_draw(seed, stream, i))


def gen_locations(n: int, seed: int):
    """Jittered-grid locations (DESIGN R1-R3) -> (x, y) float64."""
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    rc = lib().oracle_gen_locations(n, seed, _p(x), _p(y))
    if rc != 0:
        raise ValueError(f"oracle_gen_locations rc={rc}")
    return x, y


def gamma(z: float) -> float:
    return lib().oracle_gamma(z)


def bessel_k(nu: float, x: float) -> float:
    return lib().oracle_bessel_k(nu, x)


def matern(r: float, theta) -> float:
    t1, t2, t3 = theta
    return lib().oracle_matern(r, t1, t2, t3)


def cov(x1, y1, x2, y2, theta) -> np.ndarray:
    """Dense m x n covariance block (Alg. 3 l.3-6), returned as an (m, n) array."""
    x1, y1, x2, y2 = _f(x1), _f(y1), _f(x2), _f(y2)
    m, n = x1.size, x2.size
    C = np.empty((n, m), np.float64)  # column-major m x n == row-major n x m
    lib().oracle_cov(m, _p(x1), _p(y1), n, _p(x2), _p(y2), *map(float, theta), _p(C), m)
    return C.T.copy()


def cholesky(A) -> np.ndarray:
    """Unblocked Cholesky; returns lower L (upper triangle zeroed)."""
    S = _f(A).copy()
    n = S.shape[0]
    p = lib().oracle_cholesky(n, _p(S))
    if p >= 0:
        raise NotPositiveDefinite(int(p))
    return np.tril(S)


def forward(L, z) -> np.ndarray:
    L, z = _f(L), _f(z)
    y = np.empty_like(z)
    lib().oracle_forward(z.size, _p(L), _p(z), _p(y))
    return y


def backward(L, y) -> np.ndarray:
    L, y = _f(L), _f(y)
    x = np.empty_like(y)
    lib().oracle_backward(y.size, _p(L), _p(y), _p(x))
    return x


def loglik(x, y, z, theta):
    """Alg. 2 / Eq. (1). Returns (loglik, logdet, quad)."""
    x, y, z = _f(x), _f(y), _f(z)
    out = np.zeros(3, np.float64)
    piv = ctypes.c_int64(-1)
    rc = lib().oracle_loglik(z.size, _p(x), _p(y), _p(z), *map(float, theta), _p(out), ctypes.byref(piv))
    if rc == -2:
        raise NotPositiveDefinite(piv.value)
    if rc != 0:
        raise RuntimeError(f"oracle_loglik rc={rc}")
    return float(out[0]), float(out[1]), float(out[2])


def simulate(x, y, theta, e) -> np.ndarray:
    """Alg. 1: z = L(theta) e."""
    x, y, e = _f(x), _f(y), _f(e)
    z = np.empty_like(e)
    piv = ctypes.c_int64(-1)
    rc = lib().oracle_simulate(e.size, _p(x), _p(y), *map(float, theta), _p(e), _p(z), ctypes.byref(piv))
    if rc == -2:
        raise NotPositiveDefinite(piv.value)
    if rc != 0:
        raise RuntimeError(f"oracle_simulate rc={rc}")
    return z


def predict(x, y, z, xnew, ynew, theta) -> np.ndarray:
    """Alg. 3 / Eq. (5): Z1 = Sigma12 Sigma22^{-1} Z2."""
    x, y, z, xnew, ynew = _f(x), _f(y), _f(z), _f(xnew), _f(ynew)
    out = np.empty(xnew.size, np.float64)
    piv = ctypes.c_int64(-1)
    rc = lib().oracle_predict(z.size, _p(x), _p(y), _p(z), xnew.size, _p(xnew), _p(ynew),
                              *map(float, theta), _p(out), ctypes.byref(piv))
    if rc == -2:
        raise NotPositiveDefinite(piv.value)
    if rc != 0:
        raise RuntimeError(f"oracle_predict rc={rc}")
    return out


def predict_var(x, y, xnew, ynew, theta) -> np.ndarray:
    """Simple-kriging (conditional) variance of Eq. (5)'s predictor at each new site,
    var_i = C(0) - sigma_i^T Sigma22^{-1} sigma_i with sigma_i = Sigma21[:, i],
    as theta1 - ||L^{-1} sigma_i||^2 by the oracle's own Cholesky and forward substitution."""
    L = cholesky(cov(x, y, x, y, theta))
    S = cov(x, y, xnew, ynew, theta)  # n x m
    out = np.empty(S.shape[1])
    for i in range(S.shape[1]):
        w = forward(L, S[:, i])
        out[i] = float(theta[0]) - float(w @ w)
    return out


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_distance(metric: str = "euclidean", radius: float = 6371.0) -> None:
    """Distance used by every oracle routine: 'euclidean' or 'great_circle'
    (haversine; x = longitude, y = latitude in degrees)."""
    lib().oracle_set_distance({"euclidean": 0, "great_circle": 1}[metric], float(radius))


def distance(x1: float, y1: float, x2: float, y2: float) -> float:
    return float(lib().oracle_distance(x1, y1, x2, y2))


def mle(x, y, z, lo, hi, start, xtol: float = 1e-10, max_evals: int = 4000):
    """Oracle MLE: maximise the oracle's l(theta) over lo <= theta <= hi.

    Library optimisers as steps (R16: any derivative-free bound-constrained search):
    scipy Nelder-Mead on log(theta) from `start`, polished by L-BFGS-B (finite
    differences). Non-PD evaluations count as l = -inf. Returns (theta_hat, l, nevals)."""
    import scipy.optimize as so

    x, y, z = _f(x), _f(y), _f(z)
    lo_u, hi_u = np.log(np.asarray(lo, float)), np.log(np.asarray(hi, float))
    cnt = [0]

    def f(u):
        cnt[0] += 1
        u = np.clip(u, lo_u, hi_u)
        try:
            return -loglik(x, y, z, np.exp(u))[0]
        except NotPositiveDefinite:
            return 1e300

    b = list(zip(lo_u, hi_u))
    r = so.minimize(f, np.log(np.asarray(start, float)), method="Nelder-Mead", bounds=b,
                    options=dict(xatol=xtol, fatol=1e-13, maxfev=max_evals, adaptive=True))
    r2 = so.minimize(f, r.x, method="L-BFGS-B", bounds=b, options=dict(ftol=1e-15, gtol=1e-10, maxfun=max_evals))
    best = r2 if r2.fun <= r.fun else r
    return tuple(np.exp(np.clip(best.x, lo_u, hi_u))), -float(best.fun), cnt[0]


def profile_sigma2(x, y, z, beta: float, nu: float) -> float:
    """theta1 maximising l for fixed (theta2, theta3): z^T R^{-1} z / n, R = Sigma(1, theta2, theta3).

    From Eq. (1) with Sigma = theta1 R: dl/dtheta1 = -n/(2 theta1) + z^T R^{-1} z / (2 theta1^2) = 0."""
    _, _, quad = loglik(x, y, z, (1.0, beta, nu))
    return quad / len(z)
