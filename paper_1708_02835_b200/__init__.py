"""paper_1708_02835_b200 -- B200-native exact Gaussian log-likelihood (ExaGeoStat hot path).

Thin ctypes binding over the C ABI in ``include/exageo.h`` (libexageo.so, built
in-tree by ``paper_1708_02835_b200.build``). The functions keep the C names
without the ``exageo_`` prefix and do argument marshalling only: every step of
the evaluation runs in the library's CUDA kernels. There is no CPU fallback --
if the shared library is missing or no CUDA device is usable, the calls raise.

Host arrays are numpy float64; the ``*_dev`` variants take torch CUDA float64
tensors (torch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libexageo.so")

OK, EINVAL, ENOTPD, ENOMEM, ECUDA, ENCCL, EFIT = 0, -1, -2, -3, -4, -5, -6

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class Theta(ctypes.Structure):
    _fields_ = [("sigma2", ctypes.c_double), ("beta", ctypes.c_double), ("nu", ctypes.c_double)]


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("nb", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("world", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("virtual_ranks", ctypes.c_int), ("ind_tiles", ctypes.c_int), ("distance", ctypes.c_int),
                ("radius", ctypes.c_double), ("graphs", ctypes.c_int), ("grid_rows", ctypes.c_int),
                ("tile_tasks", ctypes.c_int)]


class MleOpts(ctypes.Structure):
    _fields_ = [("xtol_rel", ctypes.c_double), ("max_evals", ctypes.c_int), ("profile", ctypes.c_int),
                ("method", ctypes.c_int)]


class LoglikInfo(ctypes.Structure):
    _fields_ = [("loglik", ctypes.c_double), ("logdet", ctypes.c_double), ("quad", ctypes.c_double),
                ("npd_pivot", ctypes.c_int64), ("n", ctypes.c_int64), ("nb", ctypes.c_int64),
                ("ntiles", ctypes.c_int64), ("flops", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_gen", ctypes.c_double), ("ms_chol", ctypes.c_double), ("ms_reduce", ctypes.c_double),
                ("kernels", ctypes.c_int64), ("trailing_launches", ctypes.c_int64),
                ("ms_trailing", ctypes.c_double), ("trailing_flops", ctypes.c_double),
                ("update_launches", ctypes.c_int64), ("ms_update_union", ctypes.c_double),
                ("update_flops", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


# (name, restype, argtypes) of every symbol declared in include/exageo.h
_C = ctypes.c_void_p
SIGNATURES = [
    ("exageo_strerror", ctypes.c_char_p, [ctypes.c_int]),
    ("exageo_last_error", ctypes.c_char_p, [_C]),
    ("exageo_nccl_unique_id", ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    ("exageo_create", ctypes.c_int, [ctypes.POINTER(_C), ctypes.POINTER(Opts)]),
    ("exageo_destroy", None, [_C]),
    ("exageo_workspace_bytes", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int]),
    ("exageo_rank_workspace_bytes", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_int]),
    ("exageo_set_workspace", ctypes.c_int, [_C, ctypes.c_void_p, ctypes.c_size_t]),
    ("exageo_stream_wait", ctypes.c_int, [_C, ctypes.c_void_p]),
    ("exageo_gen_locations", ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64, _f64p, _f64p]),
    ("exageo_matern_cov", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, _f64p, _f64p, ctypes.c_int64,
                                         _f64p, _f64p, _f64p, ctypes.c_int64]),
    ("exageo_loglik", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, _f64p, _f64p, _f64p, _f64p,
                                     ctypes.POINTER(LoglikInfo)]),
    ("exageo_loglik_dev", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, _f64p, ctypes.POINTER(LoglikInfo)]),
    ("exageo_simulate", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, _f64p, _f64p, _f64p, _f64p]),
    ("exageo_stage_generate_dev", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p]),
    ("exageo_stage_factor", ctypes.c_int, [_C]),
    ("exageo_stage_finish", ctypes.c_int, [_C, _f64p, _i64p]),
    ("exageo_read_lower", ctypes.c_int, [_C, _f64p, ctypes.c_int64]),
    ("exageo_read_zrow", ctypes.c_int, [_C, _f64p]),
    ("exageo_read_entries", ctypes.c_int, [_C, ctypes.c_int64, _i64p, _i64p, _f64p]),
    ("exageo_predict_var", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, _f64p, _f64p, _f64p,
                                          ctypes.c_int64, _f64p, _f64p, _f64p, _f64p]),
    ("exageo_predict", ctypes.c_int, [_C, ctypes.POINTER(Theta), ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.c_int64,
                                      _f64p, _f64p, _f64p]),
    ("exageo_mle", ctypes.c_int, [_C, ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.POINTER(Theta),
                                  ctypes.POINTER(Theta), ctypes.POINTER(Theta), ctypes.c_double, ctypes.c_int,
                                  ctypes.POINTER(Theta), _f64p, ctypes.POINTER(ctypes.c_int), _f64p]),
    ("exageo_mle_profile", ctypes.c_int, [_C, ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.POINTER(Theta),
                                          ctypes.POINTER(Theta), ctypes.POINTER(Theta), ctypes.c_double, ctypes.c_int,
                                          ctypes.POINTER(Theta), _f64p, ctypes.POINTER(ctypes.c_int), _f64p]),
    ("exageo_mle_ex", ctypes.c_int, [_C, ctypes.c_int64, _f64p, _f64p, _f64p, ctypes.POINTER(Theta),
                                     ctypes.POINTER(Theta), ctypes.POINTER(Theta), ctypes.POINTER(MleOpts),
                                     ctypes.POINTER(Theta), _f64p, ctypes.POINTER(ctypes.c_int), _f64p]),
]

_lib = None


def load_library():
    """Load libexageo.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_1708_02835_b200.build` "
                               "(this package has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class ExageoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{strerror(status)}: {msg}")
        self.status = status


class NotPositiveDefinite(ExageoError):
    def __init__(self, status: int, msg: str, pivot: int):
        super().__init__(status, msg)
        self.pivot = pivot


def strerror(status: int) -> str:
    return load_library().exageo_strerror(status).decode()


def _p(a: np.ndarray):
    return a.ctypes.data_as(_f64p)


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _theta(theta) -> Theta:
    t1, t2, t3 = (float(v) for v in theta)
    return Theta(t1, t2, t3)


def gen_locations(n: int, seed: int):
    """Jittered-grid locations (DESIGN R1-R3) -> (x, y) numpy float64."""
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    st = load_library().exageo_gen_locations(int(n), int(seed) & (2**64 - 1), _p(x), _p(y))
    if st != OK:
        raise ExageoError(st, load_library().exageo_last_error(None).decode())
    return x, y


def workspace_bytes(n: int, nb: int = 0) -> int:
    return int(load_library().exageo_workspace_bytes(int(n), int(nb)))


def rank_workspace_bytes(n: int, nb: int, world: int, grid_rows: int, rank: int) -> int:
    """Device workspace of one rank of a grid_rows x (world / grid_rows) process grid (host-only)."""
    return int(load_library().exageo_rank_workspace_bytes(int(n), int(nb), int(world), int(grid_rows), int(rank)))


@dataclass
class Result:
    loglik: float
    logdet: float
    quad: float
    info: dict


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (create on rank 0, share with every rank)."""
    import torch  # noqa: F401  -- load torch's libnccl first; the library then reuses it

    buf = ctypes.create_string_buffer(128)
    st = load_library().exageo_nccl_unique_id(buf, 128)
    if st != OK:
        raise ExageoError(st, load_library().exageo_last_error(None).decode())
    return buf.raw


def exchange_nccl_id(rank: int, world: int) -> bytes:
    """NCCL id of rank 0, broadcast to every rank over the default torch.distributed group."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone()
    if dist.get_backend() == "nccl":
        tt = t.cuda()
        dist.broadcast(tt, 0)
        t = tt.cpu()
    else:
        dist.broadcast(t, 0)
    return bytes(t.tolist())


class Context:
    """An exageo_ctx on one CUDA device (own stream unless `stream` is given).

    Distribution: world > 1 with rank and nccl_id (bytes, identical on every rank)
    makes a collective NCCL context; virtual_ranks > 1 runs that many ranks of the
    distributed schedule inside this process on one device; grid_rows = P arranges the
    ranks as a P x (ranks / P) process grid with tile (I, J) on rank (I mod P, J mod Q) (the
    2-D block-cyclic distribution; 0/1 = 1 x ranks); ind_tiles > 0 selects the IND
    approximation with diagonal super tiles of ind_tiles tiles; graphs selects
    CUDA-graph replay of whole evaluations (0 automatic for n <= 32768, 1 always, -1 never);
    tile_tasks selects the persistent tile-task kernel for the factorization of single-rank
    contexts (0 automatic for n <= 3200, 1 always, -1 never)."""

    def __init__(self, device: int = 0, nb: int = 0, stream=None, world: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, virtual_ranks: int = 0, ind_tiles: int = 0,
                 distance: str = "euclidean", radius: float = 6371.0, graphs: int = 0, grid_rows: int = 0,
                 tile_tasks: int = 0):
        self._lib = load_library()
        self._ctx = ctypes.c_void_p()
        sp = None
        if stream is not None:
            sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._id_buf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        idp = ctypes.cast(self._id_buf, ctypes.c_void_p) if self._id_buf is not None else None
        metric = {"euclidean": 0, "great_circle": 1, "gcd": 1}[distance]
        o = Opts(int(device), int(nb), sp, int(world), int(rank), idp, int(virtual_ranks), int(ind_tiles), metric,
                 float(radius), int(graphs), int(grid_rows), int(tile_tasks))
        st = self._lib.exageo_create(ctypes.byref(self._ctx), ctypes.byref(o))
        if st != OK:
            raise ExageoError(st, self._lib.exageo_last_error(None).decode())
        self._workspace = None
        self.device = int(device)

    # -- plumbing ---------------------------------------------------------
    def close(self):
        if self._ctx:
            self._lib.exageo_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st: int, pivot: int = -1):
        if st == OK:
            return
        msg = self._lib.exageo_last_error(self._ctx).decode()
        if st == ENOTPD:
            raise NotPositiveDefinite(st, msg, pivot)
        raise ExageoError(st, msg)

    def set_workspace(self, tensor):
        """Use a caller-owned torch CUDA tensor as tile workspace (None = library-managed)."""
        if tensor is None:
            self._check(self._lib.exageo_set_workspace(self._ctx, None, 0))
        else:
            nbytes = tensor.numel() * tensor.element_size()
            self._check(self._lib.exageo_set_workspace(self._ctx, ctypes.c_void_p(tensor.data_ptr()), nbytes))
        self._workspace = tensor

    # -- API ----------------------------------------------------------------
    def matern_cov(self, x1, y1, x2, y2, theta) -> np.ndarray:
        """Dense (m, n) covariance block C_ij = C(||s1_i - s2_j||; theta) computed on the GPU."""
        x1, y1, x2, y2 = _f(x1), _f(y1), _f(x2), _f(y2)
        m, n = x1.size, x2.size
        C = np.empty((n, m), np.float64)  # column-major (m, n)
        t = _theta(theta)
        self._check(self._lib.exageo_matern_cov(self._ctx, ctypes.byref(t), m, _p(x1), _p(y1), n, _p(x2), _p(y2),
                                                _p(C), m))
        return C.T.copy()

    def loglik(self, x, y, z, theta) -> Result:
        """Eq. (1) through Alg. 2 with host arrays (H2D copies included)."""
        x, y, z = _f(x), _f(y), _f(z)
        t = _theta(theta)
        out = ctypes.c_double()
        info = LoglikInfo()
        st = self._lib.exageo_loglik(self._ctx, ctypes.byref(t), z.size, _p(x), _p(y), _p(z), ctypes.byref(out),
                                     ctypes.byref(info))
        self._check(st, info.npd_pivot)
        return Result(info.loglik, info.logdet, info.quad, info.as_dict())

    def _dev_inputs(self, *tensors):
        """Check device inputs (contiguous float64 on this context's device, equal lengths) and
        order the context stream after torch's current stream, which may still be writing them."""
        import torch

        n = None
        for a in tensors:
            if a is None:
                continue
            if not (a.is_cuda and a.dtype == torch.float64 and a.is_contiguous()):
                raise ValueError("device entry points need contiguous CUDA float64 tensors")
            if a.device.index != self.device:
                raise ValueError(f"tensor on cuda:{a.device.index}, context on cuda:{self.device}")
            if n is not None and a.numel() != n:
                raise ValueError("x, y and z must have the same length")
            n = a.numel()
        self._check(self._lib.exageo_stream_wait(self._ctx, ctypes.c_void_p(torch.cuda.current_stream(self.device)
                                                                             .cuda_stream)))

    def loglik_dev(self, x, y, z, theta) -> Result:
        """Eq. (1) with torch CUDA float64 tensors already resident on the device."""
        self._dev_inputs(x, y, z)
        t = _theta(theta)
        out = ctypes.c_double()
        info = LoglikInfo()
        st = self._lib.exageo_loglik_dev(self._ctx, ctypes.byref(t), z.numel(), ctypes.c_void_p(x.data_ptr()),
                                         ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                                         ctypes.byref(out), ctypes.byref(info))
        self._check(st, info.npd_pivot)
        return Result(info.loglik, info.logdet, info.quad, info.as_dict())

    def mle(self, x, y, z, lo, hi, start, xtol_rel: float = 1e-9, max_evals: int = 1000, profile: bool = False,
            method: str = "nelder-mead"):
        """Maximum-likelihood estimate over the box lo <= theta <= hi (exageo_mle_ex):
        profile=True profiles theta1 out in closed form (exageo_mle_profile); method
        "nelder-mead" (exageo_mle) or "trust-region" (quadratic-model trust region).

        Returns (theta_hat tuple, loglik, nevals, trace as an (nevals, 4) array)."""
        x, y, z = _f(x), _f(y), _f(z)
        tlo, thi, ts = _theta(lo), _theta(hi), _theta(start)
        th = Theta()
        ll = ctypes.c_double()
        ne = ctypes.c_int()
        trace = np.zeros((max_evals, 4), np.float64)
        o = MleOpts(float(xtol_rel), int(max_evals), int(bool(profile)),
                    {"nelder-mead": 0, "trust-region": 1}[method])
        st = self._lib.exageo_mle_ex(self._ctx, z.size, _p(x), _p(y), _p(z), ctypes.byref(tlo), ctypes.byref(thi),
                                     ctypes.byref(ts), ctypes.byref(o), ctypes.byref(th), ctypes.byref(ll),
                                     ctypes.byref(ne), _p(trace))
        self._check(st)
        return (th.sigma2, th.beta, th.nu), ll.value, ne.value, trace[: ne.value].copy()

    def predict(self, x, y, z, xnew, ynew, theta) -> np.ndarray:
        """Kriging predictions Z1 = Sigma12 Sigma22^{-1} Z2 at (xnew, ynew) (Eq. 5, Alg. 3)."""
        x, y, z, xnew, ynew = _f(x), _f(y), _f(z), _f(xnew), _f(ynew)
        out = np.empty(xnew.size, np.float64)
        t = _theta(theta)
        self._check(self._lib.exageo_predict(self._ctx, ctypes.byref(t), z.size, _p(x), _p(y), _p(z), xnew.size,
                                             _p(xnew), _p(ynew), _p(out)))
        return out

    def predict_var(self, x, y, z, xnew, ynew, theta):
        """Kriging mean and variance at (xnew, ynew) (exageo_predict_var): (znew, var)."""
        x, y, z, xnew, ynew = _f(x), _f(y), _f(z), _f(xnew), _f(ynew)
        out = np.empty(xnew.size, np.float64)
        var = np.empty(xnew.size, np.float64)
        t = _theta(theta)
        self._check(self._lib.exageo_predict_var(self._ctx, ctypes.byref(t), z.size, _p(x), _p(y), _p(z), xnew.size,
                                                 _p(xnew), _p(ynew), _p(out), _p(var)))
        return out, var

    def simulate(self, x, y, e, theta) -> np.ndarray:
        """Alg. 1: z = L(theta) e for given normal variates e."""
        x, y, e = _f(x), _f(y), _f(e)
        z = np.empty_like(e)
        t = _theta(theta)
        self._check(self._lib.exageo_simulate(self._ctx, ctypes.byref(t), e.size, _p(x), _p(y), _p(e), _p(z)))
        return z

    # -- stage-level access (tests) -------------------------------------------
    def stage_generate_dev(self, x, y, z, theta):
        self._dev_inputs(x, y, z)
        t = _theta(theta)
        zp = ctypes.c_void_p(z.data_ptr()) if z is not None else None
        self._check(self._lib.exageo_stage_generate_dev(self._ctx, ctypes.byref(t), x.numel(),
                                                        ctypes.c_void_p(x.data_ptr()),
                                                        ctypes.c_void_p(y.data_ptr()), zp))

    def stage_factor(self):
        self._check(self._lib.exageo_stage_factor(self._ctx))

    def stage_finish(self):
        out = np.zeros(3, np.float64)
        piv = ctypes.c_int64(-1)
        st = self._lib.exageo_stage_finish(self._ctx, _p(out), ctypes.byref(piv))
        self._check(st, piv.value)
        return float(out[0]), float(out[1]), float(out[2])

    def read_lower(self, n: int) -> np.ndarray:
        """Lower triangle of the workspace matrix as a dense (n, n) array (upper = 0)."""
        buf = np.zeros((n, n), np.float64)  # column-major n x n == row-major transpose
        self._check(self._lib.exageo_read_lower(self._ctx, _p(buf), n))
        return buf.T.copy()

    def read_zrow(self, n: int) -> np.ndarray:
        buf = np.empty(n, np.float64)
        self._check(self._lib.exageo_read_zrow(self._ctx, _p(buf)))
        return buf

    def read_entries(self, rows, cols) -> np.ndarray:
        """Entries (rows[i], cols[i]), cols <= rows, of the workspace matrix."""
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(r.size, np.float64)
        self._check(self._lib.exageo_read_entries(self._ctx, r.size, r.ctypes.data_as(_i64p),
                                                  c.ctypes.data_as(_i64p), _p(out)))
        return out


LOG2PI = math.log(2.0 * math.pi)
