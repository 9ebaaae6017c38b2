"""paper_2601_02826_b200 — B200-native FS-QRPPA hot path (Python binding of libfsqr.so).

This module only marshals arguments into the C ABI declared in include/fsqr.h;
every step of the iteration runs in the CUDA kernels of csrc/ (sm_100a).  There
is no CPU fallback: if libfsqr.so cannot be loaded, or no CUDA device is
present, calls raise.  PyTorch is used for device memory and streams only.

Function names mirror the C ABI (fsqr_create, fsqr_iterate, fsqr_solve,
fsqr_objective, ...).  `Solver` is a convenience holder that keeps the borrowed
design tensor alive for the lifetime of the context.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

F32_DENSE, U8, PACKED2 = 0, 1, 2
SCAD, MCP = 1, 2
BACKEND_AUTO, BACKEND_TC, BACKEND_SIMT = 0, 1, 2
ETA_LANCZOS, ETA_POWER = 0, 1
STATUS = {0: "FSQR_OK", 2: "FSQR_NOT_CONVERGED", -1: "FSQR_ERR_CONFIG", -2: "FSQR_ERR_DATA",
          -3: "FSQR_ERR_NUMERIC", -4: "FSQR_ERR_CUDA", -5: "FSQR_ERR_OOM", -6: "FSQR_ERR_STATE"}


class FsqrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


DESIGN_PACK2 = 1   # fsqr_design.flags: repack U8 codes to 2-bit at create


class fsqr_design(ctypes.Structure):
    _fields_ = [("storage", ctypes.c_int32), ("flags", ctypes.c_int32), ("n", ctypes.c_int64),
                ("p", ctypes.c_int64), ("data_dev", ctypes.c_void_p), ("ld", ctypes.c_int64),
                ("mean_dev", ctypes.c_void_p), ("scale_dev", ctypes.c_void_p)]


class fsqr_options(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int32), ("backend", ctypes.c_int32), ("mu", ctypes.c_double),
                ("eta_safety", ctypes.c_double), ("eta_host", ctypes.c_void_p), ("tol", ctypes.c_double),
                ("max_iter", ctypes.c_int64), ("power_max_iter", ctypes.c_int32), ("trace_cap", ctypes.c_int32),
                ("power_tol", ctypes.c_double), ("seed", ctypes.c_uint64), ("max_iter_point", ctypes.c_int64),
                ("eta_method", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class fsqr_tune_options(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("pad_", ctypes.c_int32), ("lam_min_frac", ctypes.c_double),
                ("B", ctypes.c_int64), ("seed", ctypes.c_uint64), ("alpha", ctypes.c_double), ("c", ctypes.c_double)]


class fsqr_result(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("total_iterations", ctypes.c_int64), ("n_rhs", ctypes.c_int32),
                ("status", ctypes.c_int32 * 16), ("R", (ctypes.c_double * 3) * 16),
                ("objective", ctypes.c_double * 16), ("wall_ms", ctypes.c_double)]


EXPORTS = ["fsqr_default_options", "fsqr_create", "fsqr_iterate", "fsqr_solve", "fsqr_objective", "fsqr_kkt",
           "fsqr_get_beta", "fsqr_get_state", "fsqr_set_state", "fsqr_set_lambda", "fsqr_lambda_max",
           "fsqr_get_eta", "fsqr_get_colstats", "fsqr_path", "fsqr_path_beta", "fsqr_trace", "fsqr_iterations",
           "fsqr_profile_iterate", "fsqr_hbic", "fsqr_set_lambda_weights", "fsqr_lla", "fsqr_pivotal", "fsqr_set_lambda2", "fsqr_path_hbic",
           "fsqr_tune", "fsqr_set_tolerance", "fsqr_launches_per_iteration", "fsqr_debug_stamps", "fsqr_backend_name", "fsqr_fit_host", "fsqr_pack2", "fsqr_last_error", "fsqr_global_error", "fsqr_status_str",
           "fsqr_destroy"]


def lib_path() -> str:
    return os.environ.get("FSQR_LIB", _build.LIB)   # FSQR_LIB: an alternative build, for measurements


def load(build_if_missing: bool = True):
    """Load libfsqr.so (building it with nvcc when stale).  Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        try:
            _build.build()
        except (OSError, FileNotFoundError) as e:  # no nvcc on this box: use the shipped .so if present
            if not os.path.exists(_build.LIB):
                raise RuntimeError(f"libfsqr.so missing and cannot be built: {e}") from e
    if not os.path.exists(_build.LIB):
        raise RuntimeError("libfsqr.so is missing: run paper_2601_02826_b200._build.build()")
    L = ctypes.CDLL(lib_path())
    P, I32, I64, D, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    ctxp = ctypes.c_void_p
    L.fsqr_default_options.argtypes = [ctypes.POINTER(fsqr_options)]
    L.fsqr_default_options.restype = None
    L.fsqr_create.argtypes = [ctypes.POINTER(fsqr_design), P, I32, P, P, P, ctypes.POINTER(fsqr_options), P,
                              ctypes.POINTER(ctxp)]
    L.fsqr_iterate.argtypes = [ctxp, I64, P]
    L.fsqr_solve.argtypes = [ctxp, ctypes.POINTER(fsqr_result), P]
    L.fsqr_objective.argtypes = [ctxp, P, P]
    L.fsqr_kkt.argtypes = [ctxp, P, P]
    L.fsqr_get_beta.argtypes = [ctxp, P, I32, P]
    L.fsqr_get_state.argtypes = [ctxp, P, P, P, P]
    L.fsqr_set_state.argtypes = [ctxp, P, P, P, P]
    L.fsqr_set_lambda.argtypes = [ctxp, P]
    L.fsqr_lambda_max.argtypes = [ctxp, P]
    L.fsqr_get_eta.argtypes = [ctxp, P]
    L.fsqr_get_colstats.argtypes = [ctxp, P, P]
    L.fsqr_path.argtypes = [ctxp, P, I32, P, P, P, P, P, P, P]
    L.fsqr_path_beta.argtypes = [ctxp, I32, I32, I64, P, P, P]
    L.fsqr_trace.argtypes = [ctxp, P, I64, P]
    L.fsqr_profile_iterate.argtypes = [ctxp, I64, P, P, P]
    L.fsqr_profile_iterate.restype = S
    L.fsqr_hbic.argtypes = [ctxp, P, P]
    L.fsqr_set_lambda2.argtypes = [ctxp, P]
    L.fsqr_path_hbic.argtypes = [ctxp, P]
    L.fsqr_tune.argtypes = [ctxp, ctypes.POINTER(fsqr_tune_options), P, P, P, P, P, P]
    L.fsqr_pivotal.argtypes = [ctxp, I32, I64, ctypes.c_uint64, P, P]
    L.fsqr_set_lambda_weights.argtypes = [ctxp, P, P]
    L.fsqr_lla.argtypes = [ctxp, I32, D, I32, P, ctypes.POINTER(fsqr_result), P]
    L.fsqr_set_tolerance.argtypes = [ctxp, D, I64]
    L.fsqr_debug_stamps.argtypes = [ctxp, P, I64]
    L.fsqr_launches_per_iteration.argtypes = [ctxp]
    L.fsqr_launches_per_iteration.restype = I32
    L.fsqr_iterations.argtypes = [ctxp]
    L.fsqr_iterations.restype = I64
    L.fsqr_backend_name.argtypes = [ctxp]
    L.fsqr_backend_name.restype = ctypes.c_char_p
    L.fsqr_fit_host.argtypes = [ctypes.POINTER(fsqr_design), P, I32, P, P, ctypes.POINTER(fsqr_options), I64, P,
                                ctypes.POINTER(fsqr_result), P]
    L.fsqr_pack2.argtypes = [P, I64, I64, I64, P, I64, P]
    L.fsqr_last_error.argtypes = [ctxp]
    L.fsqr_last_error.restype = ctypes.c_char_p
    L.fsqr_global_error.argtypes = []
    L.fsqr_global_error.restype = ctypes.c_char_p
    L.fsqr_status_str.argtypes = [S]
    L.fsqr_status_str.restype = ctypes.c_char_p
    L.fsqr_destroy.argtypes = [ctxp]
    L.fsqr_destroy.restype = None
    for name in ("fsqr_create", "fsqr_iterate", "fsqr_solve", "fsqr_objective", "fsqr_kkt", "fsqr_get_beta",
                 "fsqr_get_state", "fsqr_set_state", "fsqr_set_lambda", "fsqr_lambda_max", "fsqr_get_eta",
                 "fsqr_get_colstats", "fsqr_path", "fsqr_path_beta", "fsqr_trace", "fsqr_fit_host", "fsqr_hbic",
                 "fsqr_set_lambda_weights", "fsqr_lla", "fsqr_pivotal", "fsqr_set_lambda2", "fsqr_path_hbic", "fsqr_pack2",
                 "fsqr_tune", "fsqr_set_tolerance", "fsqr_debug_stamps"):
        getattr(L, name).restype = S
    _lib = L
    return L


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(int(a.data_ptr()))  # torch tensor


def _stream(stream):
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(st: int, ctx=None):
    if st < 0:
        L = load()
        msg = (L.fsqr_last_error(ctx) if ctx else L.fsqr_global_error()) or b""
        raise FsqrError(st, msg.decode())
    return st


def default_options(**kw) -> fsqr_options:
    o = fsqr_options()
    load().fsqr_default_options(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


# ------------------------------------------------------------------ C-ABI mirrors

def fsqr_create(X, storage: int, n: int, p: int, ld: int, y, taus, lambdas, lambda_w=None, opt=None, stream=None,
                eta=None, mean=None, scale=None, flags: int = 0):
    """X, y, lambda_w, mean, scale: CUDA tensors (borrowed X); taus, lambdas: sequences; returns ctx handle."""
    L = load()
    d = fsqr_design(storage, flags, n, p, _ptr(X).value, ld, _ptr(mean).value if mean is not None else None,
                    _ptr(scale).value if scale is not None else None)
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    lambdas = np.ascontiguousarray(lambdas, dtype=np.float64)
    o = opt if opt is not None else default_options()
    eta_arr = None
    if eta is not None:
        eta_arr = np.ascontiguousarray(eta, dtype=np.float64)
        o.eta_host = eta_arr.ctypes.data
    ctx = ctypes.c_void_p()
    st = L.fsqr_create(ctypes.byref(d), _ptr(y), len(taus), _ptr(taus), _ptr(lambdas), _ptr(lambda_w),
                       ctypes.byref(o), _stream(stream), ctypes.byref(ctx))
    _check(st)
    return ctx


def fsqr_iterate(ctx, k: int, stream=None):
    return _check(load().fsqr_iterate(ctx, int(k), _stream(stream)), ctx)


def fsqr_solve(ctx, stream=None) -> dict:
    r = fsqr_result()
    st = _check(load().fsqr_solve(ctx, ctypes.byref(r), _stream(stream)), ctx)
    R = r.n_rhs
    return dict(status=st, iterations=r.iterations, total_iterations=r.total_iterations,
                rhs_status=[r.status[i] for i in range(R)],
                R=np.array([[r.R[i][q] for q in range(3)] for i in range(R)]),
                objective=np.array([r.objective[i] for i in range(R)]), wall_ms=r.wall_ms)


def fsqr_objective(ctx, n_rhs: int, stream=None) -> np.ndarray:
    out = np.empty(n_rhs)
    _check(load().fsqr_objective(ctx, _ptr(out), _stream(stream)), ctx)
    return out


def fsqr_kkt(ctx, n_rhs: int, stream=None) -> np.ndarray:
    out = np.empty((n_rhs, 3))
    _check(load().fsqr_kkt(ctx, _ptr(out), _stream(stream)), ctx)
    return out


def fsqr_get_beta(ctx, n_rhs: int, p: int, scale: int = 0, stream=None) -> np.ndarray:
    out = np.empty((n_rhs, p + 1))
    _check(load().fsqr_get_beta(ctx, _ptr(out), int(scale), _stream(stream)), ctx)
    return out


def fsqr_get_state(ctx, n_rhs: int, n: int, p: int, stream=None):
    b, z, t = np.empty((n_rhs, p + 1)), np.empty((n_rhs, n)), np.empty((n_rhs, n))
    _check(load().fsqr_get_state(ctx, _ptr(b), _ptr(z), _ptr(t), _stream(stream)), ctx)
    return b, z, t


def fsqr_set_state(ctx, beta, z, theta, stream=None):
    b, zz, tt = (np.ascontiguousarray(a, dtype=np.float64) for a in (beta, z, theta))
    return _check(load().fsqr_set_state(ctx, _ptr(b), _ptr(zz), _ptr(tt), _stream(stream)), ctx)


def fsqr_set_lambda(ctx, lambdas):
    lam = np.ascontiguousarray(lambdas, dtype=np.float64)
    return _check(load().fsqr_set_lambda(ctx, _ptr(lam)), ctx)


def fsqr_lambda_max(ctx, n_rhs: int) -> np.ndarray:
    out = np.empty(n_rhs)
    _check(load().fsqr_lambda_max(ctx, _ptr(out)), ctx)
    return out


def fsqr_get_eta(ctx, G: int) -> np.ndarray:
    out = np.empty(G)
    _check(load().fsqr_get_eta(ctx, _ptr(out)), ctx)
    return out


def fsqr_get_colstats(ctx, p: int):
    m, s = np.empty(p), np.empty(p)
    _check(load().fsqr_get_colstats(ctx, _ptr(m), _ptr(s)), ctx)
    return m, s


def fsqr_path(ctx, lam_path, stream=None) -> dict:
    lp = np.ascontiguousarray(lam_path, dtype=np.float64)
    R, T = lp.shape
    total = ctypes.c_int64(0)
    it = np.zeros((R, T), dtype=np.int64)
    obj = np.zeros((R, T))
    RR = np.zeros((R, T, 3))
    nnz = np.zeros((R, T), dtype=np.int64)
    conv = np.zeros((R, T), dtype=np.int32)
    _check(load().fsqr_path(ctx, _ptr(lp), T, ctypes.byref(total), _ptr(it), _ptr(obj), _ptr(RR), _ptr(nnz),
                            _ptr(conv), _stream(stream)), ctx)
    return dict(total=total.value, iters=it, obj=obj, R=RR, nnz=nnz, converged=conv.astype(bool))


def fsqr_path_hbic(ctx, n_rhs: int, T: int) -> np.ndarray:
    out = np.empty((n_rhs, T))
    _check(load().fsqr_path_hbic(ctx, _ptr(out)), ctx)
    return out


def fsqr_tune(ctx, n_rhs: int, T: int = 50, lam_min_frac: float = 0.01, B: int = 0, seed: int = 0x5EED,
              alpha: float = 0.1, c: float = 1.1, stream=None) -> dict:
    """The tuning protocol (L406-412) in one C-ABI call: grid, warm-started path, HBIC, argmin."""
    o = fsqr_tune_options(int(T), 0, float(lam_min_frac), int(B), int(seed) & 0xFFFFFFFFFFFFFFFF, float(alpha),
                          float(c))
    grid, h = np.zeros((n_rhs, T)), np.zeros((n_rhs, T))
    best = np.zeros(n_rhs, dtype=np.int32)
    piv = np.zeros(n_rhs)
    total = ctypes.c_int64(0)
    _check(load().fsqr_tune(ctx, ctypes.byref(o), _ptr(grid), _ptr(h), _ptr(best), _ptr(piv), ctypes.byref(total),
                            _stream(stream)), ctx)
    return dict(grid=grid, hbic=h, best=best.astype(np.int64), lam_piv=piv, total=total.value)


def fsqr_path_beta(ctx, r: int, t: int, p: int) -> np.ndarray:
    """Dense standardised beta (length p+1) of path point t of RHS r."""
    cap = p + 1
    idx = np.zeros(cap, dtype=np.int64)
    val = np.zeros(cap)
    cnt = ctypes.c_int64(0)
    _check(load().fsqr_path_beta(ctx, r, t, cap, _ptr(idx), _ptr(val), ctypes.byref(cnt)), ctx)
    out = np.zeros(p + 1)
    m = min(cnt.value, cap)
    out[idx[:m]] = val[:m]
    return out


def fsqr_trace(ctx, n_rhs: int, cap_rows: int) -> np.ndarray:
    out = np.zeros((cap_rows, n_rhs, 5))
    rows = ctypes.c_int64(0)
    _check(load().fsqr_trace(ctx, _ptr(out), cap_rows, ctypes.byref(rows)), ctx)
    return out[: rows.value]


def fsqr_profile_iterate(ctx, k: int, stream=None):
    """k iterations as individual launches with CUDA events per stage: (stage_ms[3], total_ms)."""
    st = np.zeros(3)
    tot = ctypes.c_double(0.0)
    _check(load().fsqr_profile_iterate(ctx, int(k), _ptr(st), ctypes.byref(tot), _stream(stream)), ctx)
    return st, tot.value


def fsqr_hbic(ctx, n_rhs: int, stream=None) -> np.ndarray:
    out = np.empty(n_rhs)
    _check(load().fsqr_hbic(ctx, _ptr(out), _stream(stream)), ctx)
    return out


def fsqr_set_lambda2(ctx, lam2):
    v = np.ascontiguousarray(lam2, dtype=np.float64)
    return _check(load().fsqr_set_lambda2(ctx, _ptr(v)), ctx)


def fsqr_set_lambda_weights(ctx, weights=None, stream=None):
    """weights: [n_rhs, p+1] (or None for unit weights)."""
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    return _check(load().fsqr_set_lambda_weights(ctx, _ptr(w), _stream(stream)), ctx)


def fsqr_lla(ctx, penalty: int, a: float, L: int, stream=None) -> dict:
    it = np.zeros(L + 1, dtype=np.int64)
    r = fsqr_result()
    st = _check(load().fsqr_lla(ctx, int(penalty), float(a), int(L), _ptr(it), ctypes.byref(r), _stream(stream)), ctx)
    R = r.n_rhs
    return dict(status=st, stage_iters=it, rhs_status=[r.status[i] for i in range(R)],
                R=np.array([[r.R[i][q] for q in range(3)] for i in range(R)]),
                objective=np.array([r.objective[i] for i in range(R)]))


def fsqr_pivotal(ctx, rhs: int, B: int, seed: int = 0x5EED, stream=None) -> np.ndarray:
    out = np.empty(int(B))
    _check(load().fsqr_pivotal(ctx, int(rhs), int(B), ctypes.c_uint64(int(seed)), _ptr(out), _stream(stream)), ctx)
    return out


def fsqr_set_tolerance(ctx, tol: float, max_iter: int):
    return _check(load().fsqr_set_tolerance(ctx, float(tol), int(max_iter)), ctx)


def fsqr_debug_stamps(ctx, n: int = 2048) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    _check(load().fsqr_debug_stamps(ctx, _ptr(out), n), ctx)
    return out


def fsqr_launches_per_iteration(ctx) -> int:
    return int(load().fsqr_launches_per_iteration(ctx))


def fsqr_iterations(ctx) -> int:
    return int(load().fsqr_iterations(ctx))


def fsqr_backend_name(ctx) -> str:
    return load().fsqr_backend_name(ctx).decode()


def fsqr_fit_host(X: np.ndarray, storage: int, n: int, p: int, ld: int, y: np.ndarray, taus, lambdas, iters: int,
                  opt=None, stream=None, eta=None, flags: int = 0) -> tuple:
    """End-to-end call with HOST buffers (X should be pinned for speed); returns (beta [R, p+1], result dict)."""
    L = load()
    d = fsqr_design(storage, flags, n, p, _ptr(X).value, ld, None, None)
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    lambdas = np.ascontiguousarray(lambdas, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float64)
    o = opt if opt is not None else default_options()
    eta_arr = None
    if eta is not None:
        eta_arr = np.ascontiguousarray(eta, dtype=np.float64)
        o.eta_host = eta_arr.ctypes.data
    beta = np.empty((len(taus), p + 1))
    r = fsqr_result()
    st = L.fsqr_fit_host(ctypes.byref(d), _ptr(yy), len(taus), _ptr(taus), _ptr(lambdas), ctypes.byref(o),
                         int(iters), _ptr(beta), ctypes.byref(r), _stream(stream))
    _check(st)
    return beta, dict(status=st, iterations=r.iterations)


def fsqr_pack2(X8, ld8: int, n: int, p: int, X2=None, stream=None):
    """Repack u8 codes (CUDA tensor [p, ld8]) into PACKED2 layout; returns (X2 [p, ld2] uint8 tensor, ld2)."""
    import torch

    ld2 = leading_dim_packed2(n)
    if X2 is None:
        X2 = torch.empty((p, ld2), dtype=torch.uint8, device=X8.device)
    _check(load().fsqr_pack2(_ptr(X8), int(ld8), int(n), int(p), _ptr(X2), int(ld2), _stream(stream)))
    return X2, ld2


def leading_dim_packed2(n: int) -> int:
    return (((n + 3) // 4 + 15) // 16) * 16


def fsqr_destroy(ctx):
    load().fsqr_destroy(ctx)


class Solver:
    """Holds a context plus the borrowed design tensor (kept alive for the ctx lifetime)."""

    def __init__(self, X, storage: int, n: int, p: int, ld: int, y, taus, lambdas, G: int = 5, mu: float = 0.0,
                 tol: float = 1e-6, max_iter: int = 100000, backend: int = BACKEND_AUTO, eta=None, lambda_w=None,
                 max_iter_point: int = 10000, stream=None, flags: int = 0, **kw):
        import torch

        self.X = X
        self.y = y if isinstance(y, torch.Tensor) else torch.as_tensor(np.asarray(y, np.float64), device="cuda")
        self.lambda_w = lambda_w
        self.n, self.p, self.R, self.G = int(n), int(p), len(taus), int(G)
        self.max_iter = int(max_iter)
        self.taus = list(taus)
        opt = default_options(G=G, mu=mu, tol=tol, max_iter=max_iter, backend=backend,
                              max_iter_point=max_iter_point, **kw)
        self.ctx = fsqr_create(X, storage, n, p, ld, self.y, taus, lambdas, lambda_w, opt, stream, eta=eta,
                               flags=flags)

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib is not None:
            _lib.fsqr_destroy(ctx)
            self.ctx = None

    def iterate(self, k: int, stream=None):
        return fsqr_iterate(self.ctx, k, stream)

    def solve(self, stream=None):
        return fsqr_solve(self.ctx, stream)

    def objective(self):
        return fsqr_objective(self.ctx, self.R)

    def kkt(self):
        return fsqr_kkt(self.ctx, self.R)

    def beta(self, scale: int = 0):
        return fsqr_get_beta(self.ctx, self.R, self.p, scale)

    def state(self):
        return fsqr_get_state(self.ctx, self.R, self.n, self.p)

    def set_state(self, beta, z, theta):
        return fsqr_set_state(self.ctx, beta, z, theta)

    def set_lambda(self, lambdas):
        return fsqr_set_lambda(self.ctx, lambdas)

    def lambda_max(self):
        return fsqr_lambda_max(self.ctx, self.R)

    def eta(self):
        return fsqr_get_eta(self.ctx, self.G)

    def colstats(self):
        return fsqr_get_colstats(self.ctx, self.p)

    def path(self, lam_path):
        return fsqr_path(self.ctx, lam_path)

    def path_hbic(self, T: int):
        return fsqr_path_hbic(self.ctx, self.R, T)

    def tune(self, T: int = 50, lam_min_frac: float = 0.01, B: int = 0, seed: int = 0x5EED, alpha: float = 0.1,
             c: float = 1.1):
        """fsqr_tune: returns dict(grid, hbic, best, lam_piv, total, beta) where beta
        [n_rhs, p+1] is the HBIC-selected point of each RHS (fsqr_path_beta)."""
        out = fsqr_tune(self.ctx, self.R, T, lam_min_frac, B, seed, alpha, c)
        out["beta"] = np.stack([self.path_beta(r, int(out["best"][r])) for r in range(self.R)])
        return out

    def path_beta(self, r: int, t: int):
        return fsqr_path_beta(self.ctx, r, t, self.p)

    def hbic(self):
        return fsqr_hbic(self.ctx, self.R)

    def set_lambda2(self, lam2):
        return fsqr_set_lambda2(self.ctx, lam2)

    def set_lambda_weights(self, weights=None):
        return fsqr_set_lambda_weights(self.ctx, weights)

    def lla(self, penalty: int, a: float, L: int = 1):
        return fsqr_lla(self.ctx, penalty, a, L)

    def pivotal(self, B: int, seed: int = 0x5EED, rhs: int = 0):
        return fsqr_pivotal(self.ctx, rhs, B, seed)

    def trace(self, rows: int = 4096):
        return fsqr_trace(self.ctx, self.R, rows)

    def set_tol(self, tol: float, max_iter: int | None = None):
        self.max_iter = self.max_iter if max_iter is None else int(max_iter)
        return fsqr_set_tolerance(self.ctx, tol, self.max_iter)

    def launches_per_iteration(self) -> int:
        return fsqr_launches_per_iteration(self.ctx)

    def iterations(self) -> int:
        return fsqr_iterations(self.ctx)

    @property
    def backend(self) -> str:
        return fsqr_backend_name(self.ctx)
