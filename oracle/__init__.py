"""Oracle: plain, slow, obviously-correct fp64 CPU FS-QRPPA (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path in ``paper_2601_02826_b200/``; the two meet only at the seeded inputs
from ``datagen/``.  The arithmetic lives in ``fsqr_oracle.c`` (plain loops,
each function cites the PAPER.md passage it follows); this module only loads
it and marshals numpy arrays.  ``lp.py`` holds the brute-force LP used to pin
the solver on tiny inputs.

Parity status per function (DESIGN.md §4 repeats this table):
  colstats        pinned: numpy mean/std(ddof=1) on small slabs
  backprod/fwd    pinned: numpy X~^T theta / X~ beta on small slabs, partition invariance
  prox_beta/z     pinned: brute-force 1-D minimisation + SPEC worked values
  dual            pinned: SPEC worked values
  power           pinned: numpy.linalg.eigvalsh, identity and rank-one closed forms
  lanczos         pinned: numpy.linalg.eigvalsh (to 1e-9 in a few steps), identity and rank-one (exact in
                  one step), the tridiagonal bisection against eigvalsh of random tridiagonals, and
                  Ritz value <= Lambda_max at every step count
  lambda_max      pinned: textbook null model (beta=0, intercept = sample quantile) just above it
  solve           pinned: LP vertex enumeration + HiGHS (tiny), Prop. 1 certificate, partition
                  invariance, fixed-point property, geometric decay (Corollary 1)
  prox_en / solve(lam2 > 0)  pinned: 1-D brute force of the elastic-net prox; lam2 = 0 bitwise
                  equals E14; converged objective equals an SLSQP solve of the QP form (tiny inputs)
  penalty_deriv   pinned: SPEC worked values (SCAD, MCP), continuity at the knots, the LASSO limit
  lla             pinned: each stage is a weighted-l1 PQR whose optimum matches the LP brute force
                  with the stage's weights; Prop. 1 certificate per stage
  pivotal         pinned: splitmix64 reference outputs, Bernoulli(tau) frequencies of the draws,
                  E[(x~_j^T psi)^2] = tau(1-tau)(n-1) (law of large numbers), invariance to
                  genotype recoding 2-x and to column order; a hand-built 3x2 case
  hbic            pinned: SPEC worked value and the closed form on a null model
  trajectory      pinned: Theorem 1's Fejer monotonicity in the H-norm on every step of 300-step
                  trajectories (the paper prints no iterates); see DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fsqr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, IEEE fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"   # build aside, then rename: a running process keeps its copy
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Design(ctypes.Structure):
    _fields_ = [("storage", ctypes.c_int32), ("pad_", ctypes.c_int32), ("n", ctypes.c_int64),
                ("p", ctypes.c_int64), ("ld", ctypes.c_int64), ("data", ctypes.c_void_p),
                ("mean", ctypes.c_void_p), ("sd", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("mu", ctypes.c_double), ("G", ctypes.c_int32),
                ("check", ctypes.c_int32), ("eta", ctypes.c_void_p), ("lam", ctypes.c_void_p),
                ("max_iter", ctypes.c_int64), ("tol", ctypes.c_double), ("lam2", ctypes.c_double)]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P, D, I64, I32, U64 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        DP = ctypes.POINTER(_Design)
        lib.orc_xt.restype = D
        lib.orc_xt.argtypes = [DP, I64, I64]
        lib.orc_colstats.restype = I64
        lib.orc_colstats.argtypes = [DP, P, P]
        lib.orc_blocks.argtypes = [I64, I32, P]
        lib.orc_backprod.argtypes = [DP, P, P]
        lib.orc_backprod_range.argtypes = [DP, P, I64, I64, P]
        lib.orc_fwdprod.argtypes = [DP, P, P]
        lib.orc_fwdprod_range.argtypes = [DP, P, I64, I64, P]
        lib.orc_prox_beta.restype = D
        lib.orc_prox_beta.argtypes = [D, D, D, D]
        lib.orc_prox_en.restype = D
        lib.orc_prox_en.argtypes = [D, D, D, D, D]
        lib.orc_objective_en.restype = D
        lib.orc_objective_en.argtypes = [DP, P, D, P, D, P]
        lib.orc_prox_z.restype = D
        lib.orc_prox_z.argtypes = [D, D, D, D, I64]
        lib.orc_dual.restype = D
        lib.orc_dual.argtypes = [D, D, D, D, I32]
        lib.orc_rho.restype = D
        lib.orc_rho.argtypes = [D, D]
        lib.orc_kkt_rel.argtypes = [DP, P, D, P, P, P, P, P]
        lib.orc_objective.restype = D
        lib.orc_objective.argtypes = [DP, P, D, P, P]
        lib.orc_kkt_cert.argtypes = [DP, P, D, P, P, P, P, P]
        lib.orc_power_start.restype = D
        lib.orc_power_start.argtypes = [U64, I64]
        lib.orc_power.restype = D
        lib.orc_power.argtypes = [DP, I64, I64, D, I64, U64, P]
        lib.orc_lanczos.restype = D
        lib.orc_lanczos.argtypes = [DP, I64, I64, D, I64, U64, P]
        lib.orc_tridiag_max_eig.restype = D
        lib.orc_tridiag_max_eig.argtypes = [P, P, ctypes.c_int]
        lib.orc_lambda_max.restype = D
        lib.orc_lambda_max.argtypes = [DP, P, D, P]
        lib.orc_solve.restype = ctypes.c_int
        lib.orc_solve.argtypes = [DP, P, ctypes.POINTER(_Opts), P, P, P, P, P, P, P]
        lib.orc_penalty_deriv.restype = D
        lib.orc_penalty_deriv.argtypes = [I32, D, D, D]
        lib.orc_lla_weights.argtypes = [I32, D, D, P, I64, P]
        lib.orc_hbic_value.restype = D
        lib.orc_hbic_value.argtypes = [D, I64, I64, I64]
        lib.orc_hbic.restype = D
        lib.orc_hbic.argtypes = [DP, P, D, P]
        lib.orc_piv_uniform.restype = D
        lib.orc_piv_uniform.argtypes = [U64, I64, I64]
        lib.orc_splitmix.restype = U64
        lib.orc_splitmix.argtypes = [U64]
        lib.orc_pivotal.argtypes = [DP, D, I64, U64, P]
        lib.orc_path.restype = I64
        lib.orc_path.argtypes = [DP, P, D, D, I32, P, P, P, I32, D, I64, P, P, P, P, P, P, P, P]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Design:
    """A stored design (same bytes the GPU reads) plus its column statistics.

    storage: 0 fp32 dense, 1 uint8 {0,1,2}, 2 2-bit packed.  X is [p, ld] column-major.
    """

    def __init__(self, storage: int, n: int, p: int, ld: int, X: np.ndarray, mean=None, sd=None):
        self.storage, self.n, self.p, self.ld = int(storage), int(n), int(p), int(ld)
        self.X = np.ascontiguousarray(X)
        self._st = _Design(self.storage, 0, self.n, self.p, self.ld, _p(self.X), None, None)
        if mean is None:
            self.mean = np.empty(self.p)
            self.sd = np.empty(self.p)
            self._st.mean, self._st.sd = _p(self.mean), _p(self.sd)
            bad = _load().orc_colstats(ctypes.byref(self._st), _p(self.mean), _p(self.sd))
            if bad != 0:
                raise ValueError(f"zero-variance column {-bad - 1}")
        else:
            self.mean, self.sd = _f64(mean), _f64(sd)
        self._st.mean, self._st.sd = _p(self.mean), _p(self.sd)

    @classmethod
    def from_problem(cls, prob) -> "Design":
        return cls(prob.storage, prob.n, prob.p, prob.ld, prob.X)

    @property
    def ref(self):
        return ctypes.byref(self._st)

    def xt(self, j: int, i: int) -> float:
        return _load().orc_xt(self.ref, j, i)

    def dense(self) -> np.ndarray:
        """X~ as an n x (p+1) fp64 matrix (small designs only; built from orc_xt)."""
        out = np.empty((self.n, self.p + 1))
        lib = _load()
        for j in range(self.p + 1):
            for i in range(self.n):
                out[i, j] = lib.orc_xt(self.ref, j, i)
        return out


def blocks(ncols: int, G: int) -> np.ndarray:
    start = np.empty(G + 1, dtype=np.int64)
    _load().orc_blocks(ncols, G, _p(start))
    return start


def backprod(d: Design, theta, j0: int = 0, j1: int | None = None) -> np.ndarray:
    j1 = d.p + 1 if j1 is None else j1
    theta = _f64(theta)
    g = np.empty(j1 - j0)
    _load().orc_backprod_range(d.ref, _p(theta), j0, j1, _p(g))
    return g


def fwdprod(d: Design, beta, j0: int = 0, j1: int | None = None) -> np.ndarray:
    j1 = d.p + 1 if j1 is None else j1
    beta = _f64(beta)
    s = np.empty(d.n)
    _load().orc_fwdprod_range(d.ref, _p(beta), j0, j1, _p(s))
    return s


def prox_beta(beta, g, lam, eta) -> float:
    return _load().orc_prox_beta(beta, g, lam, eta)


def prox_en(beta, g, lam1, lam2, eta) -> float:
    """Elastic-net block prox (Remark 3, L347-349; reading R19)."""
    return _load().orc_prox_en(beta, g, lam1, lam2, eta)


def objective_en(d: Design, y, tau, lam_vec, lam2: float, beta) -> float:
    return _load().orc_objective_en(d.ref, _p(_f64(y)), tau, _p(_f64(lam_vec)), float(lam2), _p(_f64(beta)))


def prox_z(z, theta, mu, tau, n) -> float:
    return _load().orc_prox_z(z, theta, mu, tau, n)


def dual(theta, r_new, r_old, mu, G) -> float:
    return _load().orc_dual(theta, r_new, r_old, mu, G)


def rho(u, tau) -> float:
    return _load().orc_rho(u, tau)


def power_start(seed: int, j: int) -> float:
    return _load().orc_power_start(seed, j)


def power(d: Design, j0: int, j1: int, tol: float = 1e-4, maxit: int = 1000, seed: int = 0x5EED):
    it = ctypes.c_int64(0)
    lam = _load().orc_power(d.ref, j0, j1, tol, maxit, seed, ctypes.byref(it))
    return lam, int(it.value)


def lanczos(d: Design, j0: int, j1: int, tol: float = 1e-4, maxit: int = 1000, seed: int = 0x5EED):
    it = ctypes.c_int64(0)
    lam = _load().orc_lanczos(d.ref, j0, j1, tol, maxit, seed, ctypes.byref(it))
    return lam, int(it.value)


def tridiag_max_eig(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return _load().orc_tridiag_max_eig(_p(a), _p(b if len(b) else np.zeros(1)), len(a))


def eta(d: Design, G: int, mu: float, safety: float = 1.05, tol: float = 1e-4, maxit: int = 1000,
        seed: int = 0x5EED, method: str = "power") -> np.ndarray:
    """eta_g = safety * mu * Lambda_hat(X~_g^T X~_g) (L259), Lambda_hat by the power
    method or by Lanczos (both named at L259)."""
    st = blocks(d.p + 1, G)
    fn = power if method == "power" else lanczos
    return np.array([safety * mu * fn(d, int(st[g]), int(st[g + 1]), tol, maxit, seed)[0] for g in range(G)])


def lambda_max(d: Design, y, tau: float):
    y = _f64(y)
    q = ctypes.c_double(0.0)
    lm = _load().orc_lambda_max(d.ref, _p(y), tau, ctypes.byref(q))
    return lm, q.value


def lam_vector(p: int, lam: float, weights=None) -> np.ndarray:
    v = np.full(p + 1, float(lam)) if weights is None else float(lam) * _f64(weights).copy()
    v[0] = 0.0
    return v


def kkt_rel(d: Design, y, tau, lam_vec, beta, z, theta) -> np.ndarray:
    R = np.empty(3)
    _load().orc_kkt_rel(d.ref, _p(_f64(y)), tau, _p(_f64(lam_vec)), _p(_f64(beta)), _p(_f64(z)),
                        _p(_f64(theta)), _p(R))
    return R


def kkt_cert(d: Design, y, tau, lam_vec, beta, z, theta) -> np.ndarray:
    out = np.empty(3)
    _load().orc_kkt_cert(d.ref, _p(_f64(y)), tau, _p(_f64(lam_vec)), _p(_f64(beta)), _p(_f64(z)),
                         _p(_f64(theta)), _p(out))
    return out


def objective(d: Design, y, tau, lam_vec, beta) -> float:
    return _load().orc_objective(d.ref, _p(_f64(y)), tau, _p(_f64(lam_vec)), _p(_f64(beta)))


def solve(d: Design, y, tau: float, lam_vec, eta_vec, mu: float, G: int, max_iter: int = 1000,
          tol: float = 1e-6, check: bool = True, state=None, trace: bool = False, lam2: float = 0.0) -> dict:
    """Algorithm 1 from (beta, z, theta) = state or the cold start (0, y, 0)."""
    y = _f64(y)
    lam_vec, eta_vec = _f64(lam_vec), _f64(eta_vec)
    if state is None:
        beta, z, theta = np.zeros(d.p + 1), y.copy(), np.zeros(d.n)
    else:
        beta, z, theta = (_f64(a).copy() for a in state)
    o = _Opts(tau, mu, G, 1 if check else 0, _p(eta_vec), _p(lam_vec), int(max_iter), tol, float(lam2))
    it = ctypes.c_int64(0)
    R = np.empty(3)
    obj = ctypes.c_double(0.0)
    tr = np.zeros((max_iter + 1, 5)) if trace else None
    st = _load().orc_solve(d.ref, _p(y), ctypes.byref(o), _p(beta), _p(z), _p(theta), ctypes.byref(it), _p(R),
                           ctypes.byref(obj), _p(tr))
    out = dict(status=st, iters=int(it.value), beta=beta, z=z, theta=theta, R=R, obj=obj.value)
    if trace:
        out["trace"] = tr[: out["iters"] + 1]
    return out


def path(d: Design, y, tau: float, lam_path, eta_vec, mu: float, G: int, tol: float, max_iter_point: int,
         weights=None, state=None, keep_beta: bool = True) -> dict:
    y = _f64(y)
    lam_path = _f64(lam_path)
    T = len(lam_path)
    w = np.ones(d.p + 1) if weights is None else _f64(weights).copy()
    w[0] = 0.0
    if state is None:
        beta, z, theta = np.zeros(d.p + 1), y.copy(), np.zeros(d.n)
    else:
        beta, z, theta = (_f64(a).copy() for a in state)
    iters = np.zeros(T, dtype=np.int64)
    R = np.zeros((T, 3))
    obj = np.zeros(T)
    conv = np.zeros(T, dtype=np.int32)
    bp = np.zeros((T, d.p + 1)) if keep_beta else None
    total = _load().orc_path(d.ref, _p(y), tau, mu, G, _p(_f64(eta_vec)), _p(w), _p(lam_path), T, tol,
                             int(max_iter_point), _p(beta), _p(z), _p(theta), _p(iters), _p(R), _p(obj), _p(bp),
                             _p(conv))
    return dict(total=int(total), iters=iters, R=R, obj=obj, converged=conv.astype(bool), beta_path=bp,
                beta=beta, z=z, theta=theta)


SCAD, MCP = 1, 2


def penalty_deriv(kind: int, a: float, lam: float, b: float) -> float:
    """p'_lambda(|b|): SCAD (E16, L354-361) or MCP (E17, L363-369)."""
    return _load().orc_penalty_deriv(int(kind), float(a), float(lam), float(b))


def lla_weights(kind: int, a: float, lam: float, beta) -> np.ndarray:
    """w_j = p'_lambda(|beta_j|)/lambda for j >= 1, w_0 = 0 (Algorithm 2)."""
    beta = _f64(beta)
    w = np.empty_like(beta)
    _load().orc_lla_weights(int(kind), float(a), float(lam), _p(beta), len(beta), _p(w))
    return w


def lla(d: Design, y, tau: float, lam: float, kind: int, a: float, L: int, eta_vec, mu: float, G: int,
        tol: float = 1e-6, max_iter: int = 100000) -> dict:
    """Algorithm 2: the LASSO fit with lambda_j = lambda, then L reweighted
    l1 fits, each warm-started from the previous (beta~, z~, theta~) with
    lambda~_j = p'_lambda(|beta~_j|)."""
    stages = []
    w = np.ones(d.p + 1)
    w[0] = 0.0
    state = None
    for l in range(L + 1):
        out = solve(d, y, tau, lam_vector(d.p, lam, w), eta_vec, mu, G, max_iter=max_iter, tol=tol, state=state)
        stages.append(dict(weights=w.copy(), beta=out["beta"].copy(), iters=out["iters"], obj=out["obj"],
                           status=out["status"]))
        state = (out["beta"], out["z"], out["theta"])
        w = lla_weights(kind, a, lam, out["beta"])
    return dict(stages=stages, beta=stages[-1]["beta"], z=state[1], theta=state[2])


def hbic_value(loss: float, active: int, n: int, p: int) -> float:
    return _load().orc_hbic_value(float(loss), int(active), int(n), int(p))


def hbic(d: Design, y, tau: float, beta) -> float:
    """HBIC (E18, L408-411) with C_n = log p."""
    return _load().orc_hbic(d.ref, _p(_f64(y)), float(tau), _p(_f64(beta)))


def splitmix(x: int) -> int:
    """One splitmix64 output for state x (x + golden gamma, then the finaliser)."""
    return int(_load().orc_splitmix(int(x) & 0xFFFFFFFFFFFFFFFF))


def piv_uniform(seed: int, b: int, i: int) -> float:
    return _load().orc_piv_uniform(int(seed), int(b), int(i))


def pivotal(d: Design, tau: float, B: int, seed: int = 0x5EED) -> np.ndarray:
    """Lambda_b = max_j |sum_i x~_ij (tau - 1{U_ib <= tau})| / n, b < B (L412, reading R18)."""
    out = np.empty(int(B))
    _load().orc_pivotal(d.ref, float(tau), int(B), int(seed), _p(out))
    return out


def pivotal_lambda(Lambda, alpha: float = 0.1, c: float = 1.1) -> float:
    """c times the (1-alpha) empirical quantile (order statistic ceil((1-alpha) B)) of Lambda_b."""
    s = np.sort(np.asarray(Lambda, np.float64))
    k = int(np.ceil((1.0 - alpha) * len(s)))
    return float(c * s[max(k, 1) - 1])
