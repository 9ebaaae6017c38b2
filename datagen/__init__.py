"""Seeded synthetic workloads for the FS-QRPPA hot path (shared input infrastructure).

Both the oracle (``oracle/``) and the CUDA path consume what this module
produces; it contains none of the method's arithmetic (see datagen.c header).
Recipes follow BASELINE.json ``configs`` / SURVEY.md §8(d); DESIGN.md §3 restates
them.  Every config can be instantiated at reduced (n, p) for tests while
keeping its recipe (storage, MAF law, effect law, noise law, tau, lambda
fraction, G).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "datagen.c")
_LIB = os.path.join(_HERE, "libdatagen.so")
_lib = None

BASE_SEED = 2601028260

STORAGE_F32, STORAGE_U8, STORAGE_P2 = 0, 1, 2
STORAGE_NAMES = {STORAGE_F32: "f32", STORAGE_U8: "u8", STORAGE_P2: "p2"}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P, I64, U64, D, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        lib.dg_u64.restype = U64
        lib.dg_u64.argtypes = [U64, U64, U64]
        lib.dg_unif.restype = D
        lib.dg_unif.argtypes = [U64, U64, U64]
        lib.dg_normal.restype = D
        lib.dg_normal.argtypes = [U64, U64, U64]
        lib.dg_probit.restype = D
        lib.dg_probit.argtypes = [D]
        lib.dg_causal.argtypes = [U64, I64, I64, P]
        lib.dg_maf.argtypes = [U64, I64, D, D, P]
        lib.dg_genotypes.argtypes = [U64, I64, I64, P, INT, I64, P]
        lib.dg_genotypes_ld.argtypes = [U64, I64, I64, P, D, I64, INT, I64, P]
        lib.dg_gauss_f32.argtypes = [U64, I64, I64, I64, P]
        lib.dg_linpred.argtypes = [INT, I64, P, I64, P, I64, P, P, P]
        lib.dg_effects.argtypes = [U64, U64, I64, INT, D, D, P]
        lib.dg_noise.argtypes = [U64, I64, INT, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def round_up(a: int, b: int) -> int:
    return (a + b - 1) // b * b


def leading_dim(storage: int, n: int) -> int:
    """Column stride: bytes for u8 / 2-bit, floats for f32 (SURVEY §8(d) padding)."""
    if storage == STORAGE_U8:
        return round_up(n, 16)
    if storage == STORAGE_P2:
        return round_up((n + 3) // 4, 16)
    return round_up(n, 4)


@dataclass
class Problem:
    name: str
    storage: int
    n: int
    p: int
    ld: int
    X: np.ndarray            # [p, ld] uint8 or float32, column-major design (data column c = model j-1)
    y: np.ndarray            # [n] float64
    taus: list
    lam_frac: float          # lambda = lam_frac * lambda_max(tau)
    G: int
    causal: np.ndarray       # data-column indices of the causal SNPs
    effects: np.ndarray
    maf: np.ndarray | None
    path_points: int = 1     # >1: geometric lambda path from lambda_max to lam_min_frac*lambda_max
    lam_min_frac: float = 0.01
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def nbytes(self) -> int:
        return int(self.X.nbytes)


# name -> (index, recipe)
CONFIGS = {
    "c1": dict(idx=0, storage=STORAGE_F32, n=200, p=2000, design="gauss", k=10, effect=("unif", 0.5, 2.0),
               noise=1, taus=[0.5], lam=0.1, G=5),
    "c2": dict(idx=1, storage=STORAGE_U8, n=2000, p=50000, design="binom", maf=(0.05, 0.5), k=50,
               effect=("norm", 0.3), noise=0, taus=[0.1, 0.5, 0.9], lam=0.05, G=5),
    "c3": dict(idx=2, storage=STORAGE_U8, n=10000, p=500000, design="binom", maf=(0.01, 0.5), k=100,
               effect=("norm", 0.2), noise=0, hetero=(20, 0.2, 0.5), taus=[0.9], lam=0.02, G=48),
    "c4": dict(idx=3, storage=STORAGE_P2, n=20000, p=2000000, design="ld", maf=(0.01, 0.5), rho=0.6, blk=100,
               k=200, effect=("norm", 0.1), noise=2, taus=[0.5], lam=0.02, G=48),
    "c5": dict(idx=4, storage=STORAGE_U8, n=10000, p=1000000, design="binom", maf=(0.05, 0.5), k=100,
               effect=("norm", 0.2), noise=3, taus=[0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9], lam=1.0,
               path=20, lam_min=0.01, G=48),
    # metric workload: the C5 design and response, single RHS tau=0.5 (BASELINE.json metric)
    "m": dict(idx=4, storage=STORAGE_U8, n=10000, p=1000000, design="binom", maf=(0.05, 0.5), k=100,
              effect=("norm", 0.2), noise=3, taus=[0.5], lam=0.02, G=48),
}


def make(name: str, n: int | None = None, p: int | None = None, seed: int | None = None,
         storage: int | None = None, G: int | None = None, k: int | None = None) -> Problem:
    """Instantiate config `name`, optionally at reduced size (n, p) with the same recipe."""
    lib = _load()
    cfg = dict(CONFIGS[name])
    n = int(n or cfg["n"])
    p = int(p or cfg["p"])
    storage = cfg["storage"] if storage is None else storage
    seed = BASE_SEED + cfg["idx"] if seed is None else int(seed)
    k = min(int(k or cfg["k"]), p)
    ld = leading_dim(storage, n)

    maf = None
    if cfg["design"] == "gauss":
        if storage != STORAGE_F32:
            raise ValueError("gaussian design is stored as f32")
        X = np.empty((p, ld), dtype=np.float32)
        lib.dg_gauss_f32(seed, n, p, ld, _p(X))
    else:
        if storage == STORAGE_F32:
            raise ValueError("genotype designs are u8 or 2-bit")
        maf = np.empty(p, dtype=np.float64)
        lib.dg_maf(seed, p, cfg["maf"][0], cfg["maf"][1], _p(maf))
        X = np.empty((p, ld), dtype=np.uint8)
        packed = 1 if storage == STORAGE_P2 else 0
        if cfg["design"] == "ld":
            lib.dg_genotypes_ld(seed, n, p, _p(maf), cfg["rho"], cfg["blk"], packed, ld, _p(X))
        else:
            lib.dg_genotypes(seed, n, p, _p(maf), packed, ld, _p(X))

    causal = np.empty(k, dtype=np.int64)
    lib.dg_causal(seed, p, k, _p(causal))
    eff = np.empty(k, dtype=np.float64)
    kind, *par = cfg["effect"]
    if kind == "norm":
        lib.dg_effects(seed, 4, k, 0, par[0], 0.0, _p(eff))
    else:
        lib.dg_effects(seed, 4, k, 1, par[0], par[1], _p(eff))
    mafp = _p(maf) if maf is not None else None
    lin = np.empty(n, dtype=np.float64)
    lib.dg_linpred(storage, n, _p(X), ld, mafp, k, _p(causal), _p(eff), _p(lin))
    eps = np.empty(n, dtype=np.float64)
    lib.dg_noise(seed, n, cfg["noise"], _p(eps))
    meta = {}
    if "hetero" in cfg:
        kg, sd, coef = cfg["hetero"]
        kg = min(kg, k)
        gam = np.empty(kg, dtype=np.float64)
        lib.dg_effects(seed, 6, kg, 0, sd, 0.0, _p(gam))
        cg = np.ascontiguousarray(causal[:kg])
        hg = np.empty(n, dtype=np.float64)
        lib.dg_linpred(storage, n, _p(X), ld, mafp, kg, _p(cg), _p(gam), _p(hg))
        y = lin + (1.0 + coef * np.abs(hg)) * eps
        meta["gamma"] = gam
    else:
        y = lin + eps
    return Problem(name=name, storage=storage, n=n, p=p, ld=ld, X=X, y=np.ascontiguousarray(y),
                   taus=list(cfg["taus"]), lam_frac=cfg["lam"], G=int(G or cfg["G"]), causal=causal,
                   effects=eff, maf=maf, path_points=cfg.get("path", 1), lam_min_frac=cfg.get("lam_min", 0.01),
                   seed=seed, meta=meta)


def splitmix_u64(seed: int, stream: int, idx: int) -> int:
    return int(_load().dg_u64(seed, stream, idx))


def probit(q: float) -> float:
    return float(_load().dg_probit(q))
