#!/usr/bin/env python
"""Full-size ORACLE reference trajectories for the GPU parity tests (tests/test_gpu_fullref.py).

TEST INFRASTRUCTURE: this script calls only ``oracle/`` (the fp64 CPU FS-QRPPA) and ``datagen/``
(the seeded inputs); nothing here comes from the CUDA path.  For each BASELINE.json config at its
full size it runs, from the cold start (beta = 0, z = y, theta = 0; reading R5):

  * the oracle's own power method (or Lanczos, --eta-method) for eta_g = 1.05 mu Lambda_max(X~_g^T X~_g)
    (L259, reading R3),
  * lambda = frac * lambda_max(tau) (reading R4; frac from the config, C5 at a mid-path point),
  * exactly K = 200 iterations of Algorithm 1 (``oracle.solve(check=False)``),
  * R(w^K) (reading R1) and the objective E1 at beta^K,

and stores eta, lambda, the sparse beta^K, z^K, theta^K, R and the objective in
``tests/golden/oracle_ref/<config>_tau<tau>.npz`` together with a checksum of the generated design
and response, so a test on the GPU box can confirm it regenerated the same bytes.

  python tools/oracle_ref.py --configs m,c5,c3,c4 [--iters 200]

Runs on the local 8-core CPU box (no GPU): M/C5 ~5 s per oracle pass, C4 ~20 s.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_ref")
# C5 is a 20-point geometric path lambda_max -> 0.01 lambda_max; the reference sits at point 10
# (0-based) of it, lambda = lambda_max * 0.01^(10/19), for tau in {0.1, 0.5, 0.9}
C5_POINT, C5_TAUS = 10, (0.1, 0.5, 0.9)


def design_checksum(prob) -> str:
    """sha256 over y and every 997th stored column (plus the last one): cheap, and any change of
    the generator's bytes moves it."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(prob.y).tobytes())
    cols = np.unique(np.append(np.arange(0, prob.p, 997), prob.p - 1))
    h.update(np.ascontiguousarray(prob.X[cols]).tobytes())
    h.update(f"{prob.storage}:{prob.n}:{prob.p}:{prob.ld}".encode())
    return h.hexdigest()


def lam_frac(name: str, prob) -> float:
    if name == "c5":   # the C5 recipe's path (the M instance shares the design but has no path)
        cfg = datagen.CONFIGS["c5"]
        return cfg["lam_min"] ** (C5_POINT / (cfg["path"] - 1))
    return prob.lam_frac


def cached_eta(name: str, cks: str):
    """eta of an earlier run of this script on the same design (M and C5 share it), else None."""
    key = ("m", "c5") if name in ("m", "c5") else (name,)
    if not os.path.isdir(OUT):
        return None
    for fn in sorted(os.listdir(OUT)):
        if fn.split("_tau")[0] in key:
            z = np.load(os.path.join(OUT, fn))
            if json.loads(str(z["meta"]))["checksum"] == cks:
                return z["eta"]
    return None


def run(name: str, iters: int, prob=None, d=None, eta=None, log=print, eta_method: str = "power"):
    t0 = time.perf_counter()
    if prob is None:
        prob = datagen.make(name)
        d = oracle.Design.from_problem(prob)
    t_gen = time.perf_counter() - t0
    cks = design_checksum(prob)
    mu, G = 2.0 / prob.n, prob.G
    t_eta = 0.0
    if eta is None:
        eta = cached_eta(name, cks)
    if eta is None:
        t0 = time.perf_counter()
        eta = oracle.eta(d, G, mu, method=eta_method)
        t_eta = time.perf_counter() - t0
    log(f"{name}: datagen {t_gen:.1f} s, eta {t_eta:.1f} s")
    taus = C5_TAUS if name == "c5" else prob.taus
    frac = lam_frac(name, prob)
    os.makedirs(OUT, exist_ok=True)
    for tau in taus:
        lm, q = oracle.lambda_max(d, prob.y, tau)
        lam = frac * lm
        lv = oracle.lam_vector(prob.p, lam)
        t0 = time.perf_counter()
        o = oracle.solve(d, prob.y, tau, lv, eta, mu, G, max_iter=iters, check=False)
        t_solve = time.perf_counter() - t0
        R = oracle.kkt_rel(d, prob.y, tau, lv, o["beta"], o["z"], o["theta"])
        obj = oracle.objective(d, prob.y, tau, lv, o["beta"])
        nz = np.flatnonzero(o["beta"])
        fn = os.path.join(OUT, f"{name}_tau{tau:.1f}.npz")
        meta = dict(config=name, tau=tau, n=prob.n, p=prob.p, G=G, mu=mu, lam_frac=frac, iters=iters, eta_method=eta_method,
                    checksum=cks, oracle_s_per_iter=t_solve / iters, threads=os.cpu_count(),
                    script="tools/oracle_ref.py (oracle/ + datagen/ only)")
        np.savez_compressed(fn, eta=eta, lam=lam, lambda_max=lm, q=q, beta_idx=nz.astype(np.int64),
                            beta_val=o["beta"][nz], z=o["z"], theta=o["theta"], R=R, obj=obj,
                            meta=json.dumps(meta))
        log(f"{name} tau={tau}: {iters} it in {t_solve:.0f} s, |S|={len(nz)}, R={R}, obj={obj:.8g} -> {fn}")
    return prob, d, eta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="m,c5,c3,c4")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--eta-method", dest="eta_method", default="power", choices=["power", "lanczos"])
    a = ap.parse_args()
    names = a.configs.split(",")
    cache = {}
    for name in names:
        # M and C5 share the design, the response and G, hence eta
        key = "m" if name in ("m", "c5") else name
        prob, d, eta = cache.get(key, (None, None, None))
        prob, d, eta = run(name, a.iters, prob, d, eta, log=lambda s: print(s, flush=True), eta_method=a.eta_method)
        cache = {key: (prob, d, eta)}


if __name__ == "__main__":
    main()
