#!/usr/bin/env python
"""ORACLE reference of the paper's tuning path at C2 full size (tests/test_gpu_fullref.py).

TEST INFRASTRUCTURE: calls only oracle/ and datagen/.  C2 (n = 2000, p = 50000, the dimensions of
the paper's Table 2) at tau = 0.5 with G = 5 (the paper's simulation setting, L416): the oracle's own
power-method eta, lambda_max (reading R4), a geometric grid of T points from lambda_max down to
lam_min_frac * lambda_max (reading R20 with B = 0), the warm-started path of reading R10
(oracle.path, tol 1e-4) and HBIC (E18) of every point.  Stored: grid, per-point update counts,
convergence flags, objectives, R, HBIC and the sparse beta of every point, plus the design
checksum, in tests/golden/oracle_ref/c2_path_tau0.5.npz.

  python tools/oracle_path_ref.py [--T 12] [--lam-min-frac 0.05]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import datagen  # noqa: E402
import oracle  # noqa: E402
from oracle_ref import OUT, design_checksum  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=12)
    ap.add_argument("--lam-min-frac", dest="lam_min_frac", type=float, default=0.05)
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iter-point", dest="max_iter_point", type=int, default=20000)
    a = ap.parse_args()
    prob = datagen.make("c2")
    d = oracle.Design.from_problem(prob)
    tau, G, mu = 0.5, prob.G, 2.0 / prob.n
    t0 = time.perf_counter()
    eta = oracle.eta(d, G, mu)
    t_eta = time.perf_counter() - t0
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    T = a.T
    grid = np.array([lm * (a.lam_min_frac) ** (t / (T - 1)) for t in range(T)])
    t0 = time.perf_counter()
    res = oracle.path(d, prob.y, tau, grid, eta, mu, G, a.tol, a.max_iter_point)
    t_path = time.perf_counter() - t0
    hb = np.array([oracle.hbic(d, prob.y, tau, res["beta_path"][t]) for t in range(T)])
    idx = [np.flatnonzero(res["beta_path"][t]) for t in range(T)]
    cnt = np.array([len(i) for i in idx])
    meta = dict(config="c2", tau=tau, n=prob.n, p=prob.p, G=G, mu=mu, T=T, lam_min_frac=a.lam_min_frac, tol=a.tol,
                max_iter_point=a.max_iter_point, checksum=design_checksum(prob), eta_s=t_eta, path_s=t_path,
                threads=os.cpu_count(), script="tools/oracle_path_ref.py (oracle/ + datagen/ only)")
    os.makedirs(OUT, exist_ok=True)
    fn = os.path.join(OUT, "c2_path_tau0.5.npz")
    np.savez_compressed(fn, eta=eta, lambda_max=lm, grid=grid, iters=res["iters"], converged=res["converged"],
                        obj=res["obj"], R=res["R"], hbic=hb, beta_cnt=cnt, beta_idx=np.concatenate(idx).astype(np.int64),
                        beta_val=np.concatenate([res["beta_path"][t][idx[t]] for t in range(T)]), total=res["total"],
                        meta=json.dumps(meta))
    print(f"c2 path: eta {t_eta:.0f} s, path {t_path:.0f} s, {res['total']} updates, iters {res['iters'].tolist()}, "
          f"hbic argmin {int(np.argmin(hb))} -> {fn}", flush=True)


if __name__ == "__main__":
    main()
