#!/usr/bin/env python
"""The paper's tuning protocol on the GPU, timed: one fsqr_tune call = a
warm-started path over T = 50 geometric lambda values (reading R20) + HBIC of every point + the
argmin, through the C ABI.  Reported beside the paper's own wall time for the same dimensions
(context, not a target: Table 2, n = 2000, p = 50000, tau = 0.5, LASSO, 50-lambda path with HBIC:
12.25 s on an Apple M4 Max CPU, G = 5).

  python tools/tune_protocol.py [--configs c2,m] [--T 50] [--tol 1e-4]

JSON line per config: setup_s (create: column statistics, power method, lambda_max), tune_s (the
fsqr_tune call), total passes over X, per-point update counts, the selected point and its support.
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

import datagen  # noqa: E402

PAPER = {"c2": {"seconds": 12.25, "sd": 0.31, "hardware": "Apple M4 Max CPU, 64 GB (PAPER.md:L416)",
                "setting": "n=2000, p=50000, tau=0.5, LASSO, 50 lambdas, HBIC, G=5, Gaussian AR(1) design "
                           "(Table 2, PAPER.md:L517-519)"}}


def main():
    import torch

    import paper_2601_02826_b200 as fs

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,m")
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--lam-min-frac", dest="lam_min_frac", type=float, default=0.01)
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iter-point", dest="max_iter_point", type=int, default=20000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    for name in a.configs.split(","):
        prob = datagen.make(name)
        X = torch.from_numpy(prob.X).cuda()
        y = torch.from_numpy(prob.y).cuda()
        tau = 0.5
        G = 5 if name == "c2" else prob.G
        pack = prob.storage == fs.U8 and name != "c2"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [1.0], G=G, mu=2.0 / prob.n, tol=a.tol,
                      max_iter_point=a.max_iter_point, flags=fs.DESIGN_PACK2 if pack else 0)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        out = S.tune(T=a.T, lam_min_frac=a.lam_min_frac)
        torch.cuda.synchronize()
        tune = time.perf_counter() - t0
        best = int(out["best"][0])
        line = dict(config=name, n=prob.n, p=prob.p, tau=tau, G=G, T=a.T, lam_min_frac=a.lam_min_frac, tol=a.tol,
                    storage="u8 repacked to 2 bits" if pack else datagen.STORAGE_NAMES[prob.storage],
                    setup_s=setup, tune_s=tune, total_s=setup + tune, passes_over_X=out["total"],
                    best=best, lambda_best=float(out["grid"][0, best]), hbic_best=float(out["hbic"][0, best]),
                    support_best=int(np.count_nonzero(out["beta"][0][1:])), paper=PAPER.get(name))
        print(json.dumps(line), flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(json.dumps(line) + "\n")
        del S, X, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
