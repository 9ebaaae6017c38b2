#!/usr/bin/env python
"""Iterations (and seconds) to the KKT tolerance as a function of the paper's free parameters mu
("pre-specified"; reading R2) and G (Remark 1, L307-310), on one B200.

  python tools/sweep_mu.py [--config m] [--tol 1e-4] [--mus 0.5,1,2,4,8] [--Gs 5,48]

mu is given in units of 1/n.  One JSON line per (G, mu).  The power method runs per G (eta_g
depends on the blocks); the solve starts from the cold start each time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="m")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--mus", default="0.5,1,2,4,8")
    ap.add_argument("--Gs", default="5,48")
    ap.add_argument("--max-iter", dest="max_iter", type=int, default=40000)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2601_02826_b200 as fs

    prob = datagen.make(args.config)
    X = torch.from_numpy(prob.X).cuda()
    y = torch.from_numpy(prob.y).cuda()
    tau = prob.taus[0]
    for G in [int(g) for g in args.Gs.split(",")]:
        for m in [float(v) for v in args.mus.split(",")]:
            mu = m / prob.n
            t0 = time.perf_counter()
            S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [1.0], G=G, mu=mu, tol=args.tol,
                          max_iter=args.max_iter)
            setup = time.perf_counter() - t0
            lam = prob.lam_frac * S.lambda_max()[0]
            S.set_lambda([lam])
            t0 = time.perf_counter()
            res = S.solve()
            dt = time.perf_counter() - t0
            line = dict(config=args.config, G=G, mu_times_n=m, tol=args.tol, status=res["status"],
                        iterations=res["iterations"], solve_s=dt, setup_s=setup, R=res["R"][0].tolist(),
                        objective=float(res["objective"][0]), support=int(S.trace(1)[-1, 0, 4]))
            print(json.dumps(line), flush=True)
            if args.out:
                with open(args.out, "a") as f:
                    f.write(json.dumps(line) + "\n")
            del S
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
