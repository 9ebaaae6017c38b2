#!/usr/bin/env python
"""Run a few iterations of a config with ALL its quantile levels in lockstep (for ncu captures of the
multi-RHS kernels).  python tools/iter_rhs.py [--config c5] [--burn-in 20] [--steps 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--burn-in", dest="burn_in", type=int, default=20)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2601_02826_b200 as fs

    prob = datagen.make(args.config)
    X = torch.from_numpy(prob.X).cuda()
    y = torch.from_numpy(prob.y).cuda()
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, prob.taus, [1.0] * len(prob.taus), G=prob.G,
                  mu=2.0 / prob.n)
    S.set_lambda([0.05 * v for v in S.lambda_max()])
    S.iterate(args.burn_in)
    st, tot = fs.fsqr_profile_iterate(S.ctx, args.steps)
    print("stage_ms", (st / args.steps).tolist(), "total_ms", tot / args.steps)


if __name__ == "__main__":
    main()
