#!/usr/bin/env python
"""Per-config measurement of the FS-QRPPA hot path on one B200 (all BASELINE.json configs).

For each config: setup time (a0 column stats, a0' power method, lambda_max), PPA iterations/s
over a timed window after a burn-in (CUDA events per stage, fsqr_profile_iterate), the X-stream
GB/s, and time-to-KKT (fsqr_solve to R(w) <= tol from the cold start).  C5 runs its 20-point
geometric lambda path for the 9 quantile levels jointly.  One JSON line per measurement.

  python tools/bench_configs.py [--configs c2,c3,c4,c5,m] [--steps 50] [--burn-in 200]
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


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def emit(d, out):
    line = json.dumps(d)
    print(line, flush=True)
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


def run(name, args):
    import torch

    import paper_2601_02826_b200 as fs

    t0 = time.perf_counter()
    prob = datagen.make(name)
    t_gen = time.perf_counter() - t0
    X = torch.from_numpy(prob.X).cuda()
    y = torch.from_numpy(prob.y).cuda()
    mu = 2.0 / prob.n
    pack = args.pack2 and prob.storage == datagen.STORAGE_U8
    xbytes = prob.n * prob.p // 4 if pack else prob.X.nbytes   # bytes each K2 pass streams
    taus = prob.taus
    base = dict(config=name, n=prob.n, p=prob.p,
                storage=datagen.STORAGE_NAMES[prob.storage] + (" -> 2-bit (FSQR_DESIGN_PACK2)" if pack else ""), G=prob.G,
                x_bytes=xbytes, datagen_s=t_gen)
    groups = [taus] if (name == "c5" or len(taus) == 1) else [[t] for t in taus] + [taus]
    for tg in groups:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, tg, [1.0] * len(tg), G=prob.G, mu=mu,
                      tol=args.tol, max_iter=args.max_iter, backend=args.backend,
                      flags=fs.DESIGN_PACK2 if pack else 0)
        lm = S.lambda_max()
        setup_s = time.perf_counter() - t0
        rec = dict(base, taus=tg, backend=S.backend, setup_s=setup_s, lambda_max=lm.tolist())
        if name == "c5":
            T = prob.path_points
            grid = np.array([[l * prob.lam_min_frac ** (t / (T - 1)) for t in range(T)] for l in lm])
            S.set_lambda(grid[:, 0])
            S.iterate(args.burn_in)
            st, tot = fs.fsqr_profile_iterate(S.ctx, args.steps)
            rec.update(mode="iters", lam=grid[:, 0].tolist(), steps=args.steps, ms_per_step=tot / args.steps,
                       iters_per_s=args.steps / (tot / 1e3), rhs_iters_per_s=len(tg) * args.steps / (tot / 1e3),
                       stage_ms=(st / args.steps).tolist(), x_gbs=xbytes / (tot / args.steps / 1e3) / 1e9,
                       k2_frac_of_peak=xbytes / (st[0] / args.steps / 1e3) / 1e9 / peak(),
                       support=int(S.trace(1)[-1, :, 4].max()))
            emit(rec, args.out)
            if args.no_kkt:
                continue
            # the full warm-started path from the cold start
            S.set_state(np.zeros((len(tg), prob.p + 1)), np.tile(prob.y, (len(tg), 1)),
                        np.zeros((len(tg), prob.n)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = S.path(grid)
            dt = time.perf_counter() - t0
            rec2 = dict(base, taus=tg, mode="path", T=T, tol=args.tol, total_iters=res["total"], path_s=dt,
                        iters_per_s=res["total"] / dt, converged_points=int(res["converged"].sum()),
                        points=int(res["converged"].size), iters_per_point=res["iters"].tolist(),
                        nnz_last=res["nnz"][:, -1].tolist())
            emit(rec2, args.out)
            continue
        lam = [prob.lam_frac * v for v in lm]
        S.set_lambda(lam)
        S.iterate(args.burn_in)
        # graph-chunk iterations (the solver's own launch path), device time with CUDA events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kg = max(args.steps, 4 * 16)
        e0.record()
        S.iterate(kg)
        e1.record()
        torch.cuda.synchronize()
        graph_ips = kg / (e0.elapsed_time(e1) / 1e3)
        st, tot = fs.fsqr_profile_iterate(S.ctx, args.steps)
        rec.update(mode="iters", lam=lam, burn_in=args.burn_in, steps=args.steps, ms_per_step=tot / args.steps,
                   graph_iters_per_s=graph_ips,
                   iters_per_s=args.steps / (tot / 1e3), stage_ms=(st / args.steps).tolist(),
                   x_gbs=xbytes / (tot / args.steps / 1e3) / 1e9,
                   k2_frac_of_peak=xbytes / (st[0] / args.steps / 1e3) / 1e9 / peak(),
                   support=int(S.trace(1)[-1, :, 4].max()))
        emit(rec, args.out)
        if args.pivotal and prob.storage == datagen.STORAGE_U8 and not pack and len(tg) == 1:
            S.pivotal(128, seed=1)          # first call allocates and builds its tensor maps
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L = S.pivotal(args.pivotal, seed=7)
            dt = time.perf_counter() - t0
            s_ = np.sort(L)
            emit(dict(base, taus=tg, mode="pivotal", B=args.pivotal, seconds=dt,
                      passes=(args.pivotal + 127) // 128, x_gbs_per_pass=xbytes * ((args.pivotal + 127) // 128) / dt / 1e9,
                      lambda_piv=float(1.1 * s_[int(np.ceil(0.9 * len(s_))) - 1]), lambda_max=float(lm[0])), args.out)
        if args.no_kkt:
            continue
        # time to KKT tolerance from the cold start
        S.set_state(np.zeros((len(tg), prob.p + 1)), np.tile(prob.y, (len(tg), 1)), np.zeros((len(tg), prob.n)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = S.solve()
        dt = time.perf_counter() - t0
        emit(dict(base, taus=tg, mode="kkt", tol=args.tol, status=res["status"], iterations=res["iterations"],
                  wall_s=dt, device_ms=res["wall_ms"], R=res["R"].tolist(), objective=res["objective"].tolist(),
                  support=int(S.trace(1)[-1, :, 4].max())), args.out)
        del S
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5,m")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--burn-in", dest="burn_in", type=int, default=200)
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iter", dest="max_iter", type=int, default=20000)
    ap.add_argument("--backend", type=int, default=0)
    ap.add_argument("--no-kkt", action="store_true")
    ap.add_argument("--pivotal", type=int, default=0, help="also time B pivotal replicates (u8, one RHS)")
    ap.add_argument("--pack2", action="store_true", help="repack u8 designs to 2 bits at create")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    for name in args.configs.split(","):
        run(name.strip(), args)


if __name__ == "__main__":
    main()
