#!/usr/bin/env python
"""bench.py — FS-QRPPA hot path on B200: PPA iterations/s and X-streaming HBM GB/s.

Workload (BASELINE.json metric): the C5 design and response (n=10k, p=1M uint8 genotypes,
MAF ~ U(0.05, 0.5), skew-normal noise) with a single RHS tau=0.5, lambda = 0.02 lambda_max,
G=48 ("m" in datagen.CONFIGS).  A step is one outer FS-QRPPA iteration (all SURVEY §8(a)
rows a1-a6), timed through the solver's own launch path (CUDA-graph chunks): one pass over X (10 GB) through the tcgen05 X~^T theta + beta-prox kernel, the
support-gather forward product and the finalize kernel.  Before the warm-up the solver runs a
200-iteration cold-start burn-in so the support is non-trivial.
X (10 GB) is far larger than L2 (126 MB), so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: the path is single-GPU by north_star ("replicas only"); with N ranks
each GPU runs an independent replica and value = total iterations / max time over ranks.
--impl reference: the oracle (oracle/, plain fp64 C, all host cores) on a column sample of the
same workload, reported in the same unit (iterations/s of the full problem).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

STATUS_NAMES = {0: "converged", 2: "max_iter"}
METRIC = "PPA iters/sec and X-streaming HBM GB/s (% of peak) at n=10k, p=1M, tau=0.5"
FALLBACK_HBM = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx: int, path: str):
        self.path = path
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(idx), f"--query-gpu={q}", "--format=csv,noheader",
                                       "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                mx = float(parts[2].split()[0])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def k2_traffic(name: str):
    """dram bytes per K2 launch from the committed ncu --set full capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def max_over_ranks(ms: float, device) -> float:
    """Max of a per-rank device time over all ranks (the whole job ends with its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ms
    t = torch.tensor([ms], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(steps: int, ws: int, max_ms: float) -> float:
    """Weak scaling, replicas only: every rank runs `steps` iterations of its own replica."""
    return steps * ws / (max_ms / 1000.0)


def cpu_baseline(prob, lam_frac, tau, G, mu, budget_s=20.0):
    """The oracle as it stands (plain fp64 C, OpenMP over all host cores) on a contiguous column
    sample of the same workload; scaled to iterations/s of the full problem."""
    import oracle

    cores = os.cpu_count()
    p_s = max(1000, min(prob.p, 60000))
    X = prob.X[:p_s]
    d = oracle.Design(prob.storage, prob.n, p_s, prob.ld, X)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(p_s, lam_frac * lm)
    st = oracle.blocks(p_s + 1, G)
    eta = 1.05 * mu * (prob.n - 1) * np.diff(st).astype(np.float64)  # trace bound >= Lambda_max
    t0 = time.perf_counter()
    oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False)
    t1 = time.perf_counter()
    k = max(1, min(50, int(budget_s / max(t1 - t0, 1e-3))))
    t0 = time.perf_counter()
    oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=k, check=False)
    dt = time.perf_counter() - t0
    frac = p_s / prob.p
    return {"value": k * frac / dt, "unit": "iters/s", "cores": cores, "kind": "oracle",
            "sample": f"{k} oracle iterations on columns 0..{p_s - 1} of {prob.p} ({frac:.4f} of X), "
                      f"rate scaled by the column fraction; OMP threads = {cores}"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    prob = datagen.make(args.config)
    tau = prob.taus[0]
    G = prob.G
    mu = 2.0 / prob.n
    import oracle

    cores = os.cpu_count()
    # size the column sample so that warmup + steps fit in ~150 s of host time
    p_probe = min(prob.p, 20000)
    d = oracle.Design(prob.storage, prob.n, p_probe, prob.ld, prob.X[:p_probe])
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(p_probe, prob.lam_frac * lm)
    eta = 1.05 * mu * (prob.n - 1) * np.diff(oracle.blocks(p_probe + 1, G)).astype(np.float64)
    t0 = time.perf_counter()
    oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False)
    per_col = (time.perf_counter() - t0) / p_probe
    p_s = int(min(prob.p, max(1000, 150.0 / max(args.steps + args.warmup, 1) / per_col)))
    d = oracle.Design(prob.storage, prob.n, p_s, prob.ld, prob.X[:p_s])
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(p_s, prob.lam_frac * lm)
    eta = 1.05 * mu * (prob.n - 1) * np.diff(oracle.blocks(p_s + 1, G)).astype(np.float64)
    w = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=args.warmup, check=False)
    st = (w["beta"], w["z"], w["theta"])
    t0 = time.perf_counter()
    oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=args.steps, check=False, state=st)
    dt = time.perf_counter() - t0
    frac = p_s / prob.p
    value = args.steps * frac / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1000.0 / args.steps / frac,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C5 design/response, single RHS tau=0.5 (BASELINE metric)", "n": prob.n,
                   "p": prob.p, "storage": "u8", "tau": tau, "lambda_frac": prob.lam_frac, "G": G,
                   "column_sample": p_s},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step = one oracle iteration on columns 0..{p_s - 1} ({frac:.4f} of X); "
                                   f"rate scaled by the column fraction"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch

    import paper_2601_02826_b200 as fs

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t_gen = time.perf_counter()
    prob = datagen.make(args.config)
    t_gen = time.perf_counter() - t_gen
    tau = prob.taus[0]
    G = prob.G
    mu = 2.0 / prob.n
    Xd = torch.from_numpy(prob.X).to(dev)
    yd = torch.from_numpy(prob.y).to(dev)
    torch.cuda.synchronize()

    pack = args.storage == "pack2" and prob.storage == fs.U8
    flags = fs.DESIGN_PACK2 if pack else 0
    # the process's first-use costs (lazy module loading, function attributes, tensor-map entry
    # point) on a small slice of the same design, reported apart from setup as setup_first_use_s
    t0 = time.perf_counter()
    pw = min(prob.p, 256 * G)
    Sw = fs.Solver(Xd.reshape(-1)[: pw * prob.ld], prob.storage, prob.n, pw, prob.ld, yd, [tau], [1.0], G=G, mu=mu,
                   flags=flags)
    Sw.iterate(2)
    del Sw
    torch.cuda.synchronize()
    t_first = time.perf_counter() - t0

    # setup (a0, a0', lambda_max) timed separately; lambda = frac * lambda_max from the GPU
    t0 = time.perf_counter()
    kkt_tols = [float(v) for v in str(args.kkt_tol).split(",") if v]
    S = fs.Solver(Xd, prob.storage, prob.n, prob.p, prob.ld, yd, [tau], [1.0], G=G, mu=mu,
                  tol=kkt_tols[0] if kkt_tols else 1e-4, max_iter=args.kkt_max_iter, flags=flags)
    lm = float(S.lambda_max()[0])
    S.set_lambda([prob.lam_frac * lm])
    t_setup = time.perf_counter() - t0
    eta = S.eta()

    S.iterate(args.burn_in)
    S.iterate(args.warmup)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local, os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ".",
                                     f"clocks_rank{rank}.csv"))
    # timed region: blocks of exactly K iterations through the solver's own launch path (CUDA-graph
    # chunks of K2 -> K1(+finalize) with programmatic dependent launch), each bracketed by a barrier
    # and device synchronisation, CUDA events on the launching stream.  The block is repeated until
    # the sampled window is >= --min-window seconds (>= 3 blocks; nvidia-smi samples every 50 ms) and
    # the value uses the median block (each block's time is the max over ranks).
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed_block():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        S.iterate(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(ev0.elapsed_time(ev1), dev)

    first = timed_block()
    nblocks = max(3, int(np.ceil(args.min_window * 1000.0 / max(first, 1e-3))))
    nblocks = min(nblocks, args.max_blocks)
    if ws > 1:
        nb_t = torch.tensor([nblocks], device=dev, dtype=torch.int64)
        dist.all_reduce(nb_t, op=dist.ReduceOp.MAX)
        nblocks = int(nb_t.item())
    block_ms = [first] + [timed_block() for _ in range(nblocks - 1)]
    clocks = clk.stop()
    total_ms = statistics.median(block_ms)
    if ws > 1:
        dist.barrier()
    k = args.steps
    value = whole_job_value(k, ws, total_ms)
    nnz = int(S.trace(1)[-1, 0, 4]) if k > 0 else 0
    # per-stage breakdown (and the dominant kernel's duration for the roofline): the same K
    # iterations again as individual launches with CUDA events around every kernel
    stage_ms, prof_total_ms = fs.fsqr_profile_iterate(S.ctx, args.steps)

    # roofline of the dominant kernel (K2: X~^T theta + beta prox), algorithmic bytes per launch
    two_bit = pack or prob.storage == fs.PACKED2
    # every stored element read once: 2-bit codes, u8 codes, or fp32 values (C1)
    xbytes = prob.n * prob.p // 4 if two_bit else prob.n * prob.p * (4 if prob.storage == fs.F32_DENSE else 1)
    state_bytes = 28 * prob.p                       # beta r/w (16 B) + colsum (4 B) + 1/s_j (8 B) per column
    k2_ms = stage_ms[0] / k
    peak, peak_kind = peaks()
    achieved = (xbytes + state_bytes) / (k2_ms / 1000.0) / 1e9
    traffic = k2_traffic(args.config + ("_pack2" if pack else ""))
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "kernel": ("k2_tc2_kernel<16,1>" if two_bit else "k2_tc_kernel<16,1>") if S.backend == "tc" else "k2_simt", "peak_source": peak_kind,
            "algorithmic_bytes_per_launch": xbytes + state_bytes,
            "kernel_share_of_step": stage_ms[0] / prof_total_ms}
    # cross-check from the timed graph itself: the step minus the other kernels' profiled time
    k2_graph_ms = total_ms / k - (stage_ms[1] + stage_ms[2]) / k
    roof["graph_check"] = {"k2_ms_estimate": k2_graph_ms,
                           "frac": (xbytes + state_bytes) / (k2_graph_ms / 1000.0) / 1e9 / peak,
                           "note": "median timed-block step minus the profiled forward-product (+finalize) time"}

    # the same iterations with the u8 codes streamed as stored (no repack), for comparison
    u8_line = None
    if pack:
        S8 = fs.Solver(Xd, prob.storage, prob.n, prob.p, prob.ld, yd, [tau], [prob.lam_frac * lm], G=G, mu=mu,
                       eta=eta)
        S8.iterate(args.burn_in)
        torch.cuda.synchronize()
        ev0.record(stream)
        S8.iterate(k)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms8 = max_over_ranks(ev0.elapsed_time(ev1), dev)
        u8_line = {"value": whole_job_value(k, ws, ms8), "unit": "iters/s", "ms_per_step": ms8 / k,
                   "x_stream_gbs": prob.n * prob.p / (ms8 / k / 1000.0) / 1e9, "backend": S8.backend}
        del S8

    # e2e through the public C-ABI host-buffer entry (fsqr_fit_host): H2D copy of X and y from pinned
    # memory, setup, k iterations and the D2H read of beta all inside the timed region.
    e2e = None
    if not args.no_e2e:
        # page-lock the generator's own buffer in place (no second 10 GB host copy per rank: at
        # N = 8 every rank holds its own replica); fall back to a pinned copy
        Xh, registered = None, False
        try:
            registered = int(torch.cuda.cudart().cudaHostRegister(prob.X.ctypes.data, prob.X.nbytes, 0)) == 0
        except Exception:
            registered = False
        if registered:
            Xh = prob.X
        else:
            Xp = torch.empty(prob.X.shape, dtype=torch.uint8, pin_memory=True)
            Xp.numpy()[:] = prob.X
            Xh = Xp.numpy()
        yp = torch.empty(prob.n, dtype=torch.float64, pin_memory=True)
        yp.numpy()[:] = prob.y
        # one untimed warm-up call (first-use costs: kernel module loading, stream-ordered pool growth)
        fs.fsqr_fit_host(Xh, prob.storage, prob.n, prob.p, prob.ld, yp.numpy(), [tau], [prob.lam_frac * lm],
                         args.warmup, opt=fs.default_options(G=G, mu=mu), eta=eta, flags=flags)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        beta_h, _ = fs.fsqr_fit_host(Xh, prob.storage, prob.n, prob.p, prob.ld, yp.numpy(), [tau],
                                     [prob.lam_frac * lm], k, opt=fs.default_options(G=G, mu=mu), eta=eta,
                                     flags=flags)
        torch.cuda.synchronize()
        dt = max_over_ranks((time.perf_counter() - t0) * 1000.0, dev) / 1000.0
        e2e = {"value": whole_job_value(k, ws, dt * 1000.0), "unit": "iters/s", "h2d_bytes_per_step": (prob.X.nbytes + prob.y.nbytes) / k,
               "d2h_bytes_per_step": beta_h.nbytes / k,
               "note": "one fsqr_fit_host call after one untimed warm-up call: H2D of X,y (pinned, u8) + setup (eta given"
                       + (", 2-bit repack" if pack else "") + ") + k iterations + D2H beta"}
        if registered:
            torch.cuda.cudart().cudaHostUnregister(prob.X.ctypes.data)
        else:
            del Xp
        e2e["host_buffer"] = "generator buffer page-locked in place" if registered else "pinned copy"

    # time to KKT tolerance: fsqr_solve from the cold start (beta=0, z=y, theta=0),
    # device time of the whole solve (graph chunks, device-side stopping test)
    kkt = None
    if not args.no_kkt:
        kkt = []
        for tol in kkt_tols:
            S.set_tol(tol)
            S.set_state(np.zeros((1, prob.p + 1)), prob.y[None, :], np.zeros((1, prob.n)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = S.solve()
            wall = time.perf_counter() - t0
            kkt.append({"tol": tol, "status": STATUS_NAMES.get(res["status"], res["status"]),
                        "iterations": int(res["iterations"]), "device_s": res["wall_ms"] / 1000.0, "wall_s": wall,
                        "R": [float(v) for v in res["R"][0]], "objective": float(res["objective"][0]),
                        "support": int(S.trace(1)[-1, 0, 4])})

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(prob, prob.lam_frac, tau, G, mu)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": k, "warmup": args.warmup,
            "ms_per_step": total_ms / k, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("f64" if prob.storage == fs.F32_DENSE else
                      ("u2" if two_bit else "u8") + " codes x theta as 28-bit fixed point (4 int8 digits) -> s32 "
                      "exact integer sums; state and proxes f64"),
            "data": "synthetic",
            "config": {"workload": ("C5 design/response, single RHS tau=0.5 (BASELINE metric)" if args.config == "m"
                                    else f"config {args.config}, first tau only (not the metric workload)"), "n": prob.n,
                       "p": prob.p, "storage": {fs.U8: "u8 input", fs.PACKED2: "2-bit packed", fs.F32_DENSE: "fp32"}[prob.storage]
                       + (", repacked to 2 bits at create (FSQR_DESIGN_PACK2)" if pack else
                          (", streamed as u8" if prob.storage == fs.U8 else "")), "tau": tau, "lambda": prob.lam_frac * lm, "lambda_frac":
                       prob.lam_frac, "G": G, "mu": mu, "burn_in": args.burn_in, "support": nnz,
                       "l2": (f"X ({xbytes / 1e9:.1f} GB streamed) >> L2 (126 MB): no flush needed" if xbytes > 126e6
                              else f"X ({xbytes / 1e6:.0f} MB) fits in L2: not flushed (not the metric workload)"),
                       "parallelism": f"replicas x{ws}",
                       "backend": S.backend, "setup_s": t_setup, "setup_first_use_s": t_first, "datagen_s": t_gen},
            "u8_storage": u8_line,
            "x_stream_gbs": xbytes / (total_ms / k / 1000.0) / 1e9,
            "x_stream_frac_of_peak": xbytes / (total_ms / k / 1000.0) / 1e9 / peak,
            "stage_ms_per_step": {"k2_xt_theta_prox": stage_ms[0] / k, "k1_forward_and_finalize": stage_ms[1] / k,
                                  "finalize_separate": stage_ms[2] / k, "_note": "separate profiled pass: one launch "
                                  "per kernel with CUDA events between them (adds launch gaps); with genotype "
                                  "storage the finalize runs inside the forward-product kernel",
                                  "total_profiled_ms_per_step": prof_total_ms / k},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "time_to_kkt": kkt,
            "gpu_launches": S.launches_per_iteration() * k,
            "timing": {"blocks": len(block_ms), "block_ms_min": min(block_ms), "block_ms_median": total_ms,
                       "block_ms_max": max(block_ms), "window_s": sum(block_ms) / 1000.0,
                       "note": "value and ms_per_step use the median block of exactly K iterations"},
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)   # ~1 s timed region, so nvidia-smi sees it
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="m")
    ap.add_argument("--burn-in", dest="burn_in", type=int, default=200)
    ap.add_argument("--storage", default="pack2", choices=["u8", "pack2"],
                    help="device layout of the u8 genotype input: as is, or repacked to 2 bits at create")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kkt", action="store_true")
    ap.add_argument("--kkt-tol", dest="kkt_tol", default="1e-4,1e-6",
                    help="time to R(w) <= tol from the cold start, for each tolerance listed")
    ap.add_argument("--kkt-max-iter", dest="kkt_max_iter", type=int, default=300000)
    ap.add_argument("--min-window", dest="min_window", type=float, default=1.0,
                    help="seconds of timed blocks (clock sampling window)")
    ap.add_argument("--max-blocks", dest="max_blocks", type=int, default=400)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
