#!/usr/bin/env python
"""The ORACLE's own cost on the GPU box's host cores, per BASELINE.json config.

TEST/MEASUREMENT INFRASTRUCTURE: runs only oracle/ (plain fp64 C, OpenMP over all host cores,
fixed-order sums) on the seeded datagen/ inputs; nothing from the CUDA path.  For each config:

  * s/iter: median over K timed oracle iterations of Algorithm 1 (one X~^T theta pass over every
    column + the support forward product), after a short untimed warm-up from the cold start at the
    config's lambda, with the oracle's own eta (the committed full-size references' where they
    exist, else Lanczos), so the support, hence the forward product's cost, is the real one;
  * optionally the same with OMP_NUM_THREADS=1 (C1, C2);
  * optionally time to R <= tol from the cold start with the oracle's own power-method eta
    (C1 at 1e-6, C2 tau=0.5 at 1e-4), wall seconds and iterations.

One JSON line per measurement.  python tools/oracle_onbox.py [--configs c1,c2,c3,c4,m] [--iters 5]
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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def emit(d, out):
    line = json.dumps(d)
    print(line, flush=True)
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


def ref_eta(name: str):
    """the oracle's own eta from the committed full-size references (tools/oracle_ref.py), if any"""
    key = "m" if name in ("m", "c5") else name
    ref = os.path.join(ROOT, "tests", "golden", "oracle_ref")
    for fn in sorted(os.listdir(ref)) if os.path.isdir(ref) else []:
        if fn.startswith(("m_", "c5_") if key == "m" else (key + "_tau",)):
            return np.load(os.path.join(ref, fn))["eta"]
    return None


def s_per_iter(name: str, iters: int, warm: int):
    prob = datagen.make(name)
    d = oracle.Design.from_problem(prob)
    tau = prob.taus[0]
    G, mu = prob.G, 2.0 / prob.n
    frac = prob.lam_frac if prob.path_points == 1 else 0.1
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, frac * lm)
    eta = ref_eta(name)
    if eta is None:
        eta = oracle.eta(d, G, mu, method="lanczos")
    w = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=warm, check=False)
    state = (w["beta"], w["z"], w["theta"])
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        w = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False, state=state)
        ts.append(time.perf_counter() - t0)
        state = (w["beta"], w["z"], w["theta"])
    return dict(config=name, n=prob.n, p=prob.p, storage=datagen.STORAGE_NAMES[prob.storage], tau=tau,
                mode="s_per_iter", iters=iters, warm=warm, s_per_iter=statistics.median(ts), s_min=min(ts),
                support=int(np.count_nonzero(state[0][1:])), threads=int(os.environ.get("OMP_NUM_THREADS",
                                                                                         os.cpu_count())))


def time_to_kkt(name: str, tol: float, max_iter: int):
    prob = datagen.make(name)
    d = oracle.Design.from_problem(prob)
    tau = 0.5 if 0.5 in prob.taus else prob.taus[0]
    G, mu = prob.G, 2.0 / prob.n
    t0 = time.perf_counter()
    eta = oracle.eta(d, G, mu)
    t_eta = time.perf_counter() - t0
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, prob.lam_frac * lm)
    t0 = time.perf_counter()
    o = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=max_iter, tol=tol)
    dt = time.perf_counter() - t0
    return dict(config=name, n=prob.n, p=prob.p, tau=tau, mode="time_to_kkt", tol=tol, status=o["status"],
                iterations=o["iters"], solve_s=dt, eta_s=t_eta, R=o["R"].tolist(), objective=o["obj"],
                threads=os.cpu_count())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,m")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--single-thread", default="c1,c2")
    ap.add_argument("--kkt", default="c1:1e-6,c2:1e-4")
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", default=None, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.child:   # one measurement in a subprocess (OMP_NUM_THREADS is read once per process)
        emit(s_per_iter(a.child, a.iters, a.warm), a.out)
        return
    lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    model = next((l.split(":", 1)[1].strip() for l in lscpu.splitlines() if l.startswith("Model name")), "?")
    emit(dict(mode="host", cpu=model, cores=os.cpu_count()), a.out)
    for name in a.configs.split(","):
        emit(s_per_iter(name, a.iters, a.warm), a.out)
        if name in a.single_thread.split(","):
            env = dict(os.environ, OMP_NUM_THREADS="1")
            subprocess.run([sys.executable, __file__, "--child", name, "--iters", str(max(2, a.iters // 2)),
                            "--warm", str(a.warm)] + (["--out", a.out] if a.out else []), env=env, check=True)
    for spec in filter(None, a.kkt.split(",")):
        name, tol = spec.split(":")
        emit(time_to_kkt(name, float(tol), 400000), a.out)


if __name__ == "__main__":
    main()
