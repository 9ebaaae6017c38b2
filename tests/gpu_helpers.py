"""Shared helpers for the GPU parity tests: build the same seeded problem for the oracle and the
CUDA path.  The CUDA path is always called through the C ABI (paper_2601_02826_b200)."""
import numpy as np

import datagen
import oracle


def to_device(prob):
    import torch

    X = torch.from_numpy(prob.X).cuda()
    y = torch.from_numpy(prob.y).cuda()
    return X, y


def make_pair(name, n=None, p=None, seed=None, storage=None, G=None, taus=None, lam_frac=None, mu=None,
              backend=0, oracle_eta=True, tol=1e-6, max_iter=100000):
    """Return (prob, oracle Design, solver, dict of shared settings).  eta comes from the ORACLE
    (power method on the CPU) and is handed to the GPU, never the other way round."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make(name, n=n, p=p, seed=seed, storage=storage, G=G)
    d = oracle.Design.from_problem(prob)
    taus = list(prob.taus if taus is None else taus)
    lam_frac = prob.lam_frac if lam_frac is None else lam_frac
    G = prob.G
    mu = 2.0 / prob.n if mu is None else mu
    lm = [oracle.lambda_max(d, prob.y, t)[0] for t in taus]
    lams = [lam_frac * v for v in lm]
    eta = oracle.eta(d, G, mu) if oracle_eta else None
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, lams, G=G, mu=mu, tol=tol, max_iter=max_iter,
                  backend=backend, eta=eta)
    return prob, d, S, dict(taus=taus, lams=lams, G=G, mu=mu, eta=eta, lm=lm)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def support_mismatch(beta_gpu, beta_orc, g_margin=None):
    """Indices where exactly one side is zero."""
    return np.flatnonzero((beta_gpu != 0) != (beta_orc != 0))
