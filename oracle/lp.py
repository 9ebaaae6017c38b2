"""Brute-force penalised quantile regression on tiny inputs (TEST INFRASTRUCTURE ONLY).

f(beta) = (1/n) sum_i rho_tau(y_i - a_i^T beta) + sum_{j>=1} lam_j |beta_j|   (E1)

f is convex and piecewise linear on R^{p+1}; its kinks lie on the hyperplanes
{a_i^T beta = y_i} and {beta_j = 0, j >= 1}.  When their normals span R^{p+1}
and f is bounded below, a minimiser sits at a vertex of that arrangement, so
enumerating every (p+1)-subset with independent normals, solving the linear
system and keeping the smallest f gives the exact optimum (SURVEY §8(c),
"LP brute force").  Independent of the FS-QRPPA oracle: plain numpy only.
"""
from __future__ import annotations

import itertools

import numpy as np


def pqr_objective(A: np.ndarray, y: np.ndarray, tau: float, lam: np.ndarray, beta: np.ndarray) -> float:
    u = y - A @ beta
    return float(np.mean(np.where(u < 0, (tau - 1.0) * u, tau * u)) + np.sum(lam[1:] * np.abs(beta[1:])))


def vertex_enumeration(A: np.ndarray, y: np.ndarray, tau: float, lam: np.ndarray):
    """Exact minimum of f over all arrangement vertices.  A: n x (p+1) with the intercept column."""
    n, d = A.shape
    rows = [(A[i], y[i]) for i in range(n)]
    for j in range(1, d):
        e = np.zeros(d)
        e[j] = 1.0
        rows.append((e, 0.0))
    best, best_beta = np.inf, None
    for sub in itertools.combinations(range(len(rows)), d):
        M = np.array([rows[k][0] for k in sub])
        if abs(np.linalg.det(M)) < 1e-10:
            continue
        b = np.linalg.solve(M, np.array([rows[k][1] for k in sub]))
        f = pqr_objective(A, y, tau, lam, b)
        if f < best:
            best, best_beta = f, b
    return best, best_beta


def highs(A: np.ndarray, y: np.ndarray, tau: float, lam: np.ndarray):
    """LP form: min (1/n) sum(tau u + (1-tau) v) + sum lam_j (a_j + b_j)
    s.t. y - A beta = u - v, beta_{1..p} = a - b, u, v, a, b >= 0 (beta_0 free)."""
    from scipy.optimize import linprog

    n, d = A.shape
    p = d - 1
    # variables: beta0 (free), a (p), b (p), u (n), v (n)
    c = np.concatenate([[0.0], lam[1:], lam[1:], np.full(n, tau / n), np.full(n, (1.0 - tau) / n)])
    Aeq = np.hstack([A[:, :1], A[:, 1:], -A[:, 1:], np.eye(n), -np.eye(n)])
    bounds = [(None, None)] + [(0, None)] * (2 * p + 2 * n)
    res = linprog(c, A_eq=Aeq, b_eq=y, bounds=bounds, method="highs")
    beta = np.concatenate([[res.x[0]], res.x[1:1 + p] - res.x[1 + p:1 + 2 * p]])
    return float(res.fun), beta


def highs_saddle(A: np.ndarray, y: np.ndarray, tau: float, lam: np.ndarray):
    """The LP above with its equality duals: (beta*, z* = u - v = y - A beta*, theta*) where theta* are the
    marginals of y - A beta = u - v.  LP duality gives theta* in [(tau-1)/n, tau/n] (u, v columns),
    sum theta* = 0 (free beta_0) and |A_j^T theta*| <= lam_j (a_j, b_j columns) with complementary
    slackness: exactly the saddle-point conditions of Prop. 1."""
    from scipy.optimize import linprog

    n, d = A.shape
    p = d - 1
    c = np.concatenate([[0.0], lam[1:], lam[1:], np.full(n, tau / n), np.full(n, (1.0 - tau) / n)])
    Aeq = np.hstack([A[:, :1], A[:, 1:], -A[:, 1:], np.eye(n), -np.eye(n)])
    bounds = [(None, None)] + [(0, None)] * (2 * p + 2 * n)
    res = linprog(c, A_eq=Aeq, b_eq=y, bounds=bounds, method="highs-ds",
                  options=dict(primal_feasibility_tolerance=1e-10, dual_feasibility_tolerance=1e-10))
    beta = np.concatenate([[res.x[0]], res.x[1:1 + p] - res.x[1 + p:1 + 2 * p]])
    z = res.x[1 + 2 * p:1 + 2 * p + n] - res.x[1 + 2 * p + n:]   # u - v: exact zeros on the interpolated rows
    return beta, z, np.asarray(res.eqlin.marginals, np.float64)
