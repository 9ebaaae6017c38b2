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
              backend=0, oracle_eta=True, tol=1e-6, max_iter=100000, **kw):
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
                  backend=backend, eta=eta, **kw)
    return prob, d, S, dict(taus=taus, lams=lams, G=G, mu=mu, eta=eta, lm=lm)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def support_mismatch(beta_gpu, beta_orc, g_margin=None):
    """Indices where exactly one side is zero."""
    return np.flatnonzero((beta_gpu != 0) != (beta_orc != 0))


# ------------------------------------------------------------------ numpy one-step checker (test-local)
# Written from the paper's formulas (E14, E15, E12); it never calls the oracle, whose inputs never
# come from the CUDA path, so it can check a GPU step taken from any GPU state.

def raw_columns(prob, cols):
    """fp64 codes [len(cols), n] of the stored data columns (any storage)."""
    Xc = prob.X[cols]
    if prob.storage == datagen.STORAGE_P2:
        codes = (Xc[:, :, None] >> (2 * np.arange(4, dtype=np.uint8))) & 3
        return codes.reshape(len(cols), -1)[:, : prob.n].astype(np.float64)
    return Xc[:, : prob.n].astype(np.float64)


def block_of(j, p1, G):
    """DESIGN.md R6: contiguous blocks, the first (p+1) mod G one column larger."""
    q, rem = p1 // G, p1 % G
    big = rem * (q + 1)
    j = np.asarray(j)
    return np.where(j < big, j // (q + 1), rem + (j - big) // max(q, 1))


def prox_beta_np(b, g, lam, eta):
    a = eta * b + g
    return (np.maximum(a - lam, 0.0) - np.maximum(-a - lam, 0.0)) / eta


def forward_np(prob, beta_col):
    """s = X~ beta over the nonzero model columns (beta_col: [p+1])."""
    s = np.full(prob.n, beta_col[0])
    nz = np.flatnonzero(beta_col[1:] != 0.0)
    for a in range(0, len(nz), 2048):
        cols = nz[a:a + 2048]
        raw = raw_columns(prob, cols)
        m = raw.mean(axis=1)
        sd = raw.std(axis=1, ddof=1)
        s += ((raw - m[:, None]) / sd[:, None]).T @ beta_col[cols + 1]
    return s


def check_one_step(prob, S, taus, lams, eta, mu, G, seed=7, ncols=4000):
    import paper_2601_02826_b200 as fs

    b0, z0, t0 = S.state()
    fs.fsqr_profile_iterate(S.ctx, 1)          # exactly the launches bench.py times
    b1, z1, t1 = S.state()
    R, n, p = len(taus), prob.n, prob.p
    rng = np.random.default_rng(seed)
    sup = np.flatnonzero((b0[:, 1:] != 0).any(axis=0) | (b1[:, 1:] != 0).any(axis=0))
    cols = np.union1d(rng.choice(p, size=min(ncols, p), replace=False), sup)
    n_checked = 0
    for a in range(0, len(cols), 2048):
        cc = cols[a:a + 2048]
        raw = raw_columns(prob, cc)
        m = raw.mean(axis=1)
        sd = raw.std(axis=1, ddof=1)
        xt = (raw - m[:, None]) / sd[:, None]
        g = xt @ t0.T                      # [c, R]
        gabs = np.abs(xt) @ np.abs(t0).T   # dot-product error scale
        j = cc + 1
        e = eta[block_of(j, p + 1, G)]
        for r in range(R):
            exp = prox_beta_np(b0[r, j], g[:, r], lams[r], e)
            err = np.abs(b1[r, j] - exp)
            bound = 1e-5 * gabs[:, r] / e + 1e-300
            assert np.all(err <= bound), (r, int(np.argmax(err / bound)), float(np.max(err / bound)))
            margin = np.abs(np.abs(e * b0[r, j] + g[:, r]) - lams[r])
            clear = margin > 1e-6 * lams[r]
            assert np.array_equal((b1[r, j] != 0)[clear], (exp != 0)[clear])
            n_checked += len(j)
    # intercept (lambda_0 = 0, block 1)
    for r in range(R):
        exp0 = b0[r, 0] + t0[r].sum() / eta[0]
        assert abs(b1[r, 0] - exp0) <= 1e-5 * np.abs(t0[r]).sum() / eta[0]
    # rows: E15 for z, E12 for theta with s = X~ beta recomputed from the bytes
    sigma = mu / (G + 1)
    for r in range(R):
        tau = taus[r]
        v = z0[r] + t0[r] / mu
        z_exp = np.maximum(v - tau / (n * mu), 0.0) - np.maximum(-v - (1 - tau) / (n * mu), 0.0)
        np.testing.assert_allclose(z1[r], z_exp, rtol=1e-12, atol=1e-12 * np.abs(z_exp).max())
        s0 = forward_np(prob, b0[r])
        s1 = forward_np(prob, b1[r])
        r0 = s0 + z0[r] - prob.y
        r1 = s1 + z1[r] - prob.y
        dth = -sigma * (2 * r1 - r0)
        # E12 consumes the forward products s^k, s^{k+1}, so the dual step can differ by at most
        # sigma (2 |ds1| + |ds0|).  north_star allows products within 1e-5; the forward product here
        # is an exact integer sum of C_j = round(2^E beta_j / s_j) with 2^E max|C| <= 2^61 / (2 n |S|)
        # (fsqr_dev.cuh fwd_exponent), i.e. ~2^-33 of max|beta_j / s_j| per coefficient at M; the
        # rounding errors of |S| ~ 1e4 coefficients add to ~1e-9..1e-8 of |s| per row.  The bound is
        # 1e-7 relative: 100x tighter than north_star's, enough to see a lost digit or a mis-scaled row.
        err = np.linalg.norm((t1[r] - t0[r]) - dth)
        assert err <= 1e-7 * sigma * (2 * np.linalg.norm(s1) + np.linalg.norm(s0)), (err, np.linalg.norm(dth))
    return n_checked, len(sup)


