"""Pins for the oracle (CPU only): it is checked against what the paper and the mathematics
fix, never against itself.  Each test names the passage it pins."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import datagen
import oracle
from oracle import lp

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "worked_values.json")))


# ----------------------------------------------------------------- proxes (E14, E15, E12)

@pytest.mark.parametrize("case", GOLD["prox_beta"])
def test_prox_beta_worked_values(case):
    v = oracle.prox_beta(case["beta"], case["g"], case["lam"], case["eta"])
    assert v == pytest.approx(case["expect"], abs=1e-15), case["cite"]
    if case["expect"] == 0.0:
        assert v == 0.0  # exact zero in the dead zone


@pytest.mark.parametrize("case", GOLD["prox_z"])
def test_prox_z_worked_values(case):
    v = oracle.prox_z(case["z"], case["theta"], case["mu"], case["tau"], case["n"])
    assert v == pytest.approx(case["expect"], abs=1e-15), case["cite"]


@pytest.mark.parametrize("case", GOLD["dual"])
def test_dual_worked_values(case):
    v = oracle.dual(case["theta"], case["r_new"], case["r_old"], case["mu"], case["G"])
    assert v == pytest.approx(case["expect"], abs=1e-15), case["cite"]


@pytest.mark.parametrize("case", GOLD["rho"])
def test_rho_worked_values(case):
    assert oracle.rho(case["u"], case["tau"]) == pytest.approx(case["expect"], abs=1e-15), case["cite"]


def _argmin_1d(f, lo, hi):
    """Brute force: dense grid then golden-section refinement (independent of the closed forms)."""
    xs = np.linspace(lo, hi, 20001)
    fx = np.array([f(x) for x in xs])
    k = int(np.argmin(fx))
    a, b = xs[max(k - 1, 0)], xs[min(k + 1, len(xs) - 1)]
    gr = (np.sqrt(5) - 1) / 2
    for _ in range(200):
        c, d = b - gr * (b - a), a + gr * (b - a)
        if f(c) < f(d):
            b = d
        else:
            a = c
    return 0.5 * (a + b)


def test_prox_beta_bruteforce():
    """E13/E14: beta+ = argmin lam|b| - g b + (eta/2)(b - beta)^2."""
    rng = np.random.default_rng(1)
    for _ in range(60):
        beta, g = rng.normal(), rng.normal()
        lam, eta = abs(rng.normal()) * rng.choice([0, 0.3, 1, 3]), rng.uniform(0.2, 5)
        f = lambda b: lam * abs(b) - g * b + 0.5 * eta * (b - beta) ** 2
        ref = _argmin_1d(f, -20, 20)
        assert oracle.prox_beta(beta, g, lam, eta) == pytest.approx(ref, abs=1e-7)


def test_prox_z_bruteforce():
    """E15: z+ = argmin (1/n) rho_tau(z) - theta z + (mu/2)(z - z^k)^2."""
    rng = np.random.default_rng(2)
    for _ in range(60):
        tau = rng.uniform(0.05, 0.95)
        n = int(rng.integers(1, 50))
        mu = rng.uniform(0.05, 3)
        z0, th = rng.normal(), rng.normal() * 0.1
        f = lambda z: (tau - (z < 0)) * z / n - th * z + 0.5 * mu * (z - z0) ** 2
        ref = _argmin_1d(f, -20, 20)
        assert oracle.prox_z(z0, th, mu, tau, n) == pytest.approx(ref, abs=1e-7)


# ----------------------------------------------------------------- design + products

def _np_standardized(prob):
    """Independent numpy construction of X~ (n x (p+1)) from the stored bytes (L404)."""
    if prob.storage == datagen.STORAGE_F32:
        raw = prob.X[:, :prob.n].astype(np.float64).T
    elif prob.storage == datagen.STORAGE_U8:
        raw = prob.X[:, :prob.n].astype(np.float64).T
    else:
        b = prob.X.astype(np.int64)
        codes = np.stack([(b >> (2 * q)) & 3 for q in range(4)], axis=2).reshape(prob.p, -1)
        raw = codes[:, :prob.n].astype(np.float64).T
    m = raw.mean(axis=0)
    s = raw.std(axis=0, ddof=1)
    return np.hstack([np.ones((prob.n, 1)), (raw - m) / s]), m, s


@pytest.mark.parametrize("name,storage", [("c1", 0), ("c2", 1), ("c4", 2)])
def test_colstats_and_products_vs_numpy(name, storage):
    prob = datagen.make(name, n=37 if storage != 2 else 401, p=23, storage=storage)
    d = oracle.Design.from_problem(prob)
    A, m, s = _np_standardized(prob)
    np.testing.assert_allclose(d.mean, m, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(d.sd, s, rtol=1e-13)
    rng = np.random.default_rng(3)
    th = rng.normal(size=prob.n)
    be = rng.normal(size=prob.p + 1) * (rng.random(prob.p + 1) < 0.5)
    np.testing.assert_allclose(oracle.backprod(d, th), A.T @ th, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.fwdprod(d, be), A @ be, rtol=1e-12, atol=1e-12)
    # the standardised columns have mean 0 and sd 1
    np.testing.assert_allclose(A[:, 1:].mean(axis=0), 0, atol=1e-12)
    np.testing.assert_allclose(A[:, 1:].std(axis=0, ddof=1), 1, rtol=1e-12)


def test_partition_invariance_products():
    """X beta = sum_g X_g beta_g (L287) and X^T theta = concat_g X_g^T theta (E7)."""
    prob = datagen.make("c2", n=64, p=101)
    d = oracle.Design.from_problem(prob)
    rng = np.random.default_rng(4)
    th, be = rng.normal(size=prob.n), rng.normal(size=prob.p + 1)
    full_s, full_g = oracle.fwdprod(d, be), oracle.backprod(d, th)
    for G in (1, 2, 5, 10):
        st = oracle.blocks(prob.p + 1, G)
        s = sum(oracle.fwdprod(d, be[st[g]:st[g + 1]], st[g], st[g + 1]) for g in range(G))
        gcat = np.concatenate([oracle.backprod(d, th, st[g], st[g + 1]) for g in range(G)])
        np.testing.assert_allclose(s, full_s, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(gcat, full_g)


def test_blocks_split_rule():
    """Contiguous near-equal blocks."""
    assert list(np.diff(oracle.blocks(10, 3))) == [4, 3, 3]
    assert list(np.diff(oracle.blocks(10, 1))) == [10]
    sz = np.diff(oracle.blocks(2001, 5))
    assert sz.sum() == 2001 and set(sz) <= {400, 401}


def test_zero_variance_column_rejected():
    X = np.zeros((3, 16), dtype=np.uint8)
    X[0, :8] = [0, 1, 2, 0, 1, 2, 0, 1]
    X[2, :8] = [1, 1, 0, 0, 1, 1, 0, 2]
    with pytest.raises(ValueError, match="column 1"):
        oracle.Design(1, 8, 3, 16, X)


# ----------------------------------------------------------------- power method (L259)

def test_power_vs_eigvalsh():
    for seed, (n, p) in enumerate([(60, 9), (200, 50), (40, 39), (120, 7)]):
        prob = datagen.make("c2", n=n, p=p, seed=100 + seed)
        d = oracle.Design.from_problem(prob)
        A, _, _ = _np_standardized(prob)
        st = oracle.blocks(p + 1, 3)
        for g in range(3):
            B = A[:, st[g]:st[g + 1]]
            ref = np.linalg.eigvalsh(B.T @ B)[-1]
            est, _ = oracle.power(d, int(st[g]), int(st[g + 1]), tol=1e-12, maxit=100000)
            assert est == pytest.approx(ref, rel=1e-6)


def test_power_closed_forms():
    """identity block -> 1; rank-one block u v^T -> ||u||^2 ||v||^2."""
    n, p = 8, 5
    X = np.zeros((p, 8), dtype=np.float32)
    for c in range(p):
        X[c, c] = 1.0
    d = oracle.Design(0, n, p, 8, X, mean=np.zeros(p), sd=np.ones(p))
    est, _ = oracle.power(d, 1, p + 1, tol=1e-14, maxit=1000)
    assert est == pytest.approx(1.0, rel=1e-12)
    u = np.array([1, 2, 0, -1, 3, 0, 1, 1], dtype=np.float64)
    v = np.array([0.5, -1, 2, 1, 0.25])
    X = np.outer(v, u).astype(np.float32)
    d = oracle.Design(0, n, p, 8, X, mean=np.zeros(p), sd=np.ones(p))
    est, _ = oracle.power(d, 1, p + 1, tol=1e-14, maxit=1000)
    uu = X[0].astype(np.float64) / v[0]
    assert est == pytest.approx(np.dot(uu, uu) * np.dot(v, v), rel=1e-6)


def test_tridiag_max_eig_vs_eigvalsh():
    rng = np.random.default_rng(5)
    for k in (1, 2, 3, 7, 20, 60):
        a = rng.normal(size=k) * 3
        b = rng.normal(size=k - 1)
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        assert oracle.tridiag_max_eig(a, b) == pytest.approx(np.linalg.eigvalsh(T)[-1], rel=1e-13, abs=1e-13)


def test_lanczos_vs_eigvalsh_and_power():
    """Lanczos (L259) reaches the largest eigenvalue of X~_g^T X~_g far sooner than the power method;
    its Ritz value never exceeds Lambda_max (interlacing)."""
    for seed, (n, p) in enumerate([(60, 9), (200, 50), (40, 39), (120, 7), (300, 240)]):
        prob = datagen.make("c2", n=n, p=p, seed=100 + seed)
        d = oracle.Design.from_problem(prob)
        A, _, _ = _np_standardized(prob)
        st = oracle.blocks(p + 1, 3)
        for g in range(3):
            B = A[:, st[g]:st[g + 1]]
            ref = np.linalg.eigvalsh(B.T @ B)[-1]
            est, it = oracle.lanczos(d, int(st[g]), int(st[g + 1]), tol=1e-12, maxit=1000)
            assert est == pytest.approx(ref, rel=1e-9)
            for k in (1, 2, 3):
                e_k, _ = oracle.lanczos(d, int(st[g]), int(st[g + 1]), tol=0.0, maxit=k)
                assert e_k <= ref * (1 + 1e-12)
            e4, it4 = oracle.lanczos(d, int(st[g]), int(st[g + 1]), tol=1e-4, maxit=1000)
            p4, ip4 = oracle.power(d, int(st[g]), int(st[g + 1]), tol=1e-4, maxit=1000)
            assert abs(e4 - ref) <= 1e-3 * ref
            assert it4 <= ip4


def test_lanczos_closed_forms():
    """identity block -> 1 after one step (beta_1 = 0); rank-one block -> ||u||^2 ||v||^2 after at most two
    (the Krylov space of a rank-one matrix has dimension 2)."""
    n, p = 8, 5
    X = np.zeros((p, 8), dtype=np.float32)
    for c in range(p):
        X[c, c] = 1.0
    d = oracle.Design(0, n, p, 8, X, mean=np.zeros(p), sd=np.ones(p))
    est, it = oracle.lanczos(d, 1, p + 1, tol=1e-14, maxit=1000)
    assert est == pytest.approx(1.0, rel=1e-12) and it == 1
    u = np.array([1, 2, 0, -1, 3, 0, 1, 1], dtype=np.float64)
    v = np.array([0.5, -1, 2, 1, 0.25])
    X = np.outer(v, u).astype(np.float32)
    d = oracle.Design(0, n, p, 8, X, mean=np.zeros(p), sd=np.ones(p))
    est, it = oracle.lanczos(d, 1, p + 1, tol=1e-14, maxit=1000)
    uu = X[0].astype(np.float64) / v[0]
    assert est == pytest.approx(np.dot(uu, uu) * np.dot(v, v), rel=1e-12) and it <= 2


# ----------------------------------------------------------------- solver pins

def _tiny(seed, n=12, p=3, tau=0.5):
    prob = datagen.make("c2", n=n, p=p, seed=seed)
    d = oracle.Design.from_problem(prob)
    return prob, d


@pytest.mark.parametrize("seed,tau,lfrac", [(11, 0.5, 0.3), (12, 0.3, 0.1), (13, 0.7, 0.6), (14, 0.5, 0.0),
                                            (15, 0.2, 0.05)])
def test_solver_matches_lp_bruteforce(seed, tau, lfrac):
    """FS-QRPPA converged objective == exact PQR optimum by vertex enumeration; HiGHS agrees."""
    prob, d = _tiny(seed, tau=tau)
    A, _, _ = _np_standardized(prob)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, lfrac * lm)
    G, mu = 2, 0.1
    eta = oracle.eta(d, G, mu)
    out = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=400000, tol=1e-11)
    assert out["status"] == 0
    fstar, _ = lp.vertex_enumeration(A, prob.y, tau, lam)
    fh, _ = lp.highs(A, prob.y, tau, lam)
    assert fh == pytest.approx(fstar, rel=1e-9, abs=1e-12)
    assert out["obj"] == pytest.approx(fstar, rel=1e-8, abs=1e-12)
    assert lp.pqr_objective(A, prob.y, tau, lam, out["beta"]) == pytest.approx(fstar, rel=1e-8, abs=1e-12)


def test_kkt_certificate_and_fixed_point():
    """Prop. 1: the converged state is a saddle point; a KKT point is a fixed point of one iteration."""
    prob = datagen.make("c2", n=40, p=60, seed=21)
    d = oracle.Design.from_problem(prob)
    tau = 0.3
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, 0.2 * lm)
    G, mu = 5, 0.01
    eta = oracle.eta(d, G, mu)
    out = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=400000, tol=1e-10)
    assert out["status"] == 0
    cert = oracle.kkt_cert(d, prob.y, tau, lam, out["beta"], out["z"], out["theta"])
    assert cert.max() < 1e-6
    st = (out["beta"], out["z"], out["theta"])
    one = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False, state=st)
    for a, b in zip(st, (one["beta"], one["z"], one["theta"])):
        assert np.max(np.abs(a - b)) < 1e-8


def _kkt_example():
    c = GOLD["kkt_example"]
    X = np.zeros((1, 16), np.uint8)
    X[0, :3] = [0, 1, 2]
    d = oracle.Design(1, 3, 1, 16, X)
    return c, d


def test_kkt_rel_hand_example():
    """R = (R_p, R_beta, R_z) of reading R1 on a 3-observation example derived by hand
    (tests/golden/worked_values.json "kkt_example"): pins every normalisation term."""
    c, d = _kkt_example()
    np.testing.assert_allclose(d.mean, [1.0])
    np.testing.assert_allclose(d.sd, [1.0])
    R = oracle.kkt_rel(d, c["y"], c["tau"], c["lam"], c["beta"], c["z"], c["theta"])
    np.testing.assert_allclose(R, c["expect_R"], rtol=1e-14)


def test_kkt_cert_hand_example_negative():
    """The Prop. 1 certificate is not trivially zero: at the (non-optimal) hand example it returns
    the violations derived by hand."""
    c, d = _kkt_example()
    cert = oracle.kkt_cert(d, c["y"], c["tau"], c["lam"], c["beta"], c["z"], c["theta"])
    np.testing.assert_allclose(cert, c["expect_cert"], rtol=1e-14)


@pytest.mark.parametrize("seed,tau,lfrac", [(31, 0.5, 0.2), (32, 0.25, 0.1), (33, 0.8, 0.4)])
def test_kkt_zero_at_lp_saddle_point(seed, tau, lfrac):
    """At the LP optimum with theta* from the LP's equality duals (an exact saddle point of
    Prop. 1), R(w*) vanishes and the certificate is zero; moving one inactive coefficient off zero
    by delta gives exactly the violations that move predicts."""
    prob, d = _tiny(seed, n=30, p=40, tau=tau)
    A, _, _ = _np_standardized(prob)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, lfrac * lm)
    beta, z, theta = lp.highs_saddle(A, prob.y, tau, lam)
    assert np.all(theta >= (tau - 1) / prob.n - 1e-12) and np.all(theta <= tau / prob.n + 1e-12)
    R = oracle.kkt_rel(d, prob.y, tau, lam, beta, z, theta)
    assert R.max() <= 1e-9, R
    cert = oracle.kkt_cert(d, prob.y, tau, lam, beta, z, theta)
    assert cert.max() <= 1e-9, cert
    g = A.T @ theta
    inactive = [j for j in range(1, prob.p + 1) if beta[j] == 0.0 and abs(g[j]) < lam[j] - 1e-9]
    assert inactive
    j, delta = inactive[0], 1e-3
    b2 = beta.copy()
    b2[j] = delta
    cert2 = oracle.kkt_cert(d, prob.y, tau, lam, b2, z, theta)
    assert cert2[0] == pytest.approx(delta * np.abs(A[:, j]).max(), rel=1e-6)   # z = y - X~beta broken
    assert cert2[1] == pytest.approx(max(cert[1], abs(g[j] - lam[j])), rel=1e-6)   # g_j != lam_j sign(beta_j)
    R2 = oracle.kkt_rel(d, prob.y, tau, lam, b2, z, theta)
    # R_p: ||X~_j delta|| / (1 + ||y||); R_beta: the moved coordinate is pulled back to S_lam(delta + g_j) = 0
    assert R2[0] == pytest.approx(delta * np.linalg.norm(A[:, j]) / (1 + np.linalg.norm(prob.y)), rel=1e-5)
    bb, gg = np.linalg.norm(b2), np.linalg.norm(g)
    assert R2[1] == pytest.approx(delta / (1 + bb + gg), rel=1e-5)


def test_lambda_max_null_model():
    """At lambda >= lambda_max the solution is beta_{1..p} = 0 with intercept = the sample
    tau-quantile (textbook); just below it, some beta_j != 0."""
    prob = datagen.make("c2", n=101, p=40, seed=31)
    d = oracle.Design.from_problem(prob)
    G, mu = 4, 0.02
    eta = oracle.eta(d, G, mu)
    for tau in (0.5, 0.25):
        lm, q = oracle.lambda_max(d, prob.y, tau)
        assert q == np.sort(prob.y)[int(np.ceil(101 * tau)) - 1]
        out = oracle.solve(d, prob.y, tau, oracle.lam_vector(prob.p, 1.01 * lm), eta, mu, G,
                           max_iter=300000, tol=1e-10)
        assert out["status"] == 0
        assert np.all(out["beta"][1:] == 0.0)
        assert out["beta"][0] == pytest.approx(q, abs=1e-6)
        u = prob.y - q
        assert out["obj"] == pytest.approx(np.mean(np.where(u < 0, (tau - 1) * u, tau * u)), rel=1e-7)
        if tau == 0.5:  # mean |y - median| / 2
            assert out["obj"] == pytest.approx(np.mean(np.abs(prob.y - np.median(prob.y))) / 2, rel=1e-7)
        out = oracle.solve(d, prob.y, tau, oracle.lam_vector(prob.p, 0.9 * lm), eta, mu, G,
                           max_iter=300000, tol=1e-10)
        assert np.count_nonzero(out["beta"][1:]) >= 1


def test_partition_invariance_solution():
    """Theorem 1: the limit is a saddle point for every G."""
    prob = datagen.make("c2", n=50, p=70, seed=41)
    d = oracle.Design.from_problem(prob)
    tau = 0.5
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, 0.3 * lm)
    objs, preds = [], []
    for G in (1, 2, 5, 10):
        mu = 0.03
        eta = oracle.eta(d, G, mu)
        out = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=400000, tol=1e-9)
        assert out["status"] == 0
        objs.append(out["obj"])
        preds.append(oracle.fwdprod(d, out["beta"]))
    for o, s in zip(objs[1:], preds[1:]):
        assert o == pytest.approx(objs[0], rel=1e-6)
        np.testing.assert_allclose(s, preds[0], atol=1e-5)


def test_geometric_decay():
    """Corollary 1: dist(w^k, w_final) is dominated by a geometric sequence;
    over the last 50 pre-stop iterations the log-distance slope is negative and the median
    successive ratio <= 0.999."""
    prob = datagen.make("c2", n=50, p=60, seed=51)
    d = oracle.Design.from_problem(prob)
    tau = 0.5
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, 0.3 * lm)
    G, mu = 3, 0.05
    eta = oracle.eta(d, G, mu)
    fin = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=400000, tol=1e-12)
    assert fin["status"] == 0
    K = fin["iters"]
    k0 = max(K - 60, 0)
    w_fin = np.concatenate([fin["beta"], fin["z"], fin["theta"]])
    base = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=k0, check=False)
    st = (base["beta"], base["z"], base["theta"])
    dists = []
    for _ in range(50):
        dists.append(np.linalg.norm(np.concatenate(st) - w_fin))
        o = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False, state=st)
        st = (o["beta"], o["z"], o["theta"])
    dd = np.array(dists[-50:])
    dd = dd[dd > 0]
    slope = np.polyfit(np.arange(len(dd)), np.log(dd), 1)[0]
    assert slope < 0
    assert np.median(dd[1:] / dd[:-1]) <= 0.999


def test_thread_count_determinism():
    """Fixed per-element summation order: bitwise-identical results for 1 and 4 threads."""
    code = (
        "import datagen, oracle, numpy as np;"
        "pr=datagen.make('c2', n=70, p=130, seed=61); d=oracle.Design.from_problem(pr);"
        "lm,_=oracle.lambda_max(d, pr.y, 0.5); lam=oracle.lam_vector(pr.p, 0.2*lm);"
        "eta=oracle.eta(d, 3, 0.05);"
        "o=oracle.solve(d, pr.y, 0.5, lam, eta, 0.05, 3, max_iter=300, check=False);"
        "print(np.concatenate([o['beta'],o['z'],o['theta'],eta]).tobytes().hex())"
    )
    root = os.path.dirname(HERE)
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=root)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert outs[0] == outs[1]


def test_path_warm_start_semantics():
    """Warm-started path (L412): point t equals a cold solve at lam_t in objective (convex problem),
    and the path's lambda_max end point is the null model."""
    prob = datagen.make("c2", n=60, p=80, seed=71)
    d = oracle.Design.from_problem(prob)
    tau, G, mu = 0.5, 3, 0.03
    eta = oracle.eta(d, G, mu)
    lm, q = oracle.lambda_max(d, prob.y, tau)
    lam_path = lm * 1.01 * (0.5 ** (np.arange(4) / 3))
    res = oracle.path(d, prob.y, tau, lam_path, eta, mu, G, tol=1e-9, max_iter_point=300000)
    assert res["converged"].all()
    assert np.all(res["beta_path"][0, 1:] == 0)
    for t in range(4):
        cold = oracle.solve(d, prob.y, tau, oracle.lam_vector(prob.p, lam_path[t]), eta, mu, G,
                            max_iter=300000, tol=1e-9)
        assert cold["status"] == 0
        assert res["obj"][t] == pytest.approx(cold["obj"], rel=1e-6)


def test_path_is_chained_warm_solves():
    """Reading R10 (L412, "the solution from the preceding lambda serves as the initialization"):
    point t+1 of the path starts from the iterate recorded as point t, so the path equals a chain
    of Algorithm-1 solves, each started from the previous one's output -- same update counts and
    bitwise-identical solutions, including points capped by max_iter_point."""
    prob = datagen.make("c2", n=50, p=70, seed=73)
    d = oracle.Design.from_problem(prob)
    tau, G, mu = 0.3, 4, 0.04
    eta = oracle.eta(d, G, mu)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam_path = lm * 1.01 * (0.05 ** (np.arange(5) / 4))
    cap = 400
    res = oracle.path(d, prob.y, tau, lam_path, eta, mu, G, tol=1e-6, max_iter_point=cap)
    state = None
    for t in range(5):
        o = oracle.solve(d, prob.y, tau, oracle.lam_vector(prob.p, lam_path[t]), eta, mu, G, max_iter=cap,
                         tol=1e-6, state=state)
        assert res["iters"][t] == o["iters"], t
        assert res["converged"][t] == (o["status"] == 0)
        np.testing.assert_array_equal(res["beta_path"][t], o["beta"])
        state = (o["beta"], o["z"], o["theta"])
    assert res["total"] == res["iters"].sum()
    assert not res["converged"].all()     # the cap closed at least one point
    np.testing.assert_array_equal(res["beta"], state[0])


# ----------------------------------------------------------------- Section 5 (LLA) and HBIC pins

@pytest.mark.parametrize("case", GOLD["penalty_deriv"])
def test_penalty_deriv_worked_values(case):
    assert oracle.penalty_deriv(case["kind"], case["a"], case["lam"], case["b"]) == pytest.approx(case["expect"],
                                                                                                 abs=1e-15)


@pytest.mark.parametrize("kind,a", [(oracle.SCAD, 3.7), (oracle.SCAD, 2.5), (oracle.MCP, 3.0), (oracle.MCP, 1.5)])
def test_penalty_deriv_shape(kind, a):
    """E16/E17: continuous at the knots, even in b, non-increasing in |b|, lam at 0, 0 beyond a*lam."""
    lam = 0.8
    b = np.linspace(0, 1.2 * a * lam, 2001)
    d = np.array([oracle.penalty_deriv(kind, a, lam, v) for v in b])
    assert d[0] == pytest.approx(lam)
    assert np.all(np.diff(d) <= 1e-15)
    assert np.all(d >= 0) and d[-1] == 0.0
    assert np.max(np.abs(np.diff(d))) < 2 * lam * (b[1] - b[0]) / min(a - 1.0, 1.0) + 1e-12   # no jumps
    for v in (0.3, 1.1, 2.9):
        assert oracle.penalty_deriv(kind, a, lam, -v) == oracle.penalty_deriv(kind, a, lam, v)
    w = oracle.lla_weights(kind, a, lam, np.array([5.0, 0.0, 0.5 * lam, -10 * a * lam]))
    assert w[0] == 0.0 and w[1] == 1.0 and w[3] == 0.0


@pytest.mark.parametrize("case", GOLD["hbic"])
def test_hbic_worked_value(case):
    v = oracle.hbic_value(case["loss"], case["active"], case["n"], case["p"])
    assert v == pytest.approx(case["expect"], abs=case["tol"])


def test_hbic_null_model_closed_form():
    prob = datagen.make("c2", n=50, p=8, seed=31)
    d = oracle.Design.from_problem(prob)
    beta = np.zeros(prob.p + 1)
    beta[0] = np.median(prob.y)
    loss = np.sum(np.where(prob.y - beta[0] < 0, -0.5 * (prob.y - beta[0]), 0.5 * (prob.y - beta[0])))
    assert oracle.hbic(d, prob.y, 0.5, beta) == pytest.approx(np.log(loss), rel=1e-12)
    beta[[2, 5]] = [0.1, -0.2]
    act_term = 2 * np.log(np.log(50)) / 50 * np.log(8)
    A, _, _ = _np_standardized(prob)
    u = prob.y - A @ beta
    loss2 = np.sum(np.where(u < 0, -0.5 * u, 0.5 * u))
    assert oracle.hbic(d, prob.y, 0.5, beta) == pytest.approx(np.log(loss2) + act_term, rel=1e-10)


@pytest.mark.parametrize("kind,a,seed", [(oracle.SCAD, 3.7, 41), (oracle.MCP, 3.0, 42)])
def test_lla_stages_are_weighted_l1_optima(kind, a, seed):
    """Algorithm 2: every stage l is the weighted-l1 PQR with lam_j = p'_lam(|beta~^{l-1}_j|); its
    converged objective equals the exact optimum of that weighted problem (vertex enumeration)."""
    prob, d = _tiny(seed, n=14, p=3)
    A, _, _ = _np_standardized(prob)
    tau = 0.5
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = 0.4 * lm
    G, mu = 2, 0.1
    eta = oracle.eta(d, G, mu)
    out = oracle.lla(d, prob.y, tau, lam, kind, a, 2, eta, mu, G, tol=1e-11, max_iter=400000)
    assert len(out["stages"]) == 3
    prev = None
    for l, st in enumerate(out["stages"]):
        assert st["status"] == 0
        if l == 0:
            assert np.all(st["weights"][1:] == 1.0)
        else:
            np.testing.assert_array_equal(st["weights"], oracle.lla_weights(kind, a, lam, prev))
        lv = oracle.lam_vector(prob.p, lam, st["weights"])
        fstar, _ = lp.vertex_enumeration(A, prob.y, tau, lv)
        assert st["obj"] == pytest.approx(fstar, rel=1e-8, abs=1e-12)
        prev = st["beta"]
    # the concave penalty lightens the shrinkage of large coefficients: stage weights <= 1
    assert np.all(out["stages"][1]["weights"] <= 1.0)


# ----------------------------------------------------------------- pivotal statistic (L412, reading R18)

def test_splitmix_reference_outputs():
    g = GOLD["splitmix64"]
    for st, ex in zip(g["state"], g["expect"]):
        st = int(st, 16) if isinstance(st, str) else st
        assert oracle.splitmix(st) == int(ex, 16)


def test_pivotal_draws_are_bernoulli_tau():
    for tau in (0.1, 0.5, 0.9):
        u = np.array([[oracle.piv_uniform(77, b, i) for i in range(500)] for b in range(40)])
        assert np.all((u >= 0) & (u < 1))
        f = np.mean(u <= tau)
        assert abs(f - tau) < 4 * np.sqrt(tau * (1 - tau) / u.size)


def test_pivotal_second_moment_single_column():
    """p = 1: (n Lambda_b)^2 = (x~^T psi_b)^2 with E psi = 0, Var psi = tau(1-tau), sum x~^2 = n-1,
    so its mean over replicates is tau(1-tau)(n-1) (law of large numbers, ~2% sd at B = 4000)."""
    prob = datagen.make("c2", n=300, p=1, seed=51)
    d = oracle.Design.from_problem(prob)
    tau = 0.3
    L = oracle.pivotal(d, tau, 4000, seed=9)
    m2 = np.mean((prob.n * L) ** 2)
    assert m2 == pytest.approx(tau * (1 - tau) * (prob.n - 1), rel=0.1)


def test_pivotal_invariances():
    """Recoding every genotype as 2 - x flips the sign of x~ (|.| unchanged); permuting the
    columns leaves the maximum unchanged."""
    prob = datagen.make("c2", n=200, p=30, seed=52)
    d = oracle.Design.from_problem(prob)
    L = oracle.pivotal(d, 0.6, 50, seed=3)
    Xr = prob.X.copy()
    Xr[:, :prob.n] = 2 - Xr[:, :prob.n]
    dr = oracle.Design(prob.storage, prob.n, prob.p, prob.ld, Xr)
    np.testing.assert_allclose(oracle.pivotal(dr, 0.6, 50, seed=3), L, rtol=1e-12)
    perm = np.random.default_rng(0).permutation(prob.p)
    dp = oracle.Design(prob.storage, prob.n, prob.p, prob.ld, np.ascontiguousarray(prob.X[perm]))
    np.testing.assert_array_equal(oracle.pivotal(dp, 0.6, 50, seed=3), L)
    assert oracle.pivotal_lambda(L, 0.1, 1.1) == pytest.approx(1.1 * np.sort(L)[44])


# ----------------------------------------------------------------- elastic net (Remark 3, reading R19)

def test_prox_en_bruteforce_and_lasso_limit():
    """argmin_b lam1|b| + (lam2/2) b^2 - g b + (eta/2)(b - beta)^2 (the weighted elastic-net block
    prox); with lam2 = 0 it is E14 bit for bit."""
    rng = np.random.default_rng(3)
    for _ in range(60):
        beta, g = rng.normal(), rng.normal()
        lam1, lam2, eta = abs(rng.normal()) * rng.choice([0, 0.3, 1]), rng.uniform(0, 3), rng.uniform(0.2, 5)
        f = lambda b: lam1 * abs(b) + 0.5 * lam2 * b * b - g * b + 0.5 * eta * (b - beta) ** 2
        assert oracle.prox_en(beta, g, lam1, lam2, eta) == pytest.approx(_argmin_1d(f, -20, 20), abs=1e-7)
        assert oracle.prox_en(beta, g, lam1, 0.0, eta) == oracle.prox_beta(beta, g, lam1, eta)


@pytest.mark.parametrize("seed,tau,lam2", [(61, 0.5, 0.3), (62, 0.25, 1.0)])
def test_elastic_net_solve_matches_qp(seed, tau, lam2):
    """Algorithm 1 with the elastic-net prox converges to the optimum of
    (1/n) sum rho_tau + sum lam_j |b_j| + (lam2/2) sum_{j>=1} b_j^2, solved independently as a
    smooth QP (u, v, a, b >= 0 split) by SLSQP on a tiny instance."""
    from scipy.optimize import minimize

    prob, d = _tiny(seed, n=12, p=3)
    A, _, _ = _np_standardized(prob)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, 0.2 * lm)
    G, mu = 2, 0.1
    eta = oracle.eta(d, G, mu)
    out = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=400000, tol=1e-11, lam2=lam2)
    assert out["status"] == 0
    n, p = prob.n, prob.p
    # variables: beta0, a (p), b (p), u (n), v (n)
    def f(x):
        a, b, u, v = x[1:1 + p], x[1 + p:1 + 2 * p], x[1 + 2 * p:1 + 2 * p + n], x[1 + 2 * p + n:]
        return (tau * u.sum() + (1 - tau) * v.sum()) / n + np.sum(lam[1:] * (a + b)) + 0.5 * lam2 * np.sum((a - b) ** 2)
    def eq(x):
        beta = np.concatenate([[x[0]], x[1:1 + p] - x[1 + p:1 + 2 * p]])
        return prob.y - A @ beta - (x[1 + 2 * p:1 + 2 * p + n] - x[1 + 2 * p + n:])
    x0 = np.zeros(1 + 2 * p + 2 * n)
    x0[1 + 2 * p:1 + 2 * p + n] = np.maximum(prob.y, 0)
    x0[1 + 2 * p + n:] = np.maximum(-prob.y, 0)
    res = minimize(f, x0, method="SLSQP", constraints=[{"type": "eq", "fun": eq}],
                   bounds=[(None, None)] + [(0, None)] * (2 * p + 2 * n), options=dict(ftol=1e-14, maxiter=2000))
    assert res.success
    assert out["obj"] == pytest.approx(res.fun, rel=1e-6, abs=1e-10)
    assert oracle.objective_en(d, prob.y, tau, lam, lam2, out["beta"]) == pytest.approx(out["obj"], rel=1e-12)


# ----------------------------------------------------------------- the trajectory itself (Theorem 1)

def _H_norm2(A, eta_cols, mu, sigma, dbeta, dz, dtheta):
    """||(du, dtheta)||_H^2 with H = [[T, A^T], [A, I/sigma]], u = (beta, z), A u = X~ beta + z,
    T = diag(eta_{g(j)} I, mu I): the metric in which Algorithm 1 is a proximal point method,
    0 in F(w^{k+1}) + H (w^{k+1} - w^k) with F the (monotone) KKT operator of Prop. 1 (L319-336;
    derivation in SURVEY §8(c), App. E is missing)."""
    Au = A @ dbeta + dz
    return (np.sum(eta_cols * dbeta * dbeta) + mu * np.dot(dz, dz) + 2.0 * np.dot(dtheta, Au)
            + np.dot(dtheta, dtheta) / sigma)


@pytest.mark.parametrize("seed,tau,G", [(71, 0.5, 3), (72, 0.2, 5), (73, 0.8, 1)])
def test_trajectory_is_fejer_monotone_in_H(seed, tau, G):
    """Theorem 1: the iterates of Algorithm 1 satisfy, for a solution w*,
        ||w^{k+1} - w*||_H^2 <= ||w^k - w*||_H^2 - ||w^{k+1} - w^k||_H^2,
    a property of the whole composed step (E12-E15 in Algorithm 1's order): a dropped term, a
    wrong sign in the dual step or a wrong prox scale breaks it.  Checked on every iteration of
    a 300-step trajectory against a solution converged to 1e-12; H is built from the design
    independently of the oracle (numpy), and H > 0 is asserted first (eta_g > mu Lambda_max)."""
    prob = datagen.make("c2", n=40, p=30, seed=seed)
    d = oracle.Design.from_problem(prob)
    A, _, _ = _np_standardized(prob)
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = oracle.lam_vector(prob.p, 0.25 * lm)
    mu = 2.0 / prob.n
    eta = oracle.eta(d, G, mu)
    st = oracle.blocks(prob.p + 1, G)
    eta_cols = np.concatenate([np.full(st[g + 1] - st[g], eta[g]) for g in range(G)])
    sigma = mu / (G + 1)
    n, p1 = A.shape
    H = np.zeros((p1 + 2 * n, p1 + 2 * n))
    H[:p1, :p1] = np.diag(eta_cols)
    H[p1:p1 + n, p1:p1 + n] = mu * np.eye(n)
    Au = np.hstack([A, np.eye(n)])
    H[p1 + n:, :p1 + n] = Au
    H[:p1 + n, p1 + n:] = Au.T
    H[p1 + n:, p1 + n:] = np.eye(n) / sigma
    assert np.linalg.eigvalsh(H).min() > 0
    fin = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=2_000_000, tol=1e-12)
    assert fin["status"] == 0
    ws = (fin["beta"], fin["z"], fin["theta"])
    state = None
    prev = None
    scale = None
    for k in range(300):
        o = oracle.solve(d, prob.y, tau, lam, eta, mu, G, max_iter=1, check=False, state=state)
        cur = (o["beta"], o["z"], o["theta"])
        if state is None:
            state = (np.zeros(p1), prob.y.copy(), np.zeros(n))
        dk = _H_norm2(A, eta_cols, mu, sigma, *(a - b for a, b in zip(state, ws)))
        dk1 = _H_norm2(A, eta_cols, mu, sigma, *(a - b for a, b in zip(cur, ws)))
        step = _H_norm2(A, eta_cols, mu, sigma, *(a - b for a, b in zip(cur, state)))
        if scale is None:
            scale = dk
        assert step >= -1e-12 * scale
        assert dk1 <= dk - step + 1e-9 * scale, (k, dk, dk1, step)
        state = cur
