"""GPU parity for the warm-started lambda path and the edge
cases of the method: empty support (lambda >= lambda_max), a single column, the maximum RHS
count (16 tau levels -> 64 digit rows of the tcgen05 B operand), ragged n, and p = 0 rejected.
Every expected value comes from the fp64 oracle on the same seeded inputs."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import make_pair, rel, to_device

pytestmark = pytest.mark.gpu


def test_path_matches_oracle(cuda_ok):
    """C5 recipe at reduced size: 3 tau jointly on the GPU, a 6-point geometric grid from
    lambda_max to 0.01 lambda_max with warm starts; per point the recorded iteration count,
    objective and beta agree with the oracle's path for that tau."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c5", n=500, p=1500)
    d = oracle.Design.from_problem(prob)
    taus = [0.1, 0.5, 0.9]
    mu, G, T, tol = 2.0 / prob.n, 5, 6, 1e-5
    eta = oracle.eta(d, G, mu)
    lm = [oracle.lambda_max(d, prob.y, t)[0] for t in taus]
    grid = np.array([[l * 0.01 ** (t / (T - 1)) for t in range(T)] for l in lm])
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, grid[:, 0], G=G, mu=mu, eta=eta, tol=tol,
                  max_iter_point=4000)
    res = S.path(grid)
    for r, tau in enumerate(taus):
        o = oracle.path(d, prob.y, tau, grid[r], eta, mu, G, tol, 4000)
        # reading R10 on both sides: identical update counts at every point
        np.testing.assert_array_equal(res["iters"][r], o["iters"], err_msg=f"tau={tau}")
        np.testing.assert_array_equal(res["converged"][r], o["converged"])
        np.testing.assert_allclose(res["obj"][r], o["obj"], rtol=1e-4)
        for t in range(T):
            bg = S.path_beta(r, t)
            bo = o["beta_path"][t]
            assert rel(bg, bo) < 1e-6, (tau, t)
            assert np.array_equal(bg != 0, bo != 0), (tau, t)
        # first point at lambda_max: (near-)null model on both sides
        assert np.count_nonzero(S.path_beta(r, 0)[1:]) == np.count_nonzero(o["beta_path"][0][1:]) <= 2
    # updates plus one shared re-test pass per lambda switch (the slowest RHS sets the pace)
    assert res["total"] >= res["iters"].sum(axis=1).max() + T - 1


def test_path_beta_ordered_and_deterministic(cuda_ok):
    """fsqr_path_beta returns each point's nonzeros in ascending coefficient index, and two runs of
    the same path give bitwise-identical stores (the compaction does not depend on scheduling)."""
    import ctypes

    import paper_2601_02826_b200 as fs

    prob = datagen.make("c5", n=400, p=3000)
    taus = [0.2, 0.5, 0.8]
    X, y = to_device(prob)
    runs = []
    for _ in range(2):
        S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, [1.0] * 3, G=5, tol=1e-4,
                      max_iter_point=3000)
        lm = S.lambda_max()
        grid = np.array([[l * 0.02 ** (t / 4) for t in range(5)] for l in lm])
        S.path(grid)
        pts = []
        for r in range(3):
            for t in range(5):
                cap = prob.p + 1
                idx = np.zeros(cap, np.int64)
                val = np.zeros(cap)
                cnt = ctypes.c_int64(0)
                fs._check(fs.load().fsqr_path_beta(S.ctx, r, t, cap, fs._ptr(idx), fs._ptr(val), ctypes.byref(cnt)))
                m = cnt.value
                assert np.all(np.diff(idx[:m]) > 0), (r, t)
                assert np.all(val[:m] != 0)
                pts.append((idx[:m].copy(), val[:m].copy()))
        runs.append(pts)
        del S
    for (i0, v0), (i1, v1) in zip(*runs):
        np.testing.assert_array_equal(i0, i1)
        np.testing.assert_array_equal(v0, v1)


def test_lambda_above_max_gives_null_model(cuda_ok):
    """Empty support every iteration (K1 sees |S| = 0): beta_{1..p} = 0 and the intercept is the
    sample tau-quantile (R4), as in the oracle."""
    prob, d, S, cfg = make_pair("c2", n=900, p=700, taus=[0.3], lam_frac=1.0)
    lam = 1.01 * cfg["lm"][0]
    S.set_lambda([lam])
    res = S.solve()
    assert res["status"] == 0
    b = S.beta()[0]
    assert np.count_nonzero(b[1:]) == 0
    # the pinball minimiser is the sample 0.3-quantile; n*tau = 270 is an integer, so every point of
    # [y_(270), y_(271)] minimises (the textbook non-uniqueness of the sample quantile)
    ys = np.sort(prob.y)
    k = int(np.ceil(prob.n * 0.3))
    lo, hi = ys[k - 1], ys[k] if prob.n * 0.3 == k else ys[k - 1]
    assert lo - 1e-4 <= b[0] <= hi + 1e-4
    o = oracle.solve(d, prob.y, 0.3, oracle.lam_vector(prob.p, lam), cfg["eta"], cfg["mu"], cfg["G"],
                     max_iter=100000, tol=1e-6)
    assert S.objective()[0] == pytest.approx(o["obj"], rel=1e-4)


@pytest.mark.parametrize("storage", [0, 1, 2])
def test_single_column_ragged_n(cuda_ok, storage):
    """p = 1, n = 37 (not a multiple of 4, 16 or 128): the smallest admissible problem."""
    name = "c1" if storage == 0 else "c2"
    prob, d, S, cfg = make_pair(name, n=37, p=1, storage=storage, G=1, taus=[0.5], lam_frac=0.05)
    S.iterate(100)
    b, z, t = S.state()
    o = oracle.solve(d, prob.y, 0.5, oracle.lam_vector(1, cfg["lams"][0]), cfg["eta"], cfg["mu"], 1, max_iter=100,
                     check=False)
    assert rel(b[0], o["beta"]) < 1e-6
    assert rel(t[0], o["theta"]) < 1e-6


def test_max_rhs_sixteen_tau(cuda_ok):
    """R = 16 (FSQR_MAXR): 64 digit rows in the tcgen05 B operand; each RHS equals its oracle run."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=640, p=900)
    d = oracle.Design.from_problem(prob)
    taus = list(np.linspace(0.05, 0.95, 16))
    mu, G = 2.0 / prob.n, 5
    eta = oracle.eta(d, G, mu)
    lams = [0.05 * oracle.lambda_max(d, prob.y, t)[0] for t in taus]
    X, y = to_device(prob)
    S = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, taus, lams, G=G, mu=mu, eta=eta)
    assert S.backend == "tc"
    S.iterate(40)
    b, z, t = S.state()
    for r in (0, 7, 15):
        o = oracle.solve(d, prob.y, taus[r], oracle.lam_vector(prob.p, lams[r]), eta, mu, G, max_iter=40, check=False)
        assert rel(b[r], o["beta"]) < 1e-6, r
        assert rel(t[r], o["theta"]) < 1e-6, r
        assert np.array_equal(b[r] != 0, o["beta"] != 0), r


def test_p_zero_and_too_many_rhs_rejected(cuda_ok):
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=64, p=10)
    X, y = to_device(prob)
    with pytest.raises(fs.FsqrError) as e:
        fs.Solver(X, 1, prob.n, 0, prob.ld, y, [0.5], [0.1], G=1)
    assert e.value.status == -1
    with pytest.raises(fs.FsqrError) as e:
        fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, [0.5] * 17, [0.1] * 17)
    assert e.value.status == -1


def test_converged_parity_c2_tau09(cuda_ok):
    """C2 recipe (reduced) run to KKT tol 1e-6 at tau = 0.9: iteration count, objective, beta and
    support agree with the oracle; the GPU point passes the oracle's fp64 certificate."""
    prob, d, S, cfg = make_pair("c2", n=1200, p=4000, taus=[0.9], tol=1e-6, max_iter=200000)
    res = S.solve()
    assert res["status"] == 0, res
    lv = oracle.lam_vector(prob.p, cfg["lams"][0])
    o = oracle.solve(d, prob.y, 0.9, lv, cfg["eta"], cfg["mu"], cfg["G"], max_iter=200000, tol=1e-6)
    assert o["status"] == 0
    assert abs(res["iterations"] - o["iters"]) <= 2
    b = S.beta()[0]
    assert rel(b, o["beta"]) < 1e-4
    assert S.objective()[0] == pytest.approx(o["obj"], rel=1e-4)
    assert np.array_equal(b != 0, o["beta"] != 0)
    _, z, t = S.state()
    assert oracle.kkt_rel(d, prob.y, 0.9, lv, b, z[0], t[0]).max() < 2e-6


@pytest.mark.parametrize("storage", [1, 2])
def test_unpenalised_full_support(cuda_ok, storage):
    """lambda = 0 with p + 1 < n: classical quantile regression (Koenker-Bassett, L57); every
    column is in the support, so the forward product streams all of X; the converged objective
    equals the oracle's."""
    name = "c2" if storage == 1 else "c4"
    prob, d, S, cfg = make_pair(name, n=300, p=12, storage=storage, G=2, taus=[0.35], lam_frac=0.0, tol=1e-7,
                                max_iter=400000)
    res = S.solve()
    assert res["status"] == 0, res
    o = oracle.solve(d, prob.y, 0.35, oracle.lam_vector(prob.p, 0.0), cfg["eta"], cfg["mu"], 2, max_iter=400000,
                     tol=1e-7)
    assert o["status"] == 0
    assert np.count_nonzero(S.beta()[0][1:]) == prob.p
    assert S.objective()[0] == pytest.approx(o["obj"], rel=1e-6)


@pytest.mark.parametrize("taus", [[0.5], [0.1, 0.25, 0.9]])
def test_lambda_max_with_tied_responses(cuda_ok, taus):
    """lambda_max (reading R4) when y has many ties, including at the quantile itself: the GPU ranks
    y over the whole grid (k_ranks, ties broken by index) and gives the tie group the score that makes
    sum(psi) = 0; it must equal the oracle's lambda_max and quantile, every tau, to 1e-10."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=1500, p=800)
    prob.y = np.round(prob.y, 1)          # ~130 distinct values over 1500 observations
    d = oracle.Design.from_problem(prob)
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, [1.0] * len(taus), G=prob.G)
    lm = S.lambda_max()
    for r, t in enumerate(taus):
        lo, q = oracle.lambda_max(d, prob.y, t)
        assert lm[r] == pytest.approx(lo, rel=1e-10, abs=1e-15), (t, lm[r], lo)
