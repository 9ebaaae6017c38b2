"""GPU parity for SURVEY §8(f) NEXT #1-#2 built on the hot path: per-coefficient penalty weights
(weighted l1, E4), the L-step LLA for SCAD / MCP (Algorithm 2) and HBIC (E18,
L408-411).  Expected values come from the fp64 oracle on the same seeded inputs."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import rel, to_device

pytestmark = pytest.mark.gpu


def _setup(n=800, p=2000, tau=0.5, lam_frac=0.1, storage=None, name="c2", tol=1e-6):
    import paper_2601_02826_b200 as fs

    prob = datagen.make(name, n=n, p=p, storage=storage)
    d = oracle.Design.from_problem(prob)
    mu, G = 2.0 / prob.n, 5
    eta = oracle.eta(d, G, mu)
    lam = lam_frac * oracle.lambda_max(d, prob.y, tau)[0]
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [lam], G=G, mu=mu, eta=eta, tol=tol,
                  max_iter=200000)
    return prob, d, S, dict(mu=mu, G=G, eta=eta, lam=lam, tau=tau)


def test_weighted_l1_fixed_iterations(cuda_ok):
    """Random non-negative weights (a tenth of them zero: unpenalised coefficients)."""
    prob, d, S, c = _setup()
    rng = np.random.default_rng(5)
    w = rng.uniform(0.2, 3.0, prob.p + 1)
    w[rng.choice(prob.p, prob.p // 10, replace=False) + 1] = 0.0
    S.set_lambda_weights(w[None, :])
    S.iterate(150)
    b, z, t = S.state()
    lv = oracle.lam_vector(prob.p, c["lam"], w)
    o = oracle.solve(d, prob.y, c["tau"], lv, c["eta"], c["mu"], c["G"], max_iter=150, check=False)
    assert rel(b[0], o["beta"]) < 1e-6
    assert rel(t[0], o["theta"]) < 1e-6
    assert np.array_equal(b[0] != 0, o["beta"] != 0)
    assert S.objective()[0] == pytest.approx(oracle.objective(d, prob.y, c["tau"], lv, o["beta"]), rel=1e-6)
    # unit weights restored: identical to a fresh unweighted run of the same length from this state
    S.set_lambda_weights(None)


@pytest.mark.parametrize("kind,a", [(1, 3.7), (2, 3.0)])
def test_one_step_lla_matches_oracle(cuda_ok, kind, a):
    """The paper's protocol (one-step LLA, a = 3.7 SCAD / 3 MCP, L404) on the C2 recipe at reduced
    size: per-stage iteration counts, the final beta, support and weighted objective agree."""
    prob, d, S, c = _setup(storage=None)
    res = S.lla(kind, a, 1)
    assert res["status"] == 0, res
    o = oracle.lla(d, prob.y, c["tau"], c["lam"], kind, a, 1, c["eta"], c["mu"], c["G"], tol=1e-6, max_iter=200000)
    for l, st in enumerate(o["stages"]):
        assert st["status"] == 0
        assert abs(res["stage_iters"][l] - st["iters"]) <= 2, (l, res["stage_iters"], [s["iters"] for s in o["stages"]])
    b = S.beta()[0]
    assert rel(b, o["beta"]) < 1e-4
    assert np.array_equal(b != 0, o["beta"] != 0)
    lv = oracle.lam_vector(prob.p, c["lam"], o["stages"][-1]["weights"])
    assert S.objective()[0] == pytest.approx(oracle.objective(d, prob.y, c["tau"], lv, o["beta"]), rel=1e-4)
    # the stage-1 weights of the largest LASSO coefficients are below 1 (less shrinkage, L352)
    w1 = o["stages"][1]["weights"]
    big = np.argmax(np.abs(o["stages"][0]["beta"][1:])) + 1
    assert w1[big] < 1.0


def test_lla_on_two_bit_storage(cuda_ok):
    """Same driver on the 2-bit packed storage (C4 recipe, tensor-core kernel), MCP, L = 2."""
    prob, d, S, c = _setup(name="c4", n=522, p=1100, storage=2)   # (n = 700, p = 1500 took 150 s in the oracle)
    assert S.backend == "tc"
    res = S.lla(2, 3.0, 2)
    assert res["status"] == 0
    o = oracle.lla(d, prob.y, c["tau"], c["lam"], 2, 3.0, 2, c["eta"], c["mu"], c["G"], tol=1e-6, max_iter=200000)
    assert rel(S.beta()[0], o["beta"]) < 1e-4
    assert np.array_equal(S.beta()[0] != 0, o["beta"] != 0)


def test_hbic_matches_oracle(cuda_ok):
    prob, d, S, c = _setup(tau=0.3)
    res = S.solve()
    assert res["status"] == 0
    o = oracle.solve(d, prob.y, c["tau"], oracle.lam_vector(prob.p, c["lam"]), c["eta"], c["mu"], c["G"],
                     max_iter=200000, tol=1e-6)
    h = S.hbic()[0]
    ho = oracle.hbic(d, prob.y, c["tau"], o["beta"])
    assert h == pytest.approx(ho, rel=1e-6)


def test_lla_bad_arguments(cuda_ok):
    import paper_2601_02826_b200 as fs

    prob, d, S, c = _setup(n=200, p=300)
    for args in ((3, 3.7, 1), (1, 1.5, 1), (2, 0.9, 1), (1, 3.7, -1)):
        with pytest.raises(fs.FsqrError) as e:
            S.lla(*args)
        assert e.value.status == -1
    bad = np.ones((1, prob.p + 1))
    bad[0, 3] = -1.0
    with pytest.raises(fs.FsqrError):
        S.set_lambda_weights(bad)


@pytest.mark.parametrize("n,p,B,tau", [(1000, 3000, 300, 0.3), (777, 513, 129, 0.9)])
def test_pivotal_statistic_matches_oracle(cuda_ok, n, p, B, tau):
    """Lambda_b (L412, reading R18) on the tensor cores vs the oracle: ragged n (K tail), ragged p
    (N tail of the 256-column tiles) and a partial last pass of 128 replicates."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c5", n=n, p=p)
    d = oracle.Design.from_problem(prob)
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [0.1], G=5, eta=[1.0] * 5)
    L = S.pivotal(B, seed=1234)
    Lo = oracle.pivotal(d, tau, B, seed=1234)
    np.testing.assert_allclose(L, Lo, rtol=1e-10)
    assert oracle.pivotal_lambda(L) == pytest.approx(oracle.pivotal_lambda(Lo), rel=1e-10)


@pytest.mark.parametrize("storage,lam2", [(1, 0.5), (2, 2.0)])
def test_elastic_net_matches_oracle(cuda_ok, storage, lam2):
    """Weighted elastic net (Remark 3, reading R19): fixed iterations and convergence to KKT 1e-6."""
    name = "c2" if storage == 1 else "c4"
    prob, d, S, c = _setup(name=name, n=700, p=1600, storage=storage)
    S.set_lambda2([lam2])
    lv = oracle.lam_vector(prob.p, c["lam"])
    S.iterate(120)
    b, z, t = S.state()
    o = oracle.solve(d, prob.y, c["tau"], lv, c["eta"], c["mu"], c["G"], max_iter=120, check=False, lam2=lam2)
    assert rel(b[0], o["beta"]) < 1e-6
    assert rel(t[0], o["theta"]) < 1e-6
    assert np.array_equal(b[0] != 0, o["beta"] != 0)
    res = S.solve()
    assert res["status"] == 0
    oc = oracle.solve(d, prob.y, c["tau"], lv, c["eta"], c["mu"], c["G"], max_iter=200000, tol=1e-6, lam2=lam2,
                      state=(o["beta"], o["z"], o["theta"]))
    assert oc["status"] == 0
    bb = S.beta()[0]
    assert rel(bb, oc["beta"]) < 1e-4
    assert S.objective()[0] == pytest.approx(oracle.objective_en(d, prob.y, c["tau"], lv, lam2, oc["beta"]), rel=1e-4)


def test_path_hbic_and_tune_match_oracle(cuda_ok):
    """The paper's sparse-setting tuning (L406-412): warm-started geometric path, HBIC (E18) per
    point, argmin.  HBIC of every recorded point equals the oracle's HBIC of the oracle's point."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=600, p=1200)
    d = oracle.Design.from_problem(prob)
    tau, G, T, tol = 0.5, 5, 8, 1e-5
    mu = 2.0 / prob.n
    eta = oracle.eta(d, G, mu)
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [1.0], G=G, mu=mu, eta=eta, tol=tol,
                  max_iter_point=5000)
    out = S.tune(T=T, lam_min_frac=0.05)
    grid = out["grid"][0]
    o = oracle.path(d, prob.y, tau, grid, eta, mu, G, tol, 5000)
    ho = np.array([oracle.hbic(d, prob.y, tau, o["beta_path"][t]) for t in range(T)])
    np.testing.assert_allclose(out["hbic"][0], ho, rtol=1e-6)
    assert out["best"][0] == int(np.argmin(ho))
    assert rel(out["beta"][0], o["beta_path"][int(np.argmin(ho))]) < 1e-4


def test_tune_with_pivotal_grid(cuda_ok):
    """fsqr_tune with B > 0 (reading R20): lambda_piv = 1.1 x the ceil(0.9 B)-th order statistic of
    the pivotal statistic (reading R18; equal to the oracle's), the grid runs geometrically from
    max(lambda_max, lambda_piv) to lam_min_frac x min(lambda_max, lambda_piv), and HBIC of every
    point equals the oracle's HBIC of the oracle path on the same grid."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=500, p=1500)
    d = oracle.Design.from_problem(prob)
    tau, G, T, tol, B, frac = 0.5, 5, 6, 1e-5, 256, 0.2
    mu = 2.0 / prob.n
    eta = oracle.eta(d, G, mu)
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [1.0], G=G, mu=mu, eta=eta, tol=tol,
                  max_iter_point=5000)
    out = S.tune(T=T, lam_min_frac=frac, B=B, seed=99)
    lpiv = oracle.pivotal_lambda(oracle.pivotal(d, tau, B, seed=99), alpha=0.1, c=1.1)
    assert out["lam_piv"][0] == pytest.approx(lpiv, rel=1e-10)
    lm = oracle.lambda_max(d, prob.y, tau)[0]
    hi, lo = max(lm, lpiv), frac * min(lm, lpiv)
    np.testing.assert_allclose(out["grid"][0], hi * (lo / hi) ** (np.arange(T) / (T - 1)), rtol=1e-12)
    o = oracle.path(d, prob.y, tau, out["grid"][0], eta, mu, G, tol, 5000)
    ho = np.array([oracle.hbic(d, prob.y, tau, o["beta_path"][t]) for t in range(T)])
    np.testing.assert_allclose(out["hbic"][0], ho, rtol=1e-6)
    assert out["best"][0] == int(np.argmin(ho))
    assert rel(out["beta"][0], o["beta_path"][int(np.argmin(ho))]) < 1e-6
