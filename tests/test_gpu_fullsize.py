"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

Two kinds of checks (the task's "sampled outputs / properties that hold at any size"):

* Full trajectories against the fp64 oracle where the oracle finishes in tens of seconds:
  C2 (n=2000, p=50k, three tau solved jointly on the GPU and separately by the oracle, 200
  iterations) and the metric workload M (n=10k, p=1M, a few iterations from the cold start,
  every element of beta, z, theta compared).  eta comes from the ORACLE's power method.
* One-step properties at C3, C4 (2-bit) and C5 (9 RHS) full size after a burn-in: the GPU's
  step w^k -> w^{k+1}, launched exactly as bench.py launches it (fsqr_profile_iterate), must
  satisfy E14 on a random column sample plus every support column, E15 and E12 on every row.
  The checker here is plain numpy written from the paper's formulas (it does not call the
  oracle, whose inputs never come from the CUDA path).

Tolerances: north_star's 1e-5 for products (componentwise-scaled by sum_i |x~_ij theta_i|,
SURVEY §8(c) #16), 1e-4 for beta / objective (the exact-integer design gives ~1e-8), and
identical supports except coordinates within 1e-6 lambda of the threshold (§8(c) #17).
"""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import check_one_step, rel, to_device

pytestmark = [pytest.mark.gpu, pytest.mark.fullsize]


# ------------------------------------------------------------------ full trajectories vs the oracle

def test_c2_full_three_taus_trajectory(cuda_ok):
    """configs[1] at full size: the 3 quantile levels run jointly (R=3) on the GPU for 200
    iterations; each is compared with its own oracle run."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2")
    d = oracle.Design.from_problem(prob)
    mu, G = 2.0 / prob.n, prob.G
    eta = oracle.eta(d, G, mu)
    lams = [prob.lam_frac * oracle.lambda_max(d, prob.y, t)[0] for t in prob.taus]
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, prob.taus, lams, G=G, mu=mu, eta=eta)
    assert S.backend == "tc"
    S.iterate(199)
    fs.fsqr_profile_iterate(S.ctx, 1)
    b, z, t = S.state()
    obj = S.objective()
    for r, tau in enumerate(prob.taus):
        lv = oracle.lam_vector(prob.p, lams[r])
        o = oracle.solve(d, prob.y, tau, lv, eta, mu, G, max_iter=200, check=False)
        assert rel(b[r], o["beta"]) < 1e-6, tau
        assert rel(z[r], o["z"]) < 1e-6, tau
        assert rel(t[r], o["theta"]) < 1e-6, tau
        assert np.count_nonzero(o["beta"][1:]) > 10
        mism = np.flatnonzero((b[r] != 0) != (o["beta"] != 0))
        assert len(mism) == 0, (tau, mism[:10])
        assert obj[r] == pytest.approx(oracle.objective(d, prob.y, tau, lv, o["beta"]), rel=1e-4)


@pytest.mark.parametrize("pack", [False, True])
def test_m_full_trajectory(cuda_ok, pack):
    """The bench workload M (n=10k, p=1M, u8, G=48) at full size: 6 iterations from the cold
    start (the last one through bench.py's launch path), every element compared; streamed as
    u8, and repacked to 2 bits at create (FSQR_DESIGN_PACK2, bench.py's default layout)."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("m")
    d = oracle.Design.from_problem(prob)
    mu, G, tau = 2.0 / prob.n, prob.G, prob.taus[0]
    eta = oracle.eta(d, G, mu, maxit=4)          # a short power run: any eta > 0 is a valid parity input
    lm, _ = oracle.lambda_max(d, prob.y, tau)
    lam = prob.lam_frac * lm
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [lam], G=G, mu=mu, eta=eta,
                  flags=fs.DESIGN_PACK2 if pack else 0)
    assert S.backend == "tc"
    np.testing.assert_allclose(S.lambda_max()[0], lm, rtol=1e-10)
    k = 6
    S.iterate(k - 1)
    fs.fsqr_profile_iterate(S.ctx, 1)
    b, z, t = S.state()
    lv = oracle.lam_vector(prob.p, lam)
    o = oracle.solve(d, prob.y, tau, lv, eta, mu, G, max_iter=k, check=False)
    nnz = np.count_nonzero(o["beta"][1:])
    assert nnz > 100, nnz
    assert rel(b[0], o["beta"]) < 1e-6
    assert rel(z[0], o["z"]) < 1e-6
    assert rel(t[0], o["theta"]) < 1e-6
    assert np.array_equal(b[0] != 0, o["beta"] != 0)


# ------------------------------------------------------------------ one-step properties at full size

@pytest.mark.parametrize("name", ["m", "m_pack2", "c3", "c4", "c5", "c5_pack2"])
def test_full_size_step_properties(cuda_ok, name):
    import paper_2601_02826_b200 as fs

    flags = fs.DESIGN_PACK2 if name.endswith("_pack2") else 0
    name = name.replace("_pack2", "")
    prob = datagen.make(name)
    X, y = to_device(prob)
    mu, G = 2.0 / prob.n, prob.G
    taus = list(prob.taus)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, [1.0] * len(taus), G=G, mu=mu, flags=flags)
    lm = S.lambda_max()
    frac = prob.lam_frac if prob.path_points == 1 else 0.1   # C5: a mid-path point (0.1 lambda_max)
    lams = [frac * v for v in lm]
    S.set_lambda(lams)
    eta = S.eta()
    S.iterate(200)
    n_checked, nsup = check_one_step(prob, S, taus, lams, eta, mu, G)
    assert nsup > 0
    assert n_checked >= 4000 * len(taus)
