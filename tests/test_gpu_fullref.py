"""Full-size parity on every BASELINE.json config against the fp64 ORACLE (SURVEY §8(d) parity gates).

1. Fixed iteration count: 200 iterations from the cold start (beta = 0, z = y, theta = 0) at full
   size, compared element by element with the oracle's own 200-iteration trajectory.  The oracle
   runs are hours of CPU time at these sizes, so they were made once by the committed script
   tools/oracle_ref.py (it calls only oracle/ and datagen/) and stored in tests/golden/oracle_ref/
   with a checksum of the generated design; eta_g and lambda come from those files (the oracle's
   own power method and lambda_max), never from the CUDA path.  The last iteration runs through
   bench.py's launch path (fsqr_profile_iterate).  Gates: beta, z, theta within 1e-6 relative
   (north_star: 1e-4; the exact-integer products give ~1e-9), identical supports, objective within
   1e-4, and the GPU's R(w^200) equal to the oracle's to 1e-5.
2. At convergence (R(w) <= 1e-4, the GPU's own stopping test), on the GPU's committed state:
   the oracle's R(w) <= 1.05 tol, the GPU's R equals the oracle's to 1e-5, the oracle's objective at
   the GPU's beta equals the GPU's to 1e-4, and one oracle iteration from the GPU's state moves
   beta and z by at most tol (relative 2-norms): the GPU stopped at a fixed point of the
   oracle's map, not merely at a point its own arithmetic calls converged.

Run on the GPU box: `pytest -m fullsize` (tens of GB of host RAM; C4 is 10 GB of 2-bit codes).
"""
import json
import os

import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import rel, to_device

pytestmark = [pytest.mark.gpu, pytest.mark.fullsize]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "tests", "golden", "oracle_ref")
C5_REF_TAUS = (0.1, 0.5, 0.9)


def design_checksum(prob) -> str:
    import importlib.util

    spec = importlib.util.spec_from_file_location("oracle_ref", os.path.join(ROOT, "tools", "oracle_ref.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.design_checksum(prob)


def load_ref(name, tau):
    fn = os.path.join(REF, f"{name}_tau{tau:.1f}.npz")
    if not os.path.exists(fn):
        pytest.skip(f"oracle reference {fn} not generated (tools/oracle_ref.py)")
    z = np.load(fn)
    out = {k: z[k] for k in z.files if k != "meta"}
    out["meta"] = json.loads(str(z["meta"]))
    beta = np.zeros(out["meta"]["p"] + 1)
    beta[out["beta_idx"]] = out["beta_val"]
    out["beta"] = beta
    return out


_PROBS = {}


def problem(name):
    """One datagen instance per design per session (C5 and M share the design)."""
    key = "m" if name in ("m", "c5") else name
    if key not in _PROBS:
        _PROBS.clear()
        _PROBS[key] = datagen.make(key)
    prob = _PROBS[key]
    if name == "c5":
        import copy

        prob = copy.copy(prob)
        prob.taus = list(datagen.CONFIGS["c5"]["taus"])
    return prob


def solver_for(name, prob, refs, pack, taus, lams, eta, tol=1e-4, max_iter=100000):
    import paper_2601_02826_b200 as fs

    X, y = to_device(prob)
    flags = fs.DESIGN_PACK2 if pack else 0
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, lams, G=prob.G, mu=2.0 / prob.n, eta=eta,
                  tol=tol, max_iter=max_iter, flags=flags)
    assert S.backend == "tc"
    return S, X


def setup_case(case):
    """(name, prob, pack, taus on the GPU, lambdas, eta, {rhs index: oracle ref})."""
    name, pack = case.replace("_pack2", ""), case.endswith("_pack2")
    prob = problem(name)
    if name == "c5":
        refs = {prob.taus.index(t): load_ref("c5", t) for t in C5_REF_TAUS}
    else:
        refs = {0: load_ref(name, prob.taus[0])}
    r0 = next(iter(refs.values()))
    assert design_checksum(prob) == r0["meta"]["checksum"], "regenerated design differs from the reference's"
    eta = r0["eta"]
    taus = list(prob.taus)
    return name, prob, pack, taus, eta, refs


def lambdas_for(S, taus, refs, frac):
    """lambda per RHS: the oracle reference's where there is one; the other C5 levels (not compared)
    at the same fraction of their lambda_max."""
    lm = S.lambda_max()
    lams = [frac * lm[r] for r in range(len(taus))]
    for r, ref in refs.items():
        np.testing.assert_allclose(lm[r], float(ref["lambda_max"]), rtol=1e-9)
        lams[r] = float(ref["lam"])
    return lams


CASES = ["m", "m_pack2", "c3", "c3_pack2", "c4", "c5", "c5_pack2"]


@pytest.mark.parametrize("case", CASES)
def test_200_iterations_match_oracle(cuda_ok, case):
    import paper_2601_02826_b200 as fs

    name, prob, pack, taus, eta, refs = setup_case(case)
    r0 = next(iter(refs.values()))
    S, X = solver_for(name, prob, refs, pack, taus, [1.0] * len(taus), eta)
    S.set_lambda(lambdas_for(S, taus, refs, r0["meta"]["lam_frac"]))
    K = int(r0["meta"]["iters"])
    S.iterate(K - 1)
    fs.fsqr_profile_iterate(S.ctx, 1)
    b, z, t = S.state()
    obj = S.objective()
    R = S.kkt()
    for r, ref in refs.items():
        tag = (case, taus[r])
        assert np.count_nonzero(ref["beta"][1:]) > 100, tag
        assert rel(b[r], ref["beta"]) < 1e-6, tag
        assert rel(z[r], ref["z"]) < 1e-6, tag
        assert rel(t[r], ref["theta"]) < 1e-6, tag
        mism = np.flatnonzero((b[r] != 0) != (ref["beta"] != 0))
        assert len(mism) == 0, (tag, mism[:10])
        assert obj[r] == pytest.approx(float(ref["obj"]), rel=1e-4), tag
        np.testing.assert_allclose(R[r], ref["R"], rtol=1e-5, err_msg=str(tag))


CONV = ["c2", "m_pack2", "c3_pack2", "c4", "c5_pack2"]


@pytest.mark.parametrize("case", CONV)
def test_converged_state_passes_oracle_checks(cuda_ok, case):
    tol = 1e-4
    name, pack = case.replace("_pack2", ""), case.endswith("_pack2")
    if name == "c2":
        prob = datagen.make("c2")
        d = oracle.Design.from_problem(prob)
        eta = oracle.eta(d, prob.G, 2.0 / prob.n)
        taus = list(prob.taus)
        refs = {}
        frac = prob.lam_frac
    else:
        name, prob, pack, taus, eta, refs = setup_case(case)
        d = oracle.Design.from_problem(prob)
        frac = next(iter(refs.values()))["meta"]["lam_frac"]
    S, X = solver_for(name, prob, refs, pack, taus, [1.0] * len(taus), eta, tol=tol, max_iter=60000)
    lams = lambdas_for(S, taus, refs, frac)
    if name == "c2":   # lambda from the oracle's lambda_max
        lams = [frac * oracle.lambda_max(d, prob.y, tt)[0] for tt in taus]
    S.set_lambda(lams)
    res = S.solve()
    assert res["status"] == 0, res
    b, z, t = S.state()
    obj = S.objective()
    Rg = S.kkt()
    check = sorted(refs) if refs else range(len(taus))
    mu, G = 2.0 / prob.n, prob.G
    for r in check:
        tau = taus[r]
        lv = oracle.lam_vector(prob.p, lams[r])
        Ro = oracle.kkt_rel(d, prob.y, tau, lv, b[r], z[r], t[r])
        assert Ro.max() <= 1.05 * tol, (case, tau, Ro)
        np.testing.assert_allclose(Rg[r], Ro, rtol=1e-5, atol=1e-12, err_msg=f"{case} tau={tau}")
        assert oracle.objective(d, prob.y, tau, lv, b[r]) == pytest.approx(obj[r], rel=1e-4)
        one = oracle.solve(d, prob.y, tau, lv, eta, mu, G, max_iter=1, check=False, state=(b[r], z[r], t[r]))
        mb = np.linalg.norm(one["beta"] - b[r]) / (1 + np.linalg.norm(b[r]))
        mz = np.linalg.norm(one["z"] - z[r]) / (1 + np.linalg.norm(z[r]))
        assert max(mb, mz) <= tol, (case, tau, mb, mz)


def test_c2_tuning_path_matches_oracle(cuda_ok):
    """The paper's tuning protocol at C2 full size (Table 2's dimensions, tau = 0.5, G = 5): fsqr_tune
    over the oracle reference's grid (50 points, lambda_max -> 0.01 lambda_max, reading R20) against the
    cached oracle path (tools/oracle_path_ref.py): the same grid, the same selected point, HBIC,
    objective, support and beta of every point, and identical update counts from the third point on.

    The first point is lambda = lambda_max itself, where beta = 0 and the fit is the sample median of
    n = 2000 observations (n tau an integer: every point of [y_(1000), y_(1001)] minimises, reading
    R17): R(w) is not monotone there and hovers around tol = 1e-4 for hundreds of iterations (the
    oracle's own R is 9.8e-5 at iteration 800, 8.7e-5 at 880, 1.2e-4 at 960), so the first iteration
    with R <= tol is decided by rounding (the GPU's theta is 28-bit fixed point) and the two sides
    may stop at different iterates of the same flat region: for the first two points the counts may
    differ, the objective and HBIC are compared at north_star's 1e-4 and the supports exactly (the
    intercept itself still moves along the flat region: 0.01455 at the oracle's iteration 787,
    0.01645 at 966, objectives equal to 5e-6)."""
    import paper_2601_02826_b200 as fs

    fn = os.path.join(REF, "c2_path_tau0.5.npz")
    if not os.path.exists(fn):
        pytest.skip("tools/oracle_path_ref.py has not been run")
    z = np.load(fn)
    meta = json.loads(str(z["meta"]))
    prob = datagen.make("c2")
    assert design_checksum(prob) == meta["checksum"]
    T, tau = meta["T"], meta["tau"]
    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [tau], [1.0], G=meta["G"], mu=meta["mu"],
                  eta=z["eta"], tol=meta["tol"], max_iter_point=meta["max_iter_point"])
    out = S.tune(T=T, lam_min_frac=meta["lam_min_frac"])
    np.testing.assert_allclose(out["grid"][0], z["grid"], rtol=1e-10)
    assert int(out["best"][0]) == int(np.argmin(z["hbic"]))
    res = S.path(out["grid"])          # the same path again, for the per-point records
    it_g, it_o = np.asarray(res["iters"][0]), np.asarray(z["iters"])
    np.testing.assert_array_equal(res["converged"][0], z["converged"])
    np.testing.assert_array_equal(it_g[2:], it_o[2:])
    off = np.concatenate([[0], np.cumsum(z["beta_cnt"])])
    for t in range(T):
        tol_t = 1e-4 if t < 2 else 1e-6
        assert res["obj"][0][t] == pytest.approx(float(z["obj"][t]), rel=tol_t), t
        assert out["hbic"][0][t] == pytest.approx(float(z["hbic"][t]), rel=tol_t), t
        bo = np.zeros(prob.p + 1)
        bo[z["beta_idx"][off[t]:off[t + 1]]] = z["beta_val"][off[t]:off[t + 1]]
        bg = S.path_beta(0, t)
        assert np.array_equal(bg != 0, bo != 0), t
        if t >= 2:   # (first two points: the flat region moves the intercept itself, ~13 % between the
            # oracle's own iterates 787 and 966 at equal objective to 5e-6).  Later points start from
            # those slightly different warm starts, so beta agrees to north_star's 1e-4 (point 2: 4.8e-5)
            assert rel(bg, bo) < 1e-4, (t, rel(bg, bo))
