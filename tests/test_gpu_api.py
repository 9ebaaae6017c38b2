"""GPU tests of the remaining C-ABI entry points (include/fsqr.h): determinism run to run,
fsqr_kkt against the oracle's R(w), original-scale coefficients (L404), warm start through
fsqr_get_state / fsqr_set_state, the host-buffer entry fsqr_fit_host, the trace and the
iteration counter.  Expected values come from the oracle or from the device path itself where
the property is an identity of the API (a round trip, bitwise repeatability)."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import make_pair, rel, to_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,storage,taus", [("c2", 1, [0.5]), ("c4", 2, [0.3, 0.7]), ("c5", 1, [0.1, 0.4, 0.6, 0.9])])
def test_bitwise_deterministic_run_to_run(cuda_ok, name, storage, taus):
    """Exact-integer products and fixed-order reductions: two contexts on the same inputs give
    bit-identical beta, z, theta and objective (header promise)."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make(name, n=900, p=2100, storage=storage)
    X, y = to_device(prob)
    outs = []
    for _ in range(2):
        S = fs.Solver(X, storage, prob.n, prob.p, prob.ld, y, taus, [0.02] * len(taus), G=5, eta=[30.0] * 5)
        S.iterate(75)
        outs.append(S.state() + (S.objective(),))
        del S
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)


def test_kkt_matches_oracle(cuda_ok):
    prob, d, S, cfg = make_pair("c2", n=700, p=1500, taus=[0.4])
    S.iterate(120)
    R = S.kkt()[0]
    b, z, t = S.state()
    Ro = oracle.kkt_rel(d, prob.y, 0.4, oracle.lam_vector(prob.p, cfg["lams"][0]), b[0], z[0], t[0])
    np.testing.assert_allclose(R, Ro, rtol=1e-5, atol=1e-12)


def test_original_scale_coefficients(cuda_ok):
    """fsqr_get_beta(scale=1): beta_j / s_j and beta_0 - sum_j m_j beta_j / s_j, so
    the original-scale fit reproduces X~ beta on the raw codes."""
    prob, d, S, cfg = make_pair("c2", n=500, p=800, taus=[0.5])
    S.iterate(200)
    bs = S.beta(0)[0]
    bo = S.beta(1)[0]
    raw = prob.X[:, :prob.n].astype(np.float64).T
    fit_orig = bo[0] + raw @ bo[1:]
    fit_std = oracle.fwdprod(d, bs)
    np.testing.assert_allclose(fit_orig, fit_std, rtol=1e-9, atol=1e-9 * np.abs(fit_std).max())


def test_state_round_trip_and_warm_start(cuda_ok):
    """set_state(get_state()) then k iterations == 2k iterations in one go, bit for bit... up to
    the fixed-point scale of the forward product, which is re-derived from the restored support
    (so compare at 1e-9)."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=800, p=1700)
    X, y = to_device(prob)
    A = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, [0.5], [0.03], G=5, eta=[25.0] * 5)
    A.iterate(80)
    st = A.state()
    A.iterate(80)
    B = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, [0.5], [0.03], G=5, eta=[25.0] * 5)
    B.set_state(*st)
    assert B.iterations() == 0
    B.iterate(80)
    assert B.iterations() == 80
    for a, b in zip(A.state(), B.state()):
        assert rel(a, b) < 1e-9


def test_fit_host_equals_device_path(cuda_ok):
    """The host-buffer entry (copies X and y itself) computes the same beta as the device path."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=600, p=1300)
    X, y = to_device(prob)
    eta = [20.0] * 5
    S = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, [0.6], [0.04], G=5, eta=eta)
    S.iterate(90)
    beta_h, res = fs.fsqr_fit_host(prob.X, 1, prob.n, prob.p, prob.ld, prob.y, [0.6], [0.04], 90,
                                   opt=fs.default_options(G=5), eta=eta)
    np.testing.assert_array_equal(beta_h, S.beta(0))


def test_trace_records_every_iteration(cuda_ok):
    """fsqr_trace rows are R(w^k) and the objective of the iterates; the last row's objective is
    the objective of the state before the last update (one-iteration lag of the KKT test)."""
    prob, d, S, cfg = make_pair("c2", n=500, p=900, taus=[0.5], tol=1e-6)
    res = S.solve()
    assert res["status"] == 0
    tr = S.trace(4096)
    assert tr.shape[0] == min(S.iterations() + 1, 4096)
    last = tr[-1, 0]
    assert max(last[0], last[1], last[2]) <= 1e-6
    np.testing.assert_allclose(last[3], S.objective()[0], rtol=1e-10)
    assert np.all(np.abs(np.diff(tr[:, 0, 3][-50:])) <= 1e-4 * abs(tr[-1, 0, 3]))   # objective settles
