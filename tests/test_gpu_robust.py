"""GPU robustness tests: the numeric-error path (FSQR_ERR_NUMERIC), input validation of
fsqr_set_state, the theta fixed-point quantisation under a large dynamic range, and stream
ordering of the create-time zero fills (a context created under a non-default stream, with and
without the 2-bit repack, gives the same state as one created on the default stream).
Expected values come from the paper's formulas (numpy one-step checker) or from API identities."""
import numpy as np
import pytest

import datagen
from gpu_helpers import check_one_step, to_device

pytestmark = pytest.mark.gpu


def _solver(prob, taus, lams, **kw):
    import paper_2601_02826_b200 as fs

    X, y = to_device(prob)
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, taus, lams, G=5, **kw)
    return S


def test_overflowing_state_is_numeric_error(cuda_ok):
    """A finite but overflowing dual iterate (theta_1 = 1e305, so n*theta is Inf in R_z) makes the
    state non-finite: fsqr_solve reports FSQR_ERR_NUMERIC instead of iterating on."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=300, p=500)
    S = _solver(prob, [0.5], [0.01], tol=1e-8, max_iter=1000)
    S.iterate(5)
    b, z, t = S.state()
    t[0, 1] = 1e305
    S.set_state(b, z, t)
    with pytest.raises(fs.FsqrError) as e:
        S.solve()
    assert e.value.status == -3
    assert "non-finite" in str(e.value)


def test_set_state_rejects_nonfinite(cuda_ok):
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=200, p=300)
    S = _solver(prob, [0.5], [0.01])
    b, z, t = S.state()
    for bad in ("beta", "z", "theta"):
        bb, zz, tt = b.copy(), z.copy(), t.copy()
        {"beta": bb, "z": zz, "theta": tt}[bad][0, 3] = np.nan
        with pytest.raises(fs.FsqrError) as e:
            S.set_state(bb, zz, tt)
        assert e.value.status == -2, bad


@pytest.mark.parametrize("storage", [1, 2])
def test_theta_quantisation_large_dynamic_range(cuda_ok, storage):
    """theta^k is quantised to 28-bit fixed point relative to max|theta|.  With one
    |theta_i| 10^4 times every other entry the GPU step still satisfies E14 on every checked column
    within north_star's componentwise product bound 1e-5 sum_i |x~_ij theta_i| (and E15/E12)."""
    prob = datagen.make("c2", n=2000, p=6000, storage=storage)
    lams = [0.03]
    S = _solver(prob, [0.5], lams, eta=[25.0] * 5)
    S.iterate(60)
    b, z, t = S.state()
    rest = np.abs(t[0]).max()
    t[0, 777] = 1e4 * rest
    S.set_state(b, z, t)
    n_checked, nsup = check_one_step(prob, S, [0.5], lams, np.full(5, 25.0), 2.0 / prob.n, 5, ncols=6000)
    assert n_checked >= 6000 and nsup > 0


@pytest.mark.parametrize("pack", [False, True])
def test_create_on_side_stream(cuda_ok, pack):
    """Create (zero fills, 2-bit repack, column statistics, power method) and iterate entirely on a
    non-blocking torch stream: the state equals the default-stream context's bit for bit."""
    import torch

    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=700, p=2500)
    X, y = to_device(prob)
    flags = fs.DESIGN_PACK2 if pack else 0
    outs = []
    for side in (False, True):
        st = torch.cuda.Stream() if side else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [0.3, 0.6], [0.02, 0.02], G=5, flags=flags)
            S.iterate(40)
        st.synchronize()
        outs.append(S.state() + (S.eta(),))
        del S
    for a, c in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, c)
