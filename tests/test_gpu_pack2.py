"""GPU tests of the u8 -> 2-bit repack (fsqr_pack2 and the FSQR_DESIGN_PACK2 create flag,
include/fsqr.h; north_star storage subsystem (1), "uint8 or 2-bit packed {0,1,2}").

The expected bytes come from the seeded generator's own PACKED2 output for the same codes
(datagen writes both layouts from one draw), never from the device path; the solver equalities
are exact because the PACKED2 kernels compute exact integer products on identical codes."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import rel, to_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(999, 300), (1024, 129), (17, 5), (2, 3), (4097, 64)])
def test_pack2_matches_generator_layout(cuda_ok, n, p):
    import torch

    import paper_2601_02826_b200 as fs

    a = datagen.make("c2", n=n, p=p, storage=fs.U8)
    b = datagen.make("c2", n=n, p=p, storage=fs.PACKED2)
    X8 = torch.from_numpy(a.X).cuda()
    X2 = torch.full((p, b.ld), 0xAB, dtype=torch.uint8, device="cuda")   # garbage: every byte must be written
    out, ld2 = fs.fsqr_pack2(X8, a.ld, n, p, X2)
    assert ld2 == b.ld
    np.testing.assert_array_equal(out.cpu().numpy(), b.X)


def test_pack2_rejects_codes_above_3(cuda_ok):
    import torch

    import paper_2601_02826_b200 as fs

    a = datagen.make("c2", n=300, p=40, storage=fs.U8)
    X = a.X.copy()
    X[37, 211] = 4
    with pytest.raises(fs.FsqrError, match="ERR_DATA"):
        fs.fsqr_pack2(torch.from_numpy(X).cuda(), a.ld, a.n, a.p)
    y = torch.from_numpy(a.y).cuda()
    with pytest.raises(fs.FsqrError, match="ERR_DATA"):
        fs.Solver(torch.from_numpy(X).cuda(), fs.U8, a.n, a.p, a.ld, y, [0.5], [0.01], flags=fs.DESIGN_PACK2)
    # code 3 is representable and accepted
    X[37, 211] = 3
    fs.fsqr_pack2(torch.from_numpy(X).cuda(), a.ld, a.n, a.p)


def test_pack2_flag_needs_u8(cuda_ok):
    import torch

    import paper_2601_02826_b200 as fs

    b = datagen.make("c2", n=300, p=40, storage=fs.PACKED2)
    X, y = to_device(b)
    with pytest.raises(fs.FsqrError, match="ERR_CONFIG"):
        fs.Solver(X, fs.PACKED2, b.n, b.p, b.ld, y, [0.5], [0.01], flags=fs.DESIGN_PACK2)
    with pytest.raises(fs.FsqrError, match="ERR_CONFIG"):
        fs.Solver(X, fs.PACKED2, b.n, b.p, b.ld, y, [0.5], [0.01], flags=4)
    del torch


@pytest.mark.parametrize("name,taus", [("c2", [0.5]), ("c5", [0.1, 0.5, 0.9]), ("c5", [0.1 * k for k in range(1, 10)])])
def test_create_pack2_equals_packed_storage(cuda_ok, name, taus):
    """A solver created from u8 codes with FSQR_DESIGN_PACK2 is the PACKED2 solver: bit-identical
    state after the same iterations, and it no longer reads the u8 buffer (freed and overwritten)."""
    import torch

    import paper_2601_02826_b200 as fs

    a = datagen.make(name, n=1500, p=2600, storage=fs.U8)
    b = datagen.make(name, n=1500, p=2600, storage=fs.PACKED2)
    eta = [40.0] * 5
    lams = [0.03] * len(taus)
    X8, y = to_device(a)
    SA = fs.Solver(X8, fs.U8, a.n, a.p, a.ld, y, taus, lams, G=5, eta=eta, flags=fs.DESIGN_PACK2)
    X8.fill_(0xFF)          # the ctx must hold its own copy
    del X8
    torch.cuda.empty_cache()
    X2, _ = to_device(b)
    SB = fs.Solver(X2, fs.PACKED2, b.n, b.p, b.ld, y, taus, lams, G=5, eta=eta)
    assert SA.backend == SB.backend == "tc"
    SA.iterate(70)
    SB.iterate(70)
    for u, v in zip(SA.state(), SB.state()):
        np.testing.assert_array_equal(u, v)
    np.testing.assert_array_equal(SA.objective(), SB.objective())
    np.testing.assert_array_equal(SA.beta(1), SB.beta(1))
    # and it is the u8 solver: the products are exact integers on the same codes
    X8, _ = to_device(a)
    SC = fs.Solver(X8, fs.U8, a.n, a.p, a.ld, y, taus, lams, G=5, eta=eta)
    SC.iterate(70)
    for u, v in zip(SA.state(), SC.state()):
        assert rel(u, v) < 1e-12


def test_fit_host_pack2(cuda_ok):
    import paper_2601_02826_b200 as fs

    a = datagen.make("c2", n=700, p=1900, storage=fs.U8)
    b = datagen.make("c2", n=700, p=1900, storage=fs.PACKED2)
    eta = [25.0] * 5
    ba, _ = fs.fsqr_fit_host(a.X, fs.U8, a.n, a.p, a.ld, a.y, [0.5], [0.04], 80, opt=fs.default_options(G=5),
                             eta=eta, flags=fs.DESIGN_PACK2)
    bb, _ = fs.fsqr_fit_host(b.X, fs.PACKED2, b.n, b.p, b.ld, b.y, [0.5], [0.04], 80, opt=fs.default_options(G=5),
                             eta=eta)
    np.testing.assert_array_equal(ba, bb)


@pytest.mark.parametrize("n,p,taus", [(1500, 2600, [0.5]), (999, 3100, [0.3, 0.7]), (4097, 1800, [0.2, 0.5, 0.8]),
                                      (2500, 2000, [0.1 * k for k in range(1, 10)]),
                                      (700, 1500, [k / 17 for k in range(1, 17)])])
def test_k1_tcp_equals_cuda_core_forward(cuda_ok, monkeypatch, n, p, taus):
    """The tensor-core forward product for 2-bit storage (k1_tcp: on-chip unpack into the
    swizzled A tile) forms the same exact fixed-point sums as the CUDA-core k1_bulk: the whole
    state after k iterations is bit-identical (several row tiles, ragged last slab, 1-16 RHS)."""
    import paper_2601_02826_b200 as fs

    b = datagen.make("c5", n=n, p=p, storage=fs.PACKED2)
    X, y = to_device(b)
    eta = [40.0] * 5
    lams = [0.02] * len(taus)
    out = []
    for mode in ("bulk", "tcp"):
        monkeypatch.setenv("FSQR_K1", mode)
        S = fs.Solver(X, fs.PACKED2, b.n, b.p, b.ld, y, taus, lams, G=5, eta=eta)
        S.iterate(60)
        out.append(S.state() + (S.objective(),))
        del S
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)


def test_pack2_drivers_equal_u8(cuda_ok):
    """The drivers built on the hot path (warm-started lambda path + HBIC, one-step LLA) give the
    same answers on a repacked context as on the u8 one: identical iteration counts and supports,
    beta to 1e-12; the pivotal statistic (computed on a temporary u8 unpack) is bit-identical."""
    import paper_2601_02826_b200 as fs

    a = datagen.make("c2", n=700, p=1500, storage=fs.U8)
    X, y = to_device(a)
    eta = [25.0] * 5
    lm = None
    out = {}
    for flags in (0, fs.DESIGN_PACK2):
        S = fs.Solver(X, fs.U8, a.n, a.p, a.ld, y, [0.5], [1.0], G=5, eta=eta, tol=1e-6, max_iter_point=20000,
                      flags=flags)
        if lm is None:
            lm = S.lambda_max()[0]
        grid = np.array([[lm * 0.05 ** (t / 5) for t in range(6)]])
        res = S.path(grid)
        betas = [S.path_beta(0, t) for t in range(6)]
        h = S.path_hbic(6)
        S2 = fs.Solver(X, fs.U8, a.n, a.p, a.ld, y, [0.5], [0.1 * lm], G=5, eta=eta, tol=1e-6, max_iter=200000,
                       flags=flags)
        lla = S2.lla(fs.SCAD, 3.7, 1)
        out[flags] = (res, betas, h, lla, S2.beta()[0])
        out.setdefault("piv", []).append(S.pivotal(200, seed=11))
        del S, S2
    (r0, b0, h0, l0, bl0), (r1, b1, h1, l1, bl1) = out[0], out[fs.DESIGN_PACK2]
    np.testing.assert_array_equal(r0["iters"], r1["iters"])
    np.testing.assert_array_equal(r0["nnz"], r1["nnz"])
    for u, v in zip(b0, b1):
        assert rel(v, u) < 1e-12
        assert np.array_equal(u != 0, v != 0)
    np.testing.assert_allclose(h1, h0, rtol=1e-12)
    assert list(l0["stage_iters"]) == list(l1["stage_iters"])
    assert rel(bl1, bl0) < 1e-12
    np.testing.assert_array_equal(out["piv"][0], out["piv"][1])   # exact integer statistic


def test_fit_host_pack2_chunked_and_bad_code(cuda_ok):
    """fsqr_fit_host repacks a u8 host design chunk by chunk (p large enough for several 256 MB
    chunks is too big for a test, so the chunking is exercised through ld: one column chunk holds
    256 MB / ld columns) and rejects a code > 3 with FSQR_ERR_DATA."""
    import paper_2601_02826_b200 as fs

    a = datagen.make("c2", n=3000, p=2500, storage=fs.U8)
    b = datagen.make("c2", n=3000, p=2500, storage=fs.PACKED2)
    eta = [30.0] * 5
    ba, _ = fs.fsqr_fit_host(a.X, fs.U8, a.n, a.p, a.ld, a.y, [0.3, 0.8], [0.03, 0.03], 60,
                             opt=fs.default_options(G=5), eta=eta, flags=fs.DESIGN_PACK2)
    bb, _ = fs.fsqr_fit_host(b.X, fs.PACKED2, b.n, b.p, b.ld, b.y, [0.3, 0.8], [0.03, 0.03], 60,
                             opt=fs.default_options(G=5), eta=eta)
    np.testing.assert_array_equal(ba, bb)
    X = a.X.copy()
    X[2400, 17] = 9
    with pytest.raises(fs.FsqrError, match="ERR_DATA"):
        fs.fsqr_fit_host(X, fs.U8, a.n, a.p, a.ld, a.y, [0.5], [0.03], 10, opt=fs.default_options(G=5), eta=eta,
                         flags=fs.DESIGN_PACK2)


@pytest.mark.parametrize("n,p,G,taus", [(37, 1, 1, [0.5]), (130, 3, 2, [0.3, 0.7]), (513, 129, 5, [0.5]),
                                        (1023, 700, 5, list(np.linspace(0.05, 0.95, 16))), (2, 7, 1, [0.5])])
def test_pack2_flag_parity_ragged(cuda_ok, n, p, G, taus):
    """FSQR_DESIGN_PACK2 on ragged and tiny shapes (n not a multiple of 4, 16, 128 or 512; a
    single column; the maximum 16 RHS) against the fp64 oracle run on the same u8 codes."""
    import paper_2601_02826_b200 as fs

    prob = datagen.make("c2", n=n, p=p, storage=fs.U8)
    d = oracle.Design.from_problem(prob)
    mu = 2.0 / prob.n
    eta = oracle.eta(d, G, mu)
    lams = [0.05 * oracle.lambda_max(d, prob.y, t)[0] for t in taus]
    X, y = to_device(prob)
    S = fs.Solver(X, fs.U8, prob.n, prob.p, prob.ld, y, taus, lams, G=G, mu=mu, eta=eta, flags=fs.DESIGN_PACK2)
    k = 60
    S.iterate(k)
    b, z, t = S.state()
    for r in sorted({0, len(taus) // 2, len(taus) - 1}):
        o = oracle.solve(d, prob.y, taus[r], oracle.lam_vector(prob.p, lams[r]), eta, mu, G, max_iter=k, check=False)
        assert rel(b[r], o["beta"]) < 1e-6, r
        assert rel(t[r], o["theta"]) < 1e-6, r
        assert np.array_equal(b[r] != 0, o["beta"] != 0), r


@pytest.mark.parametrize("esmax,taus", [(64, [0.5]), (96, [0.2, 0.6, 0.9]), (32, [k / 10 for k in range(1, 10)])])
def test_k1_tcp_many_work_items_per_cta(cuda_ok, monkeypatch, esmax, taus):
    """Full support (lambda = 0) with the per-item entry cap lowered (FSQR_K1_ESMAX) so every
    CTA of k1_tcp runs many work items in a row: the metadata ring, the per-item cp.async
    pipeline and the accumulator hand-off across items must give the CUDA-core kernel's sums."""
    import paper_2601_02826_b200 as fs

    b = datagen.make("c4", n=1100, p=3000, storage=fs.PACKED2)
    X, y = to_device(b)
    eta = [40.0] * 5
    out = []
    for mode in ("bulk", "tcp"):
        monkeypatch.setenv("FSQR_K1", mode)
        monkeypatch.setenv("FSQR_K1_ESMAX", str(esmax))
        S = fs.Solver(X, fs.PACKED2, b.n, b.p, b.ld, y, taus, [0.0] * len(taus), G=5, eta=eta)
        S.iterate(25)
        st = S.state()
        assert int(S.trace(1)[-1, 0, 4]) > 2000   # most columns in the support
        out.append(st + (S.objective(),))
        del S
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("taus", [[0.5], [0.25, 0.5, 0.75], [k / 6 for k in range(1, 6)], [k / 10 for k in range(1, 10)],
                                  [k / 17 for k in range(1, 17)]])
def test_tc2_several_tiles_per_cta_equals_simt(cuda_ok, taus):
    """p = 40,000 columns = 313 tiles of 128 over at most 148 persistent CTAs, so every CTA of the
    2-bit tensor-core kernel carries its TMA ring, A buffers and double-buffered accumulators
    across tiles (two or three tiles per CTA: with 5, 9 and 16 RHS the tile-pair order runs a full
    pair and, on the CTAs with three tiles, a single-tile tail); the exact-integer dp4a kernel gives
    the same state bit for bit."""
    import paper_2601_02826_b200 as fs

    b = datagen.make("c5", n=700, p=40000, storage=fs.PACKED2)
    X, y = to_device(b)
    eta = [60.0] * 5
    out = []
    for backend in (fs.BACKEND_TC, fs.BACKEND_SIMT):
        S = fs.Solver(X, fs.PACKED2, b.n, b.p, b.ld, y, taus, [0.03] * len(taus), G=5, eta=eta, backend=backend)
        S.iterate(20)
        out.append(S.state() + (S.objective(),))
        del S
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("n,p,taus,esmax", [(1500, 2600, [0.5], 65536), (999, 3100, [0.3, 0.7], 65536),
                                            (4097, 1800, [0.2, 0.5, 0.8], 65536),
                                            (2500, 2000, [0.1 * k for k in range(1, 10)], 65536),
                                            (700, 1500, [k / 17 for k in range(1, 17)], 65536),
                                            (1100, 3000, [0.5], 64)])
def test_k1_tcu_u8_equals_cuda_core_forward(cuda_ok, monkeypatch, n, p, taus, esmax):
    """The tensor-core forward product for u8 storage (k1_tcp<., 1>: cp.async straight into the
    swizzled A tile) forms the same exact sums as the CUDA-core k1_bulk, 1-16 RHS, ragged slabs,
    and many work items per CTA."""
    import paper_2601_02826_b200 as fs

    b = datagen.make("c5", n=n, p=p, storage=fs.U8)
    X, y = to_device(b)
    eta = [40.0] * 5
    lams = [0.02 if esmax == 65536 else 0.0] * len(taus)
    out = []
    for mode in ("bulk", "tcu"):
        monkeypatch.setenv("FSQR_K1", mode)
        monkeypatch.setenv("FSQR_K1_ESMAX", str(esmax))
        S = fs.Solver(X, fs.U8, b.n, b.p, b.ld, y, taus, lams, G=5, eta=eta)
        S.iterate(40)
        out.append(S.state() + (S.objective(),))
        del S
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)
