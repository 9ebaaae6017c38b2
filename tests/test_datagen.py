"""The seeded input generators (shared by oracle and CUDA path) follow their stated recipes."""
import numpy as np
import pytest

import datagen


def test_reproducible_and_layout():
    a = datagen.make("c2", n=300, p=50)
    b = datagen.make("c2", n=300, p=50)
    assert a.X.shape == (50, 304) and a.ld == 304
    np.testing.assert_array_equal(a.X, b.X)
    np.testing.assert_array_equal(a.y, b.y)
    assert np.all(a.X[:, 300:] == 0)            # padding rows are zero
    assert set(np.unique(a.X[:, :300])) <= {0, 1, 2}


def test_packed_matches_u8_codes():
    """2-bit layout stores the same Binomial(2, f) draws as the u8 layout (4 samples / byte)."""
    u = datagen.make("c2", n=103, p=9, storage=datagen.STORAGE_U8)
    q = datagen.make("c2", n=103, p=9, storage=datagen.STORAGE_P2)
    codes = np.stack([(q.X.astype(np.int64) >> (2 * s)) & 3 for s in range(4)], axis=2).reshape(9, -1)[:, :103]
    np.testing.assert_array_equal(codes, u.X[:, :103])
    assert q.ld == 32


def test_binomial_maf_law():
    pr = datagen.make("c2", n=20000, p=40)
    g = pr.X[:, :pr.n].astype(np.float64)
    f = pr.maf
    assert np.all((f >= 0.05) & (f <= 0.5))
    np.testing.assert_allclose(g.mean(axis=1), 2 * f, atol=0.03)
    # Hardy-Weinberg: P(G=2) = f^2
    np.testing.assert_allclose((g == 2).mean(axis=1), f ** 2, atol=0.02)


def test_ld_design_hwe_and_correlation():
    pr = datagen.make("c4", n=4000, p=200, storage=datagen.STORAGE_U8)
    g = pr.X[:, :pr.n].astype(np.float64)
    f = pr.maf
    np.testing.assert_allclose((g >= 1).mean(axis=1), 1 - (1 - f) ** 2, atol=0.04)
    np.testing.assert_allclose((g == 2).mean(axis=1), f ** 2, atol=0.03)
    # neighbours inside an LD block are positively correlated, across blocks they are not
    c_in = [np.corrcoef(g[j], g[j + 1])[0, 1] for j in range(0, 98)]
    c_out = np.corrcoef(g[99], g[100])[0, 1]
    assert np.mean(c_in) > 0.2 and abs(c_out) < 0.1


def test_probit_and_noise_laws():
    assert datagen.probit(0.975) == pytest.approx(1.959963984540054, abs=1e-9)
    assert datagen.probit(0.5) == pytest.approx(0.0, abs=1e-12)
    pr = datagen.make("c1")
    assert pr.X.dtype == np.float32 and pr.X.shape == (2000, 200)
    x = pr.X.astype(np.float64).ravel()
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    assert len(np.unique(pr.causal)) == 10
    assert np.all((np.abs(pr.effects) >= 0.5) & (np.abs(pr.effects) <= 2.0))
