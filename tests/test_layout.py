"""CPU checks of the 2-bit layout contract (include/fsqr.h FSQR_PACKED2, fsqr_pack2): the seeded
generator writes the same codes in both layouts, and the word-level packing rule the repack kernel
uses, (a | a>>6 | a>>12 | a>>18) & 0xFF per 32-bit word of four codes, reproduces the generator's
packed bytes.  (The GPU tests compare the kernel's output with the generator's bytes directly.)"""
import numpy as np

import datagen


def _pack_rule(x8: np.ndarray, n: int, ld2: int) -> np.ndarray:
    p = x8.shape[0]
    out = np.zeros((p, ld2), np.uint8)
    codes = np.zeros((p, 4 * ld2), np.uint32)
    codes[:, :n] = x8[:, :n]
    a = codes.reshape(p, ld2, 4)
    word = a[..., 0] | (a[..., 1] << 8) | (a[..., 2] << 16) | (a[..., 3] << 24)
    out[:] = ((word | (word >> 6) | (word >> 12) | (word >> 18)) & 0xFF).astype(np.uint8)
    return out


def test_generator_layouts_hold_identical_codes():
    for name, n, p in [("c2", 999, 40), ("c4", 37, 25), ("c5", 1024, 17)]:
        a = datagen.make(name, n=n, p=p, storage=datagen.STORAGE_U8)
        b = datagen.make(name, n=n, p=p, storage=datagen.STORAGE_P2)
        unpacked = np.stack([(b.X >> (2 * q)) & 3 for q in range(4)], -1).reshape(p, -1)[:, :n]
        np.testing.assert_array_equal(unpacked, a.X[:, :n])
        np.testing.assert_array_equal(a.y, b.y)
        assert b.ld == ((n + 3) // 4 + 15) // 16 * 16


def test_word_packing_rule_matches_generator():
    for name, n, p in [("c2", 999, 40), ("c2", 2, 3), ("c4", 4097, 9)]:
        a = datagen.make(name, n=n, p=p, storage=datagen.STORAGE_U8)
        b = datagen.make(name, n=n, p=p, storage=datagen.STORAGE_P2)
        np.testing.assert_array_equal(_pack_rule(a.X, n, b.ld), b.X)
