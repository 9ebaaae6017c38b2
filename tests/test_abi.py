"""The C-ABI boundary (CPU-only checks): libfsqr.so loads, exports every function that
include/fsqr.h declares (and the binding names exactly those), the host-only calls behave, and
without a GPU the compute entry fails loudly with FSQR_ERR_CUDA instead of falling back to CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsqr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(fsqr_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for must in ("fsqr_create", "fsqr_iterate", "fsqr_solve", "fsqr_objective", "fsqr_kkt", "fsqr_get_beta",
                 "fsqr_get_state", "fsqr_set_state", "fsqr_set_lambda", "fsqr_last_error", "fsqr_status_str",
                 "fsqr_destroy", "fsqr_path", "fsqr_trace"):
        assert must in names, must


def test_library_exports_every_declared_symbol():
    import paper_2601_02826_b200 as fs

    L = ctypes.CDLL(fs.lib_path())
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(fs.EXPORTS) == declared_functions()


def test_host_only_calls():
    import paper_2601_02826_b200 as fs

    L = fs.load(build_if_missing=False)
    o = fs.default_options()
    assert o.G == 5 and o.eta_safety == pytest.approx(1.05) and o.tol == pytest.approx(1e-6)
    assert o.max_iter == 100000 and o.power_max_iter == 1000 and o.trace_cap == 4096
    assert L.fsqr_status_str(0) == b"FSQR_OK"
    assert L.fsqr_status_str(-4) == b"FSQR_ERR_CUDA"
    fs.fsqr_destroy(None)   # NULL is a no-op


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2601_02826_b200 as fs

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    X = np.zeros((4, 16), dtype=np.uint8)
    X[:, :2] = [[0, 1]] * 4
    y = np.arange(16, dtype=np.float64)
    with pytest.raises(fs.FsqrError) as e:
        fs.fsqr_fit_host(X, 1, 16, 4, 16, y, [0.5], [0.1], 1, stream=0)
    assert e.value.status == -4
