"""CPU tests of the product boundary: libtsg.so is built, loads, exports
every entry point include/tsg.h declares, and refuses to run without a
CUDA device (no silent CPU fallback)."""
import os
import re

import numpy as np
import pytest

from paper_2308_16395_b200 import streaming as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tsg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tsg_create", "tsg_init", "tsg_update", "tsg_process_mode", "tsg_export_state",
              "tsg_import_state", "tsg_estimate_relative_error", "tsg_metrics_at", "tsg_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = S.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), f"libtsg.so does not export {s}"
    assert sorted(S.EXPORTED) == declared_symbols()


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except Exception:
        pass
    with pytest.raises(S.DeviceError):
        S.stream_init(np.ones((4, 3, 2)), 0.1)


def test_missing_library_fails_loudly(tmp_path):
    old = S._LIB
    S._LIB = None
    try:
        with pytest.raises(ImportError):
            S.load_library(str(tmp_path / "libtsg.so"))
    finally:
        S._LIB = old


def test_layout_helpers_roundtrip():
    t = np.random.default_rng(0).standard_normal((3, 4, 5))
    flat, dims = S._flat(t)
    assert dims == [3, 4, 5]
    assert flat[1] == t[1, 0, 0] and flat[3] == t[0, 1, 0] and flat[12] == t[0, 0, 1]
    np.testing.assert_array_equal(S._unflat(flat, dims), t)
