"""The C-ABI library loads without a GPU, exports every symbol include/isf_lossy.h
declares, and its host-only entry points behave (no device calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2407_20731_b200 import build as B
    B.build()
    from paper_2407_20731_b200 import _native
    return _native.lib()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "isf_lossy.h")).read()
    return sorted(set(re.findall(r"\b(isf_lossy_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    from paper_2407_20731_b200 import _native
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.EXPORTS) == syms


def test_host_only_entry_points(lib):
    assert lib.isf_lossy_compression_ratio(1000, 20) == (1000.0 - 20.0) / 1000.0
    assert lib.isf_lossy_error_code_name(13).decode() == "ShapeMismatch"
    assert lib.isf_lossy_error_code_name(21).decode() == "InvalidArgument"
    assert lib.isf_lossy_error_code_name(0).decode() == "Ok"
    # stream sizes: counts padded to 16 B, masks, values
    assert lib.isf_lossy_stream_header_bytes(8, 1, 5) == 32 + 64 * 5
    assert lib.isf_lossy_stream_capacity(8, 1, 5) == 32 + 64 * 5 + 4096 * 5
    assert lib.isf_lossy_stream_header_bytes(6, 3, 2) == 32 + 32 * 6


def test_error_code_names_match_reference_enum(lib):
    # proj/include/isf/core/errors.hpp:8-38 order, via the Python mirror
    from paper_2407_20731_b200.lossy import ErrorCode
    for code in ErrorCode:
        assert lib.isf_lossy_error_code_name(int(code) + 1).decode() == code.name


def test_plan_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    rc = lib.isf_lossy_plan_create(ctypes.byref(h), 8, 1, 0)
    assert rc != 0  # TaskFailed (no device) or InvalidArgument, never a crash
    rc = lib.isf_lossy_plan_create(ctypes.byref(h), 99, 1, 0)
    assert rc == 21  # InvalidArgument: P out of range is checked first


def test_matches_oracle_sizes(lib, oracle):
    for P in range(2, 17):
        for n in (1, 7, 64):
            assert lib.isf_lossy_stream_capacity(P, 1, n) == oracle.stream_capacity(P, n)
            assert lib.isf_lossy_stream_header_bytes(P, 1, n) == oracle.stream_header_bytes(P, n)
