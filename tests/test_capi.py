"""CPU-side checks of the C ABI: the in-tree library loads, exports every
symbol include/chebykan.h declares, and validates arguments with the
reference's error wording without touching a GPU."""
import ctypes
import re

import pytest

from conftest import ROOT
from paper_2511_14852_b200 import _lib

HEADER = ROOT / "include" / "chebykan.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"CK_API\s+[\w\s\*]+?\b(ck_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("ck_lut_build", "ck_expand", "ck_coeff_prepare", "ck_forward", "ck_backward", "ck_merge"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = declared_symbols()
    assert syms, "no symbols parsed from the header"
    for name in syms:
        assert hasattr(lib, name), f"{name} not exported by {_lib.LIB_PATH}"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_version_and_sizes_are_host_only():
    lib = _lib.lib()
    assert lib.ck_version() >= 10000
    small = lib.ck_coeff_prep_bytes(64, 64, 5)
    big = lib.ck_coeff_prep_bytes(4096, 4096, 9)
    assert 0 < small < big
    # bf16 hi/lo (4 bytes per coefficient) in the forward layout (K planes)
    # and the input-gradient layout (k >= 1 only)
    assert big >= 4 * 4096 * 4096 * (9 + 8)
    assert lib.ck_forward_workspace_bytes(16384, 4096, 4096, 9) > 0
    assert lib.ck_backward_workspace_bytes(16384, 4096, 4096, 9) > 0
    assert lib.ck_coeff_prep_bytes(0, 4, 2) == 0


def test_forward_without_lut_is_a_value_error():
    lib = _lib.lib()
    rc = lib.ck_forward(None, 4, 8, 8, None, None, 0, None, None, None, 0, None, 0, None)
    assert rc == _lib.CK_INVALID_ARGUMENT
    assert "LUT mode requires a LutTable" in _lib.last_error()
    with pytest.raises(ValueError, match="LUT mode requires a LutTable"):
        _lib.check(rc, "ck_forward")


def test_lut_build_argument_errors_match_reference_wording():
    lib = _lib.lib()
    h = ctypes.c_void_p()
    assert lib.ck_lut_build(0, 4, 1, 0, ctypes.byref(h)) == _lib.CK_INVALID_ARGUMENT
    assert "lut_size must be >= 2" in _lib.last_error()       # lut.py:78-79
    assert lib.ck_lut_build(0, -1, 16, 0, ctypes.byref(h)) == _lib.CK_INVALID_ARGUMENT
    assert "degree must be >= 0" in _lib.last_error()          # lut.py:80-81
    assert lib.ck_lut_build(7, 3, 16, 0, ctypes.byref(h)) == _lib.CK_INVALID_ARGUMENT
    assert "unsupported basis kind" in _lib.last_error()
    # cos(k acos t) exists only as exact evaluation (trig_rows, basis.py:144-152)
    assert lib.ck_lut_build(4, 3, 16, 0, ctypes.byref(h)) == _lib.CK_INVALID_ARGUMENT
    assert lib.ck_basis_exact(1, -2, 0, ctypes.byref(h)) == _lib.CK_INVALID_ARGUMENT


def test_merge_rejects_bad_extents():
    lib = _lib.lib()
    assert lib.ck_merge(None, 2, 4, 8, None, 0, None) == _lib.CK_INVALID_ARGUMENT


def test_chunk_rows_setter_round_trip():
    # ck_set_chunk_rows is host-only state; the workspace queries follow it
    import paper_2511_14852_b200 as ck

    lib = _lib.lib()
    prev = lib.ck_set_chunk_rows(1000)
    try:
        assert lib.ck_set_chunk_rows(2000) == 1000
    finally:
        lib.ck_set_chunk_rows(prev)
    with ck.chunk_rows(77):
        assert lib.ck_set_chunk_rows(77) == 77
    assert lib.ck_set_chunk_rows(prev) == prev
    with ck.chunk_rows(256):
        small = lib.ck_backward_workspace_bytes(65536, 1024, 1024, 9)
        cache_small = lib.ck_basis_cache_bytes(65536, 1024, 1024, 9)
    assert small < lib.ck_backward_workspace_bytes(65536, 1024, 1024, 9)
    # the basis cache holds every chunk's planes: same bytes up to alignment
    assert abs(cache_small - lib.ck_basis_cache_bytes(65536, 1024, 1024, 9)) < 256 * 512


def test_prep_check_rejects_null_and_small_buffers():
    lib = _lib.lib()
    assert lib.ck_coeff_prep_check(None, 0, 8, 8, 3) == _lib.CK_INVALID_ARGUMENT
    assert lib.ck_coeff_prep_check(ctypes.c_void_p(4096), 16, 8, 8, 3) == _lib.CK_INVALID_ARGUMENT
    assert "too small" in _lib.last_error()
    assert lib.ck_coeff_prep_check(ctypes.c_void_p(4096), 1 << 30, 8, 8, 3) == _lib.CK_INVALID_ARGUMENT
    assert "not filled by ck_coeff_prepare" in _lib.last_error()
