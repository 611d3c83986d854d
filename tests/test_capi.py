"""The C-ABI library loads, exports every declared symbol and validates
arguments on the host (no compute call is made without a GPU)."""
import ctypes

import pytest

from paper_2502_07563_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signatures out of sync with include/lasp2_b200.h"
    assert lib.lasp2_version() == 100


def test_so_is_sm100a_only():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def test_host_side_validation_returns_status_not_exception():
    lib = _lib.load()
    st = lib.lasp2_segment_states(_lib.BF16, None, None, None, 1, 128, 128, 1, None)
    assert st == 1 and b"null pointer" in lib.lasp2_last_error()
    st = lib.lasp2_fold_states(_lib.F32, ctypes.c_void_p(16), ctypes.c_void_p(16), 4, 16, 0, 9, None)
    assert st == 1 and b"bound" in lib.lasp2_last_error()
    st = lib.lasp2_causal_chunk(7, 1, 1, 1, None, None, 1, 1, 128, 128, 1, 0, 0, None)
    assert st == 1 and b"dtype" in lib.lasp2_last_error()
    st = lib.lasp2h_softmax_forward(_lib.F32, 1, 1, 1, 1, 1, 1, 8, 12, 4, 1, 0, 0, 0, None)
    assert st == 1 and b"kv_chunk" in lib.lasp2_last_error()
    st = lib.lasp2h_softmax_forward_range(_lib.F32, 1, 1, 1, 1, 1, 1, 8, 12, 4, 1, 0, 4, 0, -4, None)
    assert st == 1 and b"kv_start" in lib.lasp2_last_error()
    st = lib.lasp2h_softmax_forward_range(_lib.BF16, 1, 1, 1, 1, 1, 1, 8, 256, 64, 1, 0, 128, 0, 64, None)
    assert st == 1 and b"kv_start % 128" in lib.lasp2_last_error()
    # bfloat16 outside the tcgen05 envelope is refused (no second bf16 backend)
    st = lib.lasp2_apply_state(_lib.BF16, 16, 16, 16, 1, 256, 12, 0, 0, None)
    assert st == 1 and b"tcgen05 envelope" in lib.lasp2_last_error()
    st = lib.lasp2h_softmax_forward(_lib.BF16, 1, 1, 1, 1, 1, 1, 64, 256, 64, 1, 0, 64, 0, None)
    assert st == 1 and b"kv_chunk % 128" in lib.lasp2_last_error()
    with pytest.raises(ValueError, match="nseg"):
        _lib.call("lasp2_segment_states", _lib.F32, 16, 16, 16, 1, 128, 64, 5, None)


def test_num_segments_policy():
    lib = _lib.load()
    # tcgen05 path: one wave of 148 CTAs (16 slots x 9 segments = 144)
    assert lib.lasp2_num_segments(_lib.BF16, 16, 65536, 128, 148) == 9
    # never more segments than 128-token blocks
    assert lib.lasp2_num_segments(_lib.BF16, 1, 200, 128, 148) == 2
    assert lib.lasp2_num_segments(_lib.F64, 1, 8, 4, 148) == 1
