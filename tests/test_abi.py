"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and
exports every entry point include/zoomr.h declares; host-detectable argument
errors are reported without touching a device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "zoomr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zoomr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_10898_b200 import _build
    path = _build.build()
    return C.CDLL(path)


def test_header_declares_the_five_stages():
    fns = declared_functions()
    for f in ("zoomr_update_mean_keys", "zoomr_score", "zoomr_select_topc", "zoomr_build_index",
              "zoomr_sparse_decode_attn"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in declared_functions():
        assert hasattr(lib, f), f"libzoomr.so does not export {f}"


def test_binding_names_match_header():
    from paper_2604_10898_b200 import zoomr as Z
    assert set(Z.EXPORTS) == set(declared_functions())


def test_status_strings_and_version(lib):
    lib.zoomr_status_str.restype = C.c_char_p
    assert lib.zoomr_status_str(0) == b"ZOOMR_OK"
    assert lib.zoomr_status_str(6) == b"ZOOMR_ERR_CAPACITY"
    assert lib.zoomr_status_str(999) == b"ZOOMR_ERR_UNKNOWN"
    assert lib.zoomr_abi_version() == 9


def test_host_argument_errors_without_a_device(lib):
    from paper_2604_10898_b200 import zoomr as Z
    g = Z.Geom(32, 32, 8, 128, 64)
    # NULL pointers -> ZOOMR_ERR_INVALID_ARG, nothing enqueued
    assert lib.zoomr_score(C.byref(g), 1, None, None, None, 16, 2, None, None, None, None, None) == 1
    bad = Z.Geom(32, 30, 8, 128, 64)  # H_q % H_kv != 0
    assert lib.zoomr_score(C.byref(bad), 1, None, None, None, 16, 2, None, None, None, None, None) == 2
    odd = Z.Geom(32, 32, 8, 96, 64)   # unsupported head_dim
    assert lib.zoomr_score(C.byref(odd), 1, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), 16, 2,
                           C.c_void_p(16), None, None, None, None) == 7
    lib.zoomr_attn_workspace_bytes.restype = C.c_size_t
    assert lib.zoomr_attn_workspace_bytes(C.byref(bad), 1) == 0
    assert lib.zoomr_build_index(1, None, None, 4, 0, None, 16, None, None, None) == 1


def test_round2_entry_points_reject_bad_arguments_without_a_device(lib):
    """The entry points added in round 2 validate on the host: NULL or inconsistent
    arguments return ZOOMR_ERR_INVALID_ARG (1) before anything is enqueued."""
    from paper_2604_10898_b200 import zoomr as Z
    g = Z.Geom(32, 32, 8, 128, 64)
    i32 = C.c_int32
    # zoomr_append_track: no pools / no outputs
    assert lib.zoomr_append_track(C.byref(g), 1, None, None, 0, None, None, None, 0, 0, None, 0, None, None, None, 8,
                                  None, None, None, None, None) == 1
    kv = Z.KV(C.c_void_p(256), C.c_void_p(256), 4, C.c_void_p(256), 4)
    dummy = C.c_void_p(256)
    # a mirror pool without a page size
    mirror = Z.KV(C.c_void_p(256), C.c_void_p(256), 4, C.c_void_p(256), 4)
    assert lib.zoomr_append_track(C.byref(g), 1, C.byref(kv), C.byref(mirror), 0, dummy, dummy, dummy, 0, 1, None,
                                  0, dummy, dummy, dummy, 8, dummy, dummy, dummy, None, None) == 1
    # negative boundary count
    assert lib.zoomr_append_track(C.byref(g), 1, C.byref(kv), None, 0, dummy, dummy, dummy, 0, 1, None, -1, dummy,
                                  dummy, dummy, 8, dummy, dummy, dummy, None, None) == 1
    # zoomr_sparse_decode_attn_lse_chained needs the lse output
    assert lib.zoomr_sparse_decode_attn_lse_chained(
        C.byref(g), 1, dummy, C.byref(kv), dummy, None, dummy, 64, None, 0, 0, C.c_float(0.1), 0, 0, dummy, None,
        dummy, C.c_size_t(1 << 20), None, None) == 1
    # zoomr_select_front / zoomr_select_tail / zoomr_tier_gather_slice: NULL inputs
    assert lib.zoomr_select_front(C.byref(g), 1, None, None, None, None, 0, None, None, 2, None, None, None, None,
                                  C.c_size_t(0), None, None) == 1
    assert lib.zoomr_select_tail(C.byref(g), 1, None, None, None, None, 2, 4, 8, None, None, None, None, 16, None,
                                 None, None) == 1
    assert lib.zoomr_tier_gather_slice(C.byref(g), 1, None, None, None, 16, 0, 1, None, None, 64, 4, None, None) == 1
