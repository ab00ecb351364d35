"""ctypes marshalling for the C oracle (``oracle/zoomr_oracle.c``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function takes
numpy arrays in the layouts documented in ``zoomr_oracle.h`` (bf16 tensors as
uint16 bit patterns, logical token order, one sequence per call) and returns
numpy arrays.  No arithmetic of the method lives here: each wrapper only
allocates outputs and forwards to the C function with the same name.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "zoomr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ZO_OK, ZO_ERR_INVALID_ARG, ZO_ERR_EMPTY_SEGMENT, ZO_ERR_SEGMENT_ORDER, ZO_ERR_INDEX_RANGE, \
    ZO_ERR_CAPACITY = range(6)


class OracleError(RuntimeError):
    def __init__(self, fn: str, rc: int):
        super().__init__(f"{fn} returned {rc}")
        self.rc = rc


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "zoomr_oracle.h"))):
        cmd = ["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Geom(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_q_heads", C.c_int32),
                ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32)]


class _Params(C.Structure):
    _fields_ = [("top_k", C.c_int32), ("c", C.c_int32), ("sink", C.c_int32),
                ("window", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.zo_bf16_to_double.restype = C.c_double
        _lib.zo_bf16_to_double.argtypes = [C.c_uint16]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _geom(L, Hq, Hkv, d):
    return _Geom(int(L), int(Hq), int(Hkv), int(d))


def _check(name, rc):
    if rc != ZO_OK:
        raise OracleError(name, rc)


def _u16(a):
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint16:
        raise TypeError("bf16 inputs must be uint16 bit patterns")
    return a


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def num_threads(n: int = 0) -> int:
    return int(lib().zo_num_threads(C.c_int32(n)))


def validate_segments(seg, T):
    seg = _i32(seg).reshape(-1, 4)
    return int(lib().zo_validate_segments(_p(seg), C.c_int32(len(seg)), C.c_int32(T)))


def update_mean_keys(keys, seg, L, Hkv, d, Hq=None):
    """O1. keys: uint16 [T][L][Hkv][d]; seg int32 [n][4] -> double [L][Hkv][n][d]."""
    keys = _u16(keys)
    seg = _i32(seg).reshape(-1, 4)
    T, n = keys.shape[0], seg.shape[0]
    out = np.zeros((L, Hkv, n, d), dtype=np.float64)
    g = _geom(L, Hq or Hkv, Hkv, d)
    _check("zo_update_mean_keys", lib().zo_update_mean_keys(
        C.byref(g), _p(keys), C.c_int32(T), _p(seg), C.c_int32(n), _p(out)))
    return out


def score(q, mean_keys, top_k, L, Hq, Hkv, d):
    """O2-O4. Returns dict(alpha [L][Hq][n], topk [L*Hq][kk], votes [n], A [n], near_tie [V])."""
    q = _u16(q)
    mk = np.ascontiguousarray(mean_keys, dtype=np.float64)
    n = mk.shape[2] if mk.ndim == 4 else 0
    kk = min(top_k, n)
    V = L * Hq
    alpha = np.zeros((L, Hq, n), dtype=np.float64)
    topk = np.zeros((V, max(kk, 0)), dtype=np.int32)
    votes = np.zeros(n, dtype=np.int64)
    A = np.zeros(n, dtype=np.float64)
    nt = np.zeros(V, dtype=np.uint8)
    g = _geom(L, Hq, Hkv, d)
    _check("zo_score", lib().zo_score(C.byref(g), _p(q), _p(mk), C.c_int32(n), C.c_int32(top_k),
                                      _p(alpha), _p(topk), _p(votes), _p(A), _p(nt)))
    return dict(alpha=alpha, topk=topk, votes=votes, A=A, near_tie=nt)


def aggregate(alpha, topk, L, Hq, Hkv, d):
    """O4 from given per-voter sets."""
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    topk = _i32(topk)
    n = alpha.shape[-1]
    kk = topk.shape[1] if topk.ndim == 2 else 0
    votes = np.zeros(n, dtype=np.int64)
    A = np.zeros(n, dtype=np.float64)
    g = _geom(L, Hq, Hkv, d)
    _check("zo_aggregate", lib().zo_aggregate(C.byref(g), _p(alpha), C.c_int32(n), C.c_int32(kk),
                                              _p(topk), _p(votes), _p(A)))
    return votes, A


def select_topc(votes, A, c):
    """O5. Returns (flags uint8 [n], agreeability, cut_near_tie)."""
    votes = np.ascontiguousarray(votes, dtype=np.int64)
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = votes.shape[0]
    flags = np.zeros(n, dtype=np.uint8)
    ag = C.c_double(0.0)
    cut = C.c_uint8(0)
    _check("zo_select_topc", lib().zo_select_topc(_p(votes), _p(A), C.c_int32(n), C.c_int32(c),
                                                  _p(flags), C.byref(ag), C.byref(cut)))
    return flags, ag.value, bool(cut.value)


def build_index(seg, flags, T, sink, window, capacity=None):
    """O6. Returns int32 [count] ascending."""
    seg = _i32(seg).reshape(-1, 4)
    n = seg.shape[0]
    flags = np.ascontiguousarray(flags, dtype=np.uint8) if n else np.zeros(1, np.uint8)
    cap = int(T if capacity is None else capacity)
    idx = np.zeros(max(cap, 1), dtype=np.int32)
    cnt = C.c_int32(0)
    rc = lib().zo_build_index(_p(seg), C.c_int32(n), _p(flags), C.c_int32(T), C.c_int32(sink),
                              C.c_int32(window), _p(idx), C.c_int32(cap), C.byref(cnt))
    _check("zo_build_index", rc)
    return idx[:cnt.value].copy()


def attend_one(q_vec, k_rows, v_rows, index, scale=None):
    """O7 for one head. k_rows/v_rows: uint16 [T][d] (row-major); q_vec uint16 [d]."""
    q_vec, k_rows, v_rows = _u16(q_vec), _u16(k_rows), _u16(v_rows)
    d = q_vec.shape[-1]
    index = _i32(index)
    out = np.zeros(d, dtype=np.float64)
    sc = 1.0 / np.sqrt(d) if scale is None else float(scale)
    _check("zo_attend_one", lib().zo_attend_one(
        _p(q_vec), _p(k_rows), _p(v_rows), C.c_int64(k_rows.shape[-1]), C.c_int32(d), _p(index),
        C.c_int32(len(index)), C.c_double(sc), _p(out)))
    return out


def sparse_decode_attn(q, keys, values, index, L, Hq, Hkv, d, scale=None, threads=0):
    """O7 for all (l, h). keys/values uint16 [T][L][Hkv][d]; q uint16 [L][Hq][d]."""
    q, keys, values = _u16(q), _u16(keys), _u16(values)
    index = _i32(index)
    out = np.zeros((L, Hq, d), dtype=np.float64)
    sc = 1.0 / np.sqrt(d) if scale is None else float(scale)
    g = _geom(L, Hq, Hkv, d)
    _check("zo_sparse_decode_attn", lib().zo_sparse_decode_attn(
        C.byref(g), _p(q), _p(keys), _p(values), C.c_int32(keys.shape[0]), _p(index),
        C.c_int32(len(index)), C.c_double(sc), _p(out), C.c_int32(threads)))
    return out


def log_partition(q, keys, index, L, Hq, Hkv, d, scale=None):
    """O8: lse [L][Hq] = ln sum_{j in index} exp(q.k_j * scale). keys uint16 [T][L][Hkv][d]."""
    q, keys = _u16(q), _u16(keys)
    index = _i32(index)
    lse = np.zeros((L, Hq), dtype=np.float64)
    sc = 1.0 / np.sqrt(d) if scale is None else float(scale)
    g = _geom(L, Hq, Hkv, d)
    _check("zo_log_partition", lib().zo_log_partition(
        C.byref(g), _p(q), _p(keys), C.c_int32(keys.shape[0]), _p(index), C.c_int32(len(index)),
        C.c_double(sc), _p(lse)))
    return lse


def h2o_weights(q, keys, index, L, Hq, Hkv, d, scale=None):
    """O9: per-retained-token softmax weight averaged over (l, h): fp64 [count]."""
    q, keys = _u16(q), _u16(keys)
    index = _i32(index)
    w = np.zeros(max(len(index), 1), dtype=np.float64)
    sc = 1.0 / np.sqrt(d) if scale is None else float(scale)
    g = _geom(L, Hq, Hkv, d)
    _check("zo_h2o_weights", lib().zo_h2o_weights(
        C.byref(g), _p(q), _p(keys), C.c_int32(keys.shape[0]), _p(index), C.c_int32(len(index)),
        C.c_double(sc), _p(w)))
    return w[:len(index)]


def h2o_select(prev, score, T, sink, window, budget):
    """O9: the next retained set (sorted int32) from the previous one and fp64 scores [T]."""
    n_prev = len(prev)
    prev = _i32(prev) if n_prev else np.zeros(1, np.int32)
    score = np.ascontiguousarray(score, dtype=np.float64)
    out = np.zeros(max(int(T), 1), dtype=np.int32)
    cnt = C.c_int32(0)
    _check("zo_h2o_select", lib().zo_h2o_select(
        _p(prev), C.c_int32(n_prev), _p(score), C.c_int32(T), C.c_int32(sink), C.c_int32(window),
        C.c_int32(budget), _p(out), C.c_int32(len(out)), C.byref(cnt)))
    return out[:cnt.value].copy()


def step(q, keys, values, seg, L, Hq, Hkv, d, top_k, c, sink, window, threads=0):
    """O1..O7 for one sequence (Alg.1 order). Returns a dict of every intermediate."""
    q, keys, values = _u16(q), _u16(keys), _u16(values)
    seg = _i32(seg).reshape(-1, 4)
    T, n = keys.shape[0], seg.shape[0]
    kk = min(top_k, n)
    mk = np.zeros((L, Hkv, n, d), dtype=np.float64)
    alpha = np.zeros((L, Hq, n), dtype=np.float64)
    topk = np.zeros((L * Hq, max(kk, 1)), dtype=np.int32)
    votes = np.zeros(max(n, 1), dtype=np.int64)
    A = np.zeros(max(n, 1), dtype=np.float64)
    flags = np.zeros(max(n, 1), dtype=np.uint8)
    idx = np.zeros(T, dtype=np.int32)
    cnt = C.c_int32(0)
    out = np.zeros((L, Hq, d), dtype=np.float64)
    g = _geom(L, Hq, Hkv, d)
    prm = _Params(int(top_k), int(c), int(sink), int(window))
    _check("zo_step", lib().zo_step(
        C.byref(g), C.byref(prm), _p(q), _p(keys), _p(values), C.c_int32(T), _p(seg),
        C.c_int32(n), _p(mk), _p(alpha), _p(topk), _p(votes), _p(A), _p(flags), _p(idx),
        C.c_int32(T), C.byref(cnt), _p(out), C.c_int32(threads)))
    return dict(mean_keys=mk, alpha=alpha, topk=topk[:, :kk], votes=votes[:n], A=A[:n],
                flags=flags[:n], index=idx[:cnt.value].copy(), out=out)


def bf16_to_double(bits: int) -> float:
    return float(lib().zo_bf16_to_double(C.c_uint16(bits)))
