"""Thin Python binding of libzoomr.so (include/zoomr.h): argument marshalling only.

Every function has the name of the C entry point without the ``zoomr_`` prefix,
takes CUDA torch tensors (PyTorch supplies device memory and the stream) and
enqueues the CUDA kernels on the current stream.  No arithmetic of the method
runs here.  There is no fallback: if the library is missing or a tensor is not
a CUDA tensor of the documented dtype/shape, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZOOMR_LIB_OVERRIDE") or os.path.join(_HERE, "libzoomr.so")  # override: A/B builds only

OK, ERR_INVALID_ARG, ERR_DIM_MISMATCH, ERR_EMPTY_SEGMENT, ERR_SEGMENT_ORDER, ERR_INDEX_RANGE, \
    ERR_CAPACITY, ERR_UNSUPPORTED, ERR_CUDA, ERR_WORKSPACE = range(10)
A_FRAC_BITS = 32  # ZOOMR_A_FRAC_BITS

EXPORTS = ("zoomr_update_mean_keys", "zoomr_score", "zoomr_select_topc", "zoomr_build_index",
           "zoomr_attn_workspace_bytes", "zoomr_sparse_decode_attn", "zoomr_select_workspace_bytes",
           "zoomr_select_fused", "zoomr_append_kv", "zoomr_track_segments", "zoomr_shard_index",
           "zoomr_sparse_decode_attn_lse", "zoomr_sparse_decode_attn_lse_chained", "zoomr_merge_attn", "zoomr_sparse_decode_attn_logits",
           "zoomr_h2o_accumulate", "zoomr_h2o_select", "zoomr_tier_workspace_bytes", "zoomr_tier_fetch",
           "zoomr_write_newest_kv", "zoomr_sparse_decode_attn_chained", "zoomr_select_fused_chained",
           "zoomr_select_front", "zoomr_select_tail", "zoomr_tier_gather_slice", "zoomr_append_track",
           "zoomr_status_str", "zoomr_abi_version")


class ZoomrError(RuntimeError):
    def __init__(self, fn, rc):
        super().__init__(f"{fn}: {status_str(rc)} ({rc})")
        self.rc = rc


class Geom(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("page_size", C.c_int32)]


class KV(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("num_pages", C.c_int64),
                ("page_table", C.c_void_p), ("max_pages", C.c_int32)]


class Segments(C.Structure):
    _fields_ = [("bounds", C.c_void_p), ("num_summaries", C.c_void_p), ("seq_len", C.c_void_p),
                ("max_summaries", C.c_int32)]


ABI_VERSION = 9  # include/zoomr.h ZOOMR_ABI_VERSION
_lib = None


def lib():
    """Load libzoomr.so; raise if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA extension is required; there is no fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
        L.zoomr_update_mean_keys.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, vp]
        L.zoomr_score.argtypes = [vp, i32, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        L.zoomr_select_topc.argtypes = [i32, vp, vp, i32, i32, vp, vp, vp, vp]
        L.zoomr_build_index.argtypes = [i32, vp, vp, i32, i32, vp, i32, vp, vp, vp]
        L.zoomr_attn_workspace_bytes.argtypes = [vp, i32]
        L.zoomr_attn_workspace_bytes.restype = sz
        L.zoomr_sparse_decode_attn.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, i32, i32, C.c_float, i32, i32,
                                               vp, vp, sz, vp, vp]
        L.zoomr_sparse_decode_attn_chained.argtypes = L.zoomr_sparse_decode_attn.argtypes
        L.zoomr_select_workspace_bytes.argtypes = [vp, i32, i32]
        L.zoomr_select_workspace_bytes.restype = sz
        L.zoomr_select_fused.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, vp, i32, i32, i32, i32, vp, vp,
                                         vp, vp, vp, i32, vp, vp, vp, vp, sz, vp, vp]
        L.zoomr_select_fused.restype = C.c_int
        L.zoomr_select_front.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, vp, i32, vp, vp, vp, vp, sz, vp, vp]
        L.zoomr_select_front.restype = C.c_int
        L.zoomr_select_tail.argtypes = [vp, i32, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, i32, vp, vp, vp]
        L.zoomr_select_tail.restype = C.c_int
        L.zoomr_append_kv.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.zoomr_append_kv.restype = C.c_int
        L.zoomr_track_segments.argtypes = [i32, vp, i32, i32, vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp]
        L.zoomr_track_segments.restype = C.c_int
        L.zoomr_append_track.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp, i32, i32, vp, i32, vp, vp, vp, i32, vp, vp,
                                         vp, vp, vp]
        L.zoomr_append_track.restype = C.c_int
        L.zoomr_shard_index.argtypes = [i32, vp, vp, i32, vp, i32, i32, vp, vp, vp, vp]
        L.zoomr_shard_index.restype = C.c_int
        L.zoomr_sparse_decode_attn_lse.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, i32, i32, C.c_float, i32, i32,
                                                   vp, vp, vp, sz, vp, vp]
        L.zoomr_sparse_decode_attn_lse.restype = C.c_int
        L.zoomr_sparse_decode_attn_lse_chained.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, i32, i32, C.c_float, i32, i32,
                                                   vp, vp, vp, sz, vp, vp]
        L.zoomr_sparse_decode_attn_lse_chained.restype = C.c_int
        L.zoomr_merge_attn.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp]
        L.zoomr_merge_attn.restype = C.c_int
        L.zoomr_sparse_decode_attn_logits.argtypes = [vp, i32, vp, vp, vp, vp, i32, C.c_float, vp, vp, vp, vp, sz,
                                                      vp, vp]
        L.zoomr_sparse_decode_attn_logits.restype = C.c_int
        L.zoomr_h2o_accumulate.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp, i32, vp, vp, vp, vp]
        L.zoomr_h2o_accumulate.restype = C.c_int
        L.zoomr_h2o_select.argtypes = [i32, vp, vp, i32, vp, i32, vp, i32, i32, i32, vp, vp, vp, vp]
        L.zoomr_h2o_select.restype = C.c_int
        L.zoomr_tier_workspace_bytes.argtypes = [i32, i32, i32]
        L.zoomr_tier_workspace_bytes.restype = sz
        L.zoomr_tier_fetch.argtypes = [vp, i32, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp, sz, vp, vp]
        L.zoomr_tier_fetch.restype = C.c_int
        L.zoomr_tier_gather_slice.argtypes = [vp, i32, vp, vp, vp, i32, i32, i32, vp, vp, i32, i32, vp, vp]
        L.zoomr_tier_gather_slice.restype = C.c_int
        L.zoomr_write_newest_kv.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.zoomr_write_newest_kv.restype = C.c_int
        L.zoomr_status_str.argtypes = [C.c_int]
        L.zoomr_status_str.restype = C.c_char_p
        L.zoomr_abi_version.restype = C.c_int
        for fn in (L.zoomr_update_mean_keys, L.zoomr_score, L.zoomr_select_topc,
                   L.zoomr_build_index, L.zoomr_sparse_decode_attn, L.zoomr_sparse_decode_attn_chained):
            fn.restype = C.c_int
        if L.zoomr_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.zoomr_abi_version()}, this binding expects {ABI_VERSION}: "
                              "rebuild with __graft_entry__.build()")
        _lib = L
    return _lib


def status_str(rc: int) -> str:
    return lib().zoomr_status_str(int(rc)).decode()


def abi_version() -> int:
    return int(lib().zoomr_abi_version())


def _ptr(t, dtype=None, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _check(fn, rc):
    if rc != OK:
        raise ZoomrError(fn, rc)


@dataclass
class Shape:
    """Rank-local model geometry (zoomr_geom)."""
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int

    def c(self) -> Geom:
        return Geom(self.num_layers, self.num_q_heads, self.num_kv_heads, self.head_dim,
                    self.page_size)


def _pool_ptr(t, name, host_ok):
    """A pool's address: a CUDA tensor, or (host_ok) a pinned host tensor read through its unified address."""
    if host_ok and isinstance(t, torch.Tensor) and not t.is_cuda:
        return _host_ptr(t, name)
    return _ptr(t, torch.bfloat16, name)


def _kv(k_pool, v_pool, page_table, host_ok=False):
    if k_pool.shape != v_pool.shape or k_pool.dim() != 5:
        raise ValueError("k/v pools must be [L][num_pages][H_kv][P][d]")
    return KV(_pool_ptr(k_pool, "k_pool", host_ok), _pool_ptr(v_pool, "v_pool", host_ok),
              k_pool.shape[1], _ptr(page_table, torch.int32, "page_table"), page_table.shape[1])


def _seg(bounds, num_summaries, seq_len):
    return Segments(_ptr(bounds, torch.int32, "bounds"), _ptr(num_summaries, torch.int32, "num_summaries"),
                    _ptr(seq_len, torch.int32, "seq_len"), bounds.shape[1])


def update_mean_keys(shape: Shape, k_pool, v_pool, page_table, bounds, num_summaries, seq_len,
                     items, mean_keys, dev_status=None, stream=None):
    """a1 (zoomr_update_mean_keys). items: int32 [n][2] of (b, i)."""
    g, kv, sg = shape.c(), _kv(k_pool, v_pool, page_table), _seg(bounds, num_summaries, seq_len)
    rc = lib().zoomr_update_mean_keys(C.byref(g), bounds.shape[0], C.byref(kv), C.byref(sg),
                                      _ptr(items, torch.int32, "items"), items.shape[0],
                                      _ptr(mean_keys, torch.float32, "mean_keys"),
                                      _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_update_mean_keys", rc)


def score(shape: Shape, q, mean_keys, num_summaries, top_k, partial, alpha_out=None, topk_out=None,
          dev_status=None, stream=None):
    """a2 (zoomr_score). partial: int64 [B][2][max_summaries]."""
    g = shape.c()
    rc = lib().zoomr_score(C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"),
                           _ptr(mean_keys, torch.float32, "mean_keys"),
                           _ptr(num_summaries, torch.int32, "num_summaries"), partial.shape[2],
                           int(top_k), _ptr(partial, torch.int64, "partial"),
                           _ptr(alpha_out, torch.float32, "alpha_out"),
                           _ptr(topk_out, torch.int32, "topk_out"),
                           _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_score", rc)


def select_topc(partial, num_summaries, c, flags, agreeability=None, dev_status=None, stream=None):
    """a3 (zoomr_select_topc). flags: uint8 [B][max_summaries]."""
    rc = lib().zoomr_select_topc(partial.shape[0], _ptr(partial, torch.int64, "partial"),
                                 _ptr(num_summaries, torch.int32, "num_summaries"), partial.shape[2],
                                 int(c), _ptr(flags, torch.uint8, "flags"),
                                 _ptr(agreeability, torch.float32, "agreeability"),
                                 _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_select_topc", rc)


def build_index(bounds, num_summaries, seq_len, flags, sink, window, index, index_count,
                dev_status=None, stream=None):
    """a4 (zoomr_build_index). index: int32 [B][capacity]; index_count int32 [B]."""
    sg = _seg(bounds, num_summaries, seq_len)
    rc = lib().zoomr_build_index(bounds.shape[0], C.byref(sg), _ptr(flags, torch.uint8, "flags"),
                                 int(sink), int(window), _ptr(index, torch.int32, "index"),
                                 index.shape[1], _ptr(index_count, torch.int32, "index_count"),
                                 _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_build_index", rc)


def attn_workspace_bytes(shape: Shape, batch: int) -> int:
    g = shape.c()
    return int(lib().zoomr_attn_workspace_bytes(C.byref(g), int(batch)))


def sparse_decode_attn(shape: Shape, q, k_pool, v_pool, page_table, index, index_count, out,
                       workspace, softmax_scale=None, dev_status=None, stream=None, index_phys=None,
                       seq_len=None, sink=0, window=0, chained=False, layer_begin=0, layer_count=0):
    """a5 (zoomr_sparse_decode_attn). workspace: uint8 CUDA tensor, zeroed once.
    chained: zoomr_sparse_decode_attn_chained (a PDL-launched successor, normally
    select_fused(chained=True) of the next step, may start during this launch).
    layer_begin/layer_count: attend only those layers (0 = through the last).

    seq_len/sink/window (optional): `index` is a4's output for these values, so
    I_p and I_w are attended before the kernel waits for I_f (see zoomr.h)."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table)
    sc = shape.head_dim ** -0.5 if softmax_scale is None else float(softmax_scale)
    fn = lib().zoomr_sparse_decode_attn_chained if chained else lib().zoomr_sparse_decode_attn
    rc = fn(C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"),
                                        C.byref(kv), _ptr(index, torch.int32, "index"),
                                        _ptr(index_phys, torch.int32, "index_phys"),
                                        _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                        _ptr(seq_len, torch.int32, "seq_len"), int(sink), int(window),
                                        C.c_float(sc), int(layer_begin), int(layer_count),
                                        _ptr(out, torch.float32, "out"),
                                        _ptr(workspace, None, "workspace"), workspace.numel() *
                                        workspace.element_size(),
                                        _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_sparse_decode_attn", rc)


def sparse_decode_attn_lse(shape: Shape, q, k_pool, v_pool, page_table, index, index_count, out, lse,
                           workspace, softmax_scale=None, dev_status=None, stream=None, index_phys=None,
                           layer_begin=0, layer_count=0, seq_len=None, sink=0, window=0, chained=False):
    """a5 over any index list, also writing lse fp32 [B][L][H_q] (zoomr_sparse_decode_attn_lse;
    chained: zoomr_sparse_decode_attn_lse_chained)."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table)
    sc = shape.head_dim ** -0.5 if softmax_scale is None else float(softmax_scale)
    fn = lib().zoomr_sparse_decode_attn_lse_chained if chained else lib().zoomr_sparse_decode_attn_lse
    rc = fn(C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"),
                                            C.byref(kv), _ptr(index, torch.int32, "index"),
                                            _ptr(index_phys, torch.int32, "index_phys"),
                                            _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                            _ptr(seq_len, torch.int32, "seq_len"), int(sink), int(window),
                                            C.c_float(sc), int(layer_begin), int(layer_count),
                                            _ptr(out, torch.float32, "out"),
                                            _ptr(lse, torch.float32, "lse"), _ptr(workspace, None, "workspace"),
                                            workspace.numel() * workspace.element_size(),
                                            _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_sparse_decode_attn_lse", rc)


def shard_index(index, index_count, owner, rank, local_index, local_count, dev_status=None, stream=None):
    """I_f restricted to the tokens owned by `rank` (zoomr_shard_index). owner: uint8 [B][stride]."""
    if local_index.shape != index.shape:
        raise ValueError("local_index must have index's shape")
    rc = lib().zoomr_shard_index(index.shape[0], _ptr(index, torch.int32, "index"),
                                 _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                 _ptr(owner, torch.uint8, "owner"), owner.shape[1], int(rank),
                                 _ptr(local_index, torch.int32, "local_index"),
                                 _ptr(local_count, torch.int32, "local_count"),
                                 _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_shard_index", rc)


def merge_attn(shape: Shape, part_out, part_lse, out, part_count=None, lse=None, stream=None):
    """Combine [R][B][L][H_q][d] partial outputs by their lse [R][B][L][H_q] (zoomr_merge_attn)."""
    R, B = part_out.shape[0], part_out.shape[1]
    if part_lse.shape != part_out.shape[:-1] or out.shape != part_out.shape[1:]:
        raise ValueError("merge_attn: part_out [R][B][L][Hq][d], part_lse [R][B][L][Hq], out [B][L][Hq][d]")
    if part_count is not None and tuple(part_count.shape) != (R, B):
        raise ValueError("merge_attn: part_count must be [R][B]")
    g = shape.c()
    rc = lib().zoomr_merge_attn(C.byref(g), B, R, _ptr(part_out, torch.float32, "part_out"),
                                _ptr(part_lse, torch.float32, "part_lse"),
                                _ptr(part_count, torch.int32, "part_count"), _ptr(out, torch.float32, "out"),
                                _ptr(lse, torch.float32, "lse"), _stream(stream))
    _check("zoomr_merge_attn", rc)


def sparse_decode_attn_logits(shape: Shape, q, k_pool, v_pool, page_table, index, index_count, out, lse, logits,
                              workspace, softmax_scale=None, dev_status=None, stream=None):
    """a5 writing also lse [B][L][H_q] and logits [B][L][H_q][cap] (zoomr_sparse_decode_attn_logits)."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table)
    sc = shape.head_dim ** -0.5 if softmax_scale is None else float(softmax_scale)
    if logits.shape[-1] != index.shape[1]:
        raise ValueError("logits' last dimension must be the index capacity")
    rc = lib().zoomr_sparse_decode_attn_logits(C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"), C.byref(kv),
                                               _ptr(index, torch.int32, "index"),
                                               _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                               C.c_float(sc), _ptr(out, torch.float32, "out"),
                                               _ptr(lse, torch.float32, "lse"), _ptr(logits, torch.float32, "logits"),
                                               _ptr(workspace, None, "workspace"),
                                               workspace.numel() * workspace.element_size(),
                                               _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_sparse_decode_attn_logits", rc)


def h2o_accumulate(shape: Shape, index, index_count, logits, lse, score, index_copy=None, count_copy=None,
                   dev_status=None, stream=None):
    """score[b, index[b,i]] += mean_{l,h} exp(logits - lse) (zoomr_h2o_accumulate). score fp32 [B][stride]."""
    g = shape.c()
    rc = lib().zoomr_h2o_accumulate(C.byref(g), index.shape[0], _ptr(index, torch.int32, "index"),
                                    _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                    _ptr(logits, torch.float32, "logits"), _ptr(lse, torch.float32, "lse"),
                                    _ptr(score, torch.float32, "score"), score.shape[1],
                                    _ptr(index_copy, torch.int32, "index_copy"),
                                    _ptr(count_copy, torch.int32, "count_copy"),
                                    _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_h2o_accumulate", rc)


def h2o_select(prev_index, prev_count, score, seq_len, sink, window, budget, index, index_count, dev_status=None,
               stream=None):
    """The next H2O retained set (zoomr_h2o_select)."""
    if prev_index.shape != index.shape:
        raise ValueError("prev_index and index must have the same shape")
    rc = lib().zoomr_h2o_select(index.shape[0], _ptr(prev_index, torch.int32, "prev_index"),
                                _ptr(prev_count, torch.int32, "prev_count"), index.shape[1],
                                _ptr(score, torch.float32, "score"), score.shape[1],
                                _ptr(seq_len, torch.int32, "seq_len"), int(sink), int(window), int(budget),
                                _ptr(index, torch.int32, "index"), _ptr(index_count, torch.int32, "index_count"),
                                _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_h2o_select", rc)


def _host_ptr(t, name):
    """A pinned host tensor's unified address (device-accessible); raises if not pinned."""
    if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_pinned():
        raise TypeError(f"{name} must be a pinned host tensor")
    if t.dtype != torch.bfloat16 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous bf16")
    return C.c_void_p(t.data_ptr())


def tier_workspace_bytes(batch: int, hot_max_pages: int, hot_pages: int) -> int:
    return int(lib().zoomr_tier_workspace_bytes(int(batch), int(hot_max_pages), int(hot_pages)))


def tier_fetch(shape: Shape, host_k, host_v, page_table, hot_k, hot_v, hot_page_table, hot_owner, hot_stamp,
               index, index_count, workspace, dev_status=None, stream=None, seq_len=None):
    """Make the pages of I_f resident in the HBM hot pool (zoomr_tier_fetch). host_k/v: pinned bf16
    [L][pages][H_kv][P][d] (shape.page_size = P); hot_k/v [L][hot_pages][H_kv][Ph][d]."""
    g = shape.c()
    kv = KV(_host_ptr(host_k, "host_k"), _host_ptr(host_v, "host_v"), host_k.shape[1],
            _ptr(page_table, torch.int32, "page_table"), page_table.shape[1])
    rc = lib().zoomr_tier_fetch(C.byref(g), index.shape[0], C.byref(kv), _ptr(hot_k, torch.bfloat16, "hot_k"),
                                _ptr(hot_v, torch.bfloat16, "hot_v"), hot_k.shape[1], hot_k.shape[3],
                                _ptr(hot_page_table, torch.int32, "hot_page_table"),
                                _ptr(hot_owner, torch.int32, "hot_owner"), _ptr(hot_stamp, torch.int32, "hot_stamp"),
                                _ptr(index, torch.int32, "index"), _ptr(index_count, torch.int32, "index_count"),
                                index.shape[1], _ptr(seq_len, torch.int32, "seq_len"),
                                _ptr(workspace, None, "workspace"),
                                workspace.numel() * workspace.element_size(),
                                _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_tier_fetch", rc)


def tier_gather_slice(shape: Shape, host_k, host_v, page_table, index, index_count, layer_begin, layer_count,
                      slice_k, slice_v, dev_status=None, stream=None):
    """Rows of I_f of layers [layer_begin, +layer_count) host -> HBM slice (zoomr_tier_gather_slice).
    slice_k/v: bf16 [layer_count][B * spp][H_kv][Ps][d]."""
    g = shape.c()
    B = index.shape[0]
    if slice_k.dim() != 5 or slice_k.shape != slice_v.shape or slice_k.shape[1] % B:
        raise ValueError("slice_k/v must be [layer_count][B*spp][H_kv][Ps][d]")
    kv = KV(_host_ptr(host_k, "host_k"), _host_ptr(host_v, "host_v"), host_k.shape[1],
            _ptr(page_table, torch.int32, "page_table"), page_table.shape[1])
    rc = lib().zoomr_tier_gather_slice(C.byref(g), B, C.byref(kv), _ptr(index, torch.int32, "index"),
                                       _ptr(index_count, torch.int32, "index_count"), index.shape[1],
                                       int(layer_begin), int(layer_count), _ptr(slice_k, torch.bfloat16, "slice_k"),
                                       _ptr(slice_v, torch.bfloat16, "slice_v"), slice_k.shape[3],
                                       slice_k.shape[1] // B, _ptr(dev_status, torch.int32, "dev_status"),
                                       _stream(stream))
    _check("zoomr_tier_gather_slice", rc)


def select_workspace_bytes(shape: Shape, batch: int, max_summaries: int) -> int:
    g = shape.c()
    return int(lib().zoomr_select_workspace_bytes(C.byref(g), int(batch), int(max_summaries)))


def select_fused(shape: Shape, q, k_pool, v_pool, page_table, bounds, num_summaries, seq_len, close_items,
                 mean_keys, top_k, c, sink, window, flags, index, index_count, workspace, partial=None,
                 agreeability=None, alpha_out=None, topk_out=None, dev_status=None, stream=None,
                 index_phys=None, update=None, chained=False):
    """a1+a2+a3+a4 in one launch (zoomr_select_fused). close_items: int32 [n][2] or None
    (entries with i < 0 are skipped); update: uint8 [B] or None (0 = keep the flags).
    chained: zoomr_select_fused_chained -- the preceding kernel on the stream is a
    chained a5 (or writes none of a1/a2's inputs); a1/a2 overlap its end."""
    g, kv, sg = shape.c(), _kv(k_pool, v_pool, page_table, host_ok=True), _seg(bounds, num_summaries, seq_len)
    n_close = 0 if close_items is None else close_items.shape[0]
    rc = (lib().zoomr_select_fused_chained if chained else lib().zoomr_select_fused)(
        C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"), C.byref(kv), C.byref(sg),
        _ptr(close_items, torch.int32, "close_items") if n_close else None, n_close,
        _ptr(update, torch.uint8, "update"), _ptr(mean_keys, torch.float32, "mean_keys"), int(top_k), int(c), int(sink), int(window),
        _ptr(partial, torch.int64, "partial"), _ptr(flags, torch.uint8, "flags"),
        _ptr(agreeability, torch.float32, "agreeability"), _ptr(index, torch.int32, "index"),
        _ptr(index_phys, torch.int32, "index_phys"), index.shape[1],
        _ptr(index_count, torch.int32, "index_count"), _ptr(alpha_out, torch.float32, "alpha_out"),
        _ptr(topk_out, torch.int32, "topk_out"), _ptr(workspace, None, "workspace"),
        workspace.numel() * workspace.element_size(), _ptr(dev_status, torch.int32, "dev_status"),
        _stream(stream))
    _check("zoomr_select_fused", rc)


def select_front(shape: Shape, q, k_pool, v_pool, page_table, bounds, num_summaries, seq_len, close_items,
                 mean_keys, top_k, partial, workspace, alpha_out=None, topk_out=None, dev_status=None, update=None,
                 stream=None):
    """a1 + a2 with aggregation into partial int64 [B][2][max_summaries] (zoomr_select_front)."""
    g, kv, sg = shape.c(), _kv(k_pool, v_pool, page_table), _seg(bounds, num_summaries, seq_len)
    n_close = 0 if close_items is None else close_items.shape[0]
    rc = lib().zoomr_select_front(
        C.byref(g), q.shape[0], _ptr(q, torch.bfloat16, "q"), C.byref(kv), C.byref(sg),
        _ptr(close_items, torch.int32, "close_items") if n_close else None, n_close,
        _ptr(update, torch.uint8, "update"), _ptr(mean_keys, torch.float32, "mean_keys"), int(top_k),
        _ptr(partial, torch.int64, "partial"), _ptr(alpha_out, torch.float32, "alpha_out"),
        _ptr(topk_out, torch.int32, "topk_out"), _ptr(workspace, None, "workspace"),
        workspace.numel() * workspace.element_size(), _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_select_front", rc)


def select_tail(shape: Shape, bounds, num_summaries, seq_len, partial, c, sink, window, flags, index, index_count,
                agreeability=None, dev_status=None, update=None, page_table=None, index_phys=None, stream=None):
    """a3 + a4 from a (reduced) partial (zoomr_select_tail)."""
    g, sg = shape.c(), _seg(bounds, num_summaries, seq_len)
    kv = None
    if index_phys is not None:
        kv = KV(None, None, 1, _ptr(page_table, torch.int32, "page_table"), page_table.shape[1])
    rc = lib().zoomr_select_tail(
        C.byref(g), partial.shape[0], C.byref(kv) if kv is not None else None, C.byref(sg),
        _ptr(partial, torch.int64, "partial"), _ptr(update, torch.uint8, "update"), int(c), int(sink), int(window),
        _ptr(flags, torch.uint8, "flags"), _ptr(agreeability, torch.float32, "agreeability"),
        _ptr(index, torch.int32, "index"), _ptr(index_phys, torch.int32, "index_phys"), index.shape[1],
        _ptr(index_count, torch.int32, "index_count"), _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_select_tail", rc)


def append_kv(shape: Shape, k_pool, v_pool, page_table, k_new, v_new, seq_len, dev_status=None, stream=None):
    """a0 (zoomr_append_kv): rows k_new / v_new bf16 [B][L][H_kv][d] at position seq_len[b]; seq_len += 1.
    The pools may be pinned host tensors (the host tier)."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table, host_ok=True)
    rc = lib().zoomr_append_kv(C.byref(g), k_new.shape[0], C.byref(kv), _ptr(k_new, torch.bfloat16, "k_new"),
                               _ptr(v_new, torch.bfloat16, "v_new"), _ptr(seq_len, torch.int32, "seq_len"),
                               _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_append_kv", rc)


def write_newest_kv(shape: Shape, k_pool, v_pool, page_table, k_new, v_new, seq_len, dev_status=None, stream=None):
    """The newest token's rows at position seq_len[b] - 1 (zoomr_write_newest_kv); seq_len unchanged."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table)
    rc = lib().zoomr_write_newest_kv(C.byref(g), k_new.shape[0], C.byref(kv), _ptr(k_new, torch.bfloat16, "k_new"),
                                     _ptr(v_new, torch.bfloat16, "v_new"), _ptr(seq_len, torch.int32, "seq_len"),
                                     _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_write_newest_kv", rc)


def append_track(shape: Shape, k_pool, v_pool, page_table, k_new, v_new, token_ids, begin_id, end_id, boundary_ids,
                 seq_len, bounds, num_summaries, state, close_items, update, dev_status=None, stream=None,
                 mirror=None, mirror_page_size=0):
    """zoomr_append_track: append_kv + track_segments without a host round trip (PDL
    behind a chained a5).  The pools may be pinned host tensors (the host tier);
    mirror = (k, v, page_table) of a second pool (page size mirror_page_size) that
    also gets the rows where their page is resident (the tier's HBM hot pool)."""
    g, kv = shape.c(), _kv(k_pool, v_pool, page_table, host_ok=True)
    mkv = _kv(*mirror) if mirror is not None else None
    nb = 0 if boundary_ids is None else boundary_ids.numel()
    rc = lib().zoomr_append_track(
        C.byref(g), k_new.shape[0], C.byref(kv), C.byref(mkv) if mkv is not None else None, int(mirror_page_size),
        _ptr(k_new, torch.bfloat16, "k_new"), _ptr(v_new, torch.bfloat16, "v_new"),
        _ptr(token_ids, torch.int32, "token_ids"), int(begin_id), int(end_id),
        _ptr(boundary_ids, torch.int32, "boundary_ids") if nb else None, nb, _ptr(seq_len, torch.int32, "seq_len"),
        _ptr(bounds, torch.int32, "bounds"), _ptr(num_summaries, torch.int32, "num_summaries"), bounds.shape[1],
        _ptr(state, torch.int32, "state"), _ptr(close_items, torch.int32, "close_items"),
        _ptr(update, torch.uint8, "update"), _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_append_track", rc)


def track_segments(token_ids, begin_id, end_id, boundary_ids, seq_len, bounds, num_summaries, state,
                   close_items, update, dev_status=None, stream=None):
    """zoomr_track_segments: summary delimiters / semantic boundaries of the token just appended."""
    nb = 0 if boundary_ids is None else boundary_ids.numel()
    rc = lib().zoomr_track_segments(
        token_ids.shape[0], _ptr(token_ids, torch.int32, "token_ids"), int(begin_id), int(end_id),
        _ptr(boundary_ids, torch.int32, "boundary_ids") if nb else None, nb, _ptr(seq_len, torch.int32, "seq_len"),
        _ptr(bounds, torch.int32, "bounds"), _ptr(num_summaries, torch.int32, "num_summaries"), bounds.shape[1],
        _ptr(state, torch.int32, "state"), _ptr(close_items, torch.int32, "close_items"),
        _ptr(update, torch.uint8, "update"), _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    _check("zoomr_track_segments", rc)


# ---- NVTX: one range per enqueued stage (host-side marks; visible to ncu --nvtx / nsys) ----------
_STAGES = {
    "update_mean_keys": "a1", "score": "a2", "select_topc": "a3", "build_index": "a4",
    "sparse_decode_attn": "a5", "select_fused": "a1-a4", "select_front": "a1-a2", "select_tail": "a3-a4", "append_kv": "a0", "track_segments": "a0",
    "shard_index": "a4-shard", "sparse_decode_attn_lse": "a5-lse", "merge_attn": "a5-merge",
    "sparse_decode_attn_logits": "a5-logits", "h2o_accumulate": "h2o", "h2o_select": "h2o",
    "tier_fetch": "tier", "write_newest_kv": "a0-tier", "append_track": "a0", "tier_gather_slice": "tier-slice",
}


def _nvtx_wrap(fn, label):
    import functools

    @functools.wraps(fn)
    def w(*a, **k):
        torch.cuda.nvtx.range_push(label)
        try:
            return fn(*a, **k)
        finally:
            torch.cuda.nvtx.range_pop()
    return w


if os.environ.get("ZOOMR_NVTX", "1") != "0":
    for _n, _s in _STAGES.items():
        globals()[_n] = _nvtx_wrap(globals()[_n], f"{_s} zoomr_{_n}")
