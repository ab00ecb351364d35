"""B200-native (sm_100a) ZoomR select + sparse-decode hot path (arXiv 2604.10898).

Public API:
  zoomr       -- thin ctypes binding of libzoomr.so (include/zoomr.h), same names
  step        -- ZoomrStep: device buffers + the a1..a5 launch sequence / CUDA graph
  parallel    -- batch sharding and KV-head sharding over torch.distributed

There is no CPU fallback: importing `zoomr` functions works without a GPU, but
every call requires CUDA tensors and the built libzoomr.so.
"""
from . import zoomr  # noqa: F401

__all__ = ["zoomr"]
