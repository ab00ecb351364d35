"""ZoomR step over a host-memory KV cache.

The paper keeps the full cache in CPU memory and loads the index set per step
(P:103-109).  Here the full cache is a pinned host tensor read by the kernels
through its unified address, and an HBM hot pool caches its pages: per step
the selection (a2..a4) runs as usual, `zoomr_tier_fetch` brings in the pages
of I_f that are not resident (LRU replacement among the pages the step does
not touch), and a5 runs on the hot pool.  Marshalling only; the work is the
libzoomr kernels.
"""
from __future__ import annotations

import torch

from . import zoomr as Z
from .step import StepParams, ZoomrStep


class HostTierStep(ZoomrStep):
    def __init__(self, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int, params: StepParams,
                 host_k: torch.Tensor, host_v: torch.Tensor, page_table: torch.Tensor, hot_pages: int,
                 device="cuda", hot_page_size: int = 0):
        """shape: the host cache's geometry (page_size = P).  hot_page_size (default P) divides P:
        smaller hot pages hold I_f with less HBM (a summary drags in Ph tokens, not P)."""
        P = shape.page_size
        Ph = hot_page_size or P
        if P % Ph:
            raise ValueError("hot_page_size must divide the host page size")
        self.host_shape = shape
        shape_hot = Z.Shape(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, Ph)
        super().__init__(shape_hot, batch, max_summaries, index_capacity, params, device, early_known=False)
        if not (host_k.is_pinned() and host_v.is_pinned()):
            raise TypeError("the host tier needs pinned host tensors")
        dev = self.out.device
        L, Hkv, d = shape.num_layers, shape.num_kv_heads, shape.head_dim
        hmp = page_table.shape[1] * (P // Ph)
        self.host_k, self.host_v, self.page_table = host_k, host_v, page_table
        self.hot_k = torch.zeros(L, hot_pages, Hkv, Ph, d, dtype=torch.bfloat16, device=dev)
        self.hot_v = torch.zeros_like(self.hot_k)
        self.hot_page_table = torch.full((batch, hmp), -1, dtype=torch.int32, device=dev)
        self.hot_owner = torch.full((hot_pages,), -1, dtype=torch.int32, device=dev)
        self.hot_stamp = torch.full((hot_pages,), -1, dtype=torch.int32, device=dev)
        self.tier_ws = torch.zeros(Z.tier_workspace_bytes(batch, hmp, hot_pages), dtype=torch.uint8, device=dev)
        self.lse = torch.zeros(batch, L, shape.num_q_heads, dtype=torch.float32, device=dev)

    @property
    def hot_kv(self):
        return (self.hot_k, self.hot_v, self.hot_page_table)

    def update_mean_keys_hot(self, seg, items: torch.Tensor):
        """a1 on the hot pool: a summary closes at the newest tokens, inside the window, whose
        pages every step's I_f keeps resident."""
        self.update_mean_keys(self.hot_kv, seg, items)

    def fetched_pages(self) -> int:
        """Pages copied from the host by the last fetch (reads the device; for reporting)."""
        return int(self.tier_ws[4:8].view(torch.int32).item())

    def run(self, q, seg, update_selection: bool = True):
        bounds, nsum, seq_len = seg
        p = self.params
        if update_selection:  # a2..a4 (the caller's a1 keeps the mean keys current)
            Z.select_fused(self.shape, q, self.hot_k, self.hot_v, self.hot_page_table, bounds, nsum, seq_len, None,
                           self.mean_keys, p.top_k, p.c, p.sink, p.window, self.flags, self.index, self.count,
                           self.sel_workspace, partial=self.partial, agreeability=self.agreeability,
                           alpha_out=self.alpha, topk_out=self.topk, dev_status=self.status)
        else:
            Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count, self.status)
        Z.tier_fetch(self.host_shape, self.host_k, self.host_v, self.page_table, self.hot_k, self.hot_v,
                     self.hot_page_table, self.hot_owner, self.hot_stamp, self.index, self.count, self.tier_ws,
                     self.status)
        Z.sparse_decode_attn_lse(self.shape, q, self.hot_k, self.hot_v, self.hot_page_table, self.index, self.count,
                                 self.out, self.lse, self.workspace, dev_status=self.status)
        return self.out

    def launches_per_step(self, *args, **kwargs) -> int:
        return 4  # select, plan, copy, a5
