"""One ZoomR decode step on the device: a1 -> a2 -> [all-reduce] -> a3 -> a4 -> a5.

Owns the step's device buffers (mean-key cache, partial votes, flags, index
set, output, attention workspace) and enqueues the five libzoomr kernels in
Algorithm 1's order.  Optionally captures the whole step in a CUDA
graph so a decode step is one graph launch.  Marshalling and scheduling only:
every arithmetic step runs in the CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch

from . import zoomr as Z


@dataclass
class StepParams:
    top_k: int
    c: int
    sink: int
    window: int


class ZoomrStep:
    """Device state + launch sequence of one (rank-local) decode step."""

    def __init__(self, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int,
                 params: StepParams, device="cuda", debug_outputs: bool = False, use_phys: bool = False,
                 early_known: bool = True, chained: bool = False):
        self.shape, self.batch, self.params = shape, batch, params
        # steps enqueued back to back (several per CUDA graph): the fused select of
        # step t+1 runs a1/a2 while a5 of step t finishes (zoomr_*_chained)
        # (libzoomr checks the launch order itself: after anything but a chained a5 the
        # chained select runs like the plain one, and an a5 right behind a chained a5 on
        # the same workspace attends index-only -- zoomr.h "Chained launches")
        self.chained = chained
        self.max_summaries, self.cap = max_summaries, index_capacity
        dev = torch.device(device)
        L, Hq, Hkv, d = shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
        self.mean_keys = torch.zeros(batch, L, Hkv, max_summaries, d, dtype=torch.float32, device=dev)
        self.partial = torch.zeros(batch, 2, max_summaries, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(batch, max_summaries, dtype=torch.uint8, device=dev)
        self.index = torch.zeros(batch, index_capacity, dtype=torch.int32, device=dev)
        self.index_phys = torch.zeros(batch, index_capacity, dtype=torch.int32, device=dev)
        self.count = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.out = torch.zeros(batch, L, Hq, d, dtype=torch.float32, device=dev)
        self.agreeability = torch.zeros(batch, dtype=torch.float32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = Z.attn_workspace_bytes(shape, batch)
        self.workspace = torch.zeros(max(ws, 1), dtype=torch.uint8, device=dev)
        ws2 = Z.select_workspace_bytes(shape, batch, max_summaries)
        self.sel_workspace = torch.zeros(max(ws2, 1), dtype=torch.uint8, device=dev)
        self.alpha = self.topk = None
        if debug_outputs:
            self.alpha = torch.zeros(batch, L, Hq, max_summaries, dtype=torch.float32, device=dev)
            self.topk = torch.zeros(batch, L * Hq, params.top_k, dtype=torch.int32, device=dev)
        self.graph = None
        self.use_phys = use_phys  # fused select writes page-resolved rows for a5
        self.early_known = early_known  # a5 attends I_p, I_w before waiting for I_f

    # -- a1: mean keys for a list of closed summaries (b, i) --------------------
    def update_mean_keys(self, kv, seg, items: torch.Tensor):
        k_pool, v_pool, page_table = kv
        bounds, nsum, seq_len = seg
        Z.update_mean_keys(self.shape, k_pool, v_pool, page_table, bounds, nsum, seq_len, items,
                           self.mean_keys, self.status)

    @staticmethod
    def all_items(num_summaries: torch.Tensor) -> torch.Tensor:
        """(b, i) for every closed summary (host-side list for the initial cache build)."""
        ns = num_summaries.cpu().tolist()
        items = [(b, i) for b, n in enumerate(ns) for i in range(n)]
        t = torch.tensor(items if items else [[0, 0]], dtype=torch.int32)
        return t[: len(items)].to(num_summaries.device)

    # -- the step ----------------------------------------------------------------
    def run(self, q, kv, seg, update_selection: bool = True, close_items: Optional[torch.Tensor] = None,
            allreduce: Optional[Callable[[torch.Tensor], None]] = None, fused: bool = True):
        """Enqueue one decode step on the current stream.

        close_items: summaries that closed since the last step (a1, amortized).
        update_selection: run a2/a3 (a semantic-boundary / every-U step);
            otherwise the held flags are reused and only a4/a5 run (reading Q14).
        allreduce: the KV-head-sharded exchange of `partial` (sum over ranks).
        """
        k_pool, v_pool, page_table = kv
        bounds, nsum, seq_len = seg
        p = self.params
        if fused and update_selection and allreduce is None:
            # a1..a4 in one launch (zoomr_select_fused), then a5
            Z.select_fused(self.shape, q, k_pool, v_pool, page_table, bounds, nsum, seq_len,
                           close_items if close_items is not None and close_items.numel() else None,
                           self.mean_keys, p.top_k, p.c, p.sink, p.window, self.flags, self.index,
                           self.count, self.sel_workspace, partial=self.partial,
                           agreeability=self.agreeability, alpha_out=self.alpha, topk_out=self.topk,
                           dev_status=self.status, index_phys=self.index_phys if self.use_phys else None,
                           chained=self.chained)
            self.attend(q, kv, seq_len, chained=self.chained)
            return self.out
        if fused and update_selection:
            # KV-head-sharded: a1 + a2 (zoomr_select_front) -> all-reduce of
            # the partial -> a3 + a4 (zoomr_select_tail), then a5 (early rows overlap the tail)
            Z.select_front(self.shape, q, k_pool, v_pool, page_table, bounds, nsum, seq_len,
                           close_items if close_items is not None and close_items.numel() else None,
                           self.mean_keys, p.top_k, self.partial, self.sel_workspace, alpha_out=self.alpha,
                           topk_out=self.topk, dev_status=self.status)
            allreduce(self.partial)
            Z.select_tail(self.shape, bounds, nsum, seq_len, self.partial, p.c, p.sink, p.window, self.flags,
                          self.index, self.count, agreeability=self.agreeability, dev_status=self.status)
            self.attend(q, kv, seq_len, phys=False)
            return self.out
        if close_items is not None and close_items.numel():
            self.update_mean_keys(kv, seg, close_items)
        if update_selection:
            Z.score(self.shape, q, self.mean_keys, nsum, p.top_k, self.partial, self.alpha, self.topk,
                    self.status)
            if allreduce is not None:
                allreduce(self.partial)
            Z.select_topc(self.partial, nsum, p.c, self.flags, self.agreeability, self.status)
        Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count,
                      self.status)
        self.attend(q, kv, seq_len, phys=False)
        return self.out

    def attend(self, q, kv, seq_len, phys=None, chained=False):
        """a5 over the current I_f.  With early_known, I_p and I_w (known from
        T alone) are attended while the producer of I_f is still running."""
        k_pool, v_pool, page_table = kv
        use_phys = self.use_phys if phys is None else phys
        p = self.params
        Z.sparse_decode_attn(self.shape, q, k_pool, v_pool, page_table, self.index, self.count,
                             self.out, self.workspace, dev_status=self.status,
                             index_phys=self.index_phys if use_phys else None,
                             seq_len=seq_len if self.early_known else None, sink=p.sink, window=p.window,
                             chained=chained)

    def launches_per_step(self, update_selection=True, close=False, fused=True, sharded=False) -> int:
        """Kernel launches of libzoomr one run() enqueues (a2 = zero + score when not fused;
        the head-sharded fused path: front + tail + a5, plus the caller's all-reduce)."""
        if fused and update_selection:
            return 3 if sharded else 2
        return (1 if close else 0) + (3 if update_selection else 0) + 2

    def capture(self, q, kv, seg, update_selection=True, close_items=None, allreduce=None, fused=True, steps=1):
        """Capture `steps` back-to-back run()s into a CUDA graph (one launch per replay)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):  # warm-up outside the graph (sets kernel attributes)
                self.run(q, kv, seg, update_selection, close_items, allreduce, fused)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(steps):
                self.run(q, kv, seg, update_selection, close_items, allreduce, fused)
        return g

    def check_status(self):
        st = int(self.status.item())
        if st:
            raise Z.ZoomrError("device status", st)


class DecodeLoop(ZoomrStep):
    """Algorithm 1's whole decode step on the device:

        a0 append k_t, v_t        zoomr_append_track       (row copy + tracking kernel
        segment tracking                                    chained by PDL, T += 1:
                                                            delimiters -> segment table,
                                                            closed summary -> a1 item,
                                                            boundary token -> update flag)
        a1..a4                    zoomr_select_fused       (a2/a3 only where update[b])
        a5                        zoomr_sparse_decode_attn (early rows; chained: its end
                                                            overlaps the next a0)

    No host decision in between, so a step is one CUDA-graph replay.  The
    segment table, N_t and T live on the device (`bounds`, `num_summaries`,
    `seq_len`), initialised from the prompt by `start()`.  fused_a0=False issues
    zoomr_append_kv + zoomr_track_segments instead (same results)."""

    def __init__(self, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int,
                 params: StepParams, begin_id: int, end_id: int, boundary_ids, device="cuda",
                 debug_outputs: bool = False, early_known: bool = True, chained: bool = True,
                 fused_a0: bool = True):
        super().__init__(shape, batch, max_summaries, index_capacity, params, device, debug_outputs,
                         early_known=early_known, chained=chained)
        self.fused_a0 = fused_a0
        dev = torch.device(device)
        self.begin_id, self.end_id = int(begin_id), int(end_id)
        self.boundary_ids = torch.as_tensor(list(boundary_ids), dtype=torch.int32, device=dev)
        self.bounds = torch.zeros(batch, max_summaries, 4, dtype=torch.int32, device=dev)
        self.num_summaries = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.seq_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.track_state = torch.zeros(batch, 4, dtype=torch.int32, device=dev)
        self.close_items = torch.zeros(batch, 2, dtype=torch.int32, device=dev)
        self.update = torch.zeros(batch, dtype=torch.uint8, device=dev)

    def start(self, prompt_len):
        """After a prefill of `prompt_len` tokens (already in the pool): no summaries yet."""
        n = torch.as_tensor(prompt_len, dtype=torch.int32, device=self.seq_len.device).expand(self.batch)
        self.seq_len.copy_(n)
        self.num_summaries.zero_()
        self.bounds.zero_()
        self.flags.zero_()
        self.track_state.copy_(torch.stack([torch.full_like(n, -1), n, n, n], dim=1))

    def start_from(self, bounds, num_summaries, seq_len):
        """Continue an existing context: its segment table, N_t and T (device tensors); the
        open tail starts after the last closed summary.  Mean keys must already be cached."""
        self.bounds.copy_(bounds)
        self.num_summaries.copy_(num_summaries)
        self.seq_len.copy_(seq_len)
        self.flags.zero_()
        last = torch.clamp(num_summaries.long() - 1, min=0)
        tail = torch.where(num_summaries > 0, bounds[torch.arange(self.batch, device=bounds.device), last, 3],
                           torch.zeros_like(num_summaries))
        self.track_state.copy_(torch.stack([torch.full_like(tail, -1), tail, tail, tail], dim=1))

    def decode_step(self, kv, k_new, v_new, q, token_ids):
        """Enqueue one step; k_new/v_new bf16 [B][L][H_kv][d], q bf16 [B][L][H_q][d], token_ids int32 [B]."""
        k_pool, v_pool, page_table = kv
        p = self.params
        if self.fused_a0:
            Z.append_track(self.shape, k_pool, v_pool, page_table, k_new, v_new, token_ids, self.begin_id,
                           self.end_id, self.boundary_ids, self.seq_len, self.bounds, self.num_summaries,
                           self.track_state, self.close_items, self.update, self.status)
        else:
            Z.append_kv(self.shape, k_pool, v_pool, page_table, k_new, v_new, self.seq_len, self.status)
            Z.track_segments(token_ids, self.begin_id, self.end_id, self.boundary_ids, self.seq_len, self.bounds,
                             self.num_summaries, self.track_state, self.close_items, self.update, self.status)
        Z.select_fused(self.shape, q, k_pool, v_pool, page_table, self.bounds, self.num_summaries, self.seq_len,
                       self.close_items, self.mean_keys, p.top_k, p.c, p.sink, p.window, self.flags, self.index,
                       self.count, self.sel_workspace, partial=self.partial, agreeability=self.agreeability,
                       alpha_out=self.alpha, topk_out=self.topk, dev_status=self.status, update=self.update)
        self.attend(q, kv, self.seq_len, chained=self.chained)
        return self.out
