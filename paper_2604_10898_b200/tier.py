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


class TierDecodeLoop(HostTierStep):
    """Algorithm 1's whole decode step over the host tier, one CUDA-graph replay:

        a0 append k_t, v_t        zoomr_append_track: into the HOST cache (write-through,
        + segment tracking        T += 1) and, mirrored, into the token's hot page when it
                                  is resident (after a warm step it is: the previous fetch
                                  made the page of T resident, look-ahead); the tracking
                                  kernel chained by PDL
        a1..a4                    zoomr_select_fused (a1 reads the closing summary's rows from
                                  the host cache; a2/a3 only at semantic boundaries)
        tier fetch                zoomr_tier_fetch (pages that entered I_f + the look-ahead page)
        a5                        zoomr_sparse_decode_attn_lse on the hot pool, with the
                                  early rows (sink / window before the wait) once warm
    """

    def __init__(self, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int, params: StepParams,
                 host_k, host_v, page_table, hot_pages: int, begin_id: int, end_id: int, boundary_ids,
                 device="cuda", hot_page_size: int = 0, chained: bool = True):
        super().__init__(shape, batch, max_summaries, index_capacity, params, host_k, host_v, page_table, hot_pages,
                         device, hot_page_size)
        self.chained = chained
        dev = self.out.device
        self.begin_id, self.end_id = int(begin_id), int(end_id)
        self.boundary_ids = torch.as_tensor(list(boundary_ids), dtype=torch.int32, device=dev)
        self.bounds = torch.zeros(batch, max_summaries, 4, dtype=torch.int32, device=dev)
        self.num_summaries = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.seq_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.track_state = torch.zeros(batch, 4, dtype=torch.int32, device=dev)
        self.close_items = torch.zeros(batch, 2, dtype=torch.int32, device=dev)
        self.update = torch.zeros(batch, dtype=torch.uint8, device=dev)
        self._warm = False  # a step has run since start(): sink / window pages are resident

    def start(self, prompt_len):
        """After a prefill of `prompt_len` tokens (already in the host cache): no summaries yet."""
        self._warm = False
        n = torch.as_tensor(prompt_len, dtype=torch.int32, device=self.seq_len.device).expand(self.batch)
        self.seq_len.copy_(n)
        self.num_summaries.zero_()
        self.bounds.zero_()
        self.flags.zero_()
        self.track_state.copy_(torch.stack([torch.full_like(n, -1), n, n, n], dim=1))

    def start_from(self, bounds, num_summaries, seq_len):
        """Continue an existing context (its segment table, N_t, T); mean keys must be cached."""
        self._warm = False
        self.bounds.copy_(bounds)
        self.num_summaries.copy_(num_summaries)
        self.seq_len.copy_(seq_len)
        self.flags.zero_()
        last = torch.clamp(num_summaries.long() - 1, min=0)
        tail = torch.where(num_summaries > 0, bounds[torch.arange(self.batch, device=bounds.device), last, 3],
                           torch.zeros_like(num_summaries))
        self.track_state.copy_(torch.stack([torch.full_like(tail, -1), tail, tail, tail], dim=1))

    def decode_step(self, k_new, v_new, q, token_ids):
        """One token.  From the second step after start() / start_from() on, a5 attends
        the sink and window rows before its wait (their hot pages are resident: the
        previous step's fetch kept the next token's page resident, look-ahead)."""
        p, hs = self.params, self.host_shape
        early = self._warm
        # append into the host cache (write-through, T += 1) and into the token's hot page
        # when it is resident (after a warm step it is; else the fetch brings it), then
        # the segment tracking -- one call
        # (a separate zoomr_write_newest_kv after the tracking: +2.1 us per token, same-box A/B)
        Z.append_track(hs, self.host_k, self.host_v, self.page_table, k_new, v_new, token_ids, self.begin_id,
                       self.end_id, self.boundary_ids, self.seq_len, self.bounds, self.num_summaries,
                       self.track_state, self.close_items, self.update, self.status,
                       mirror=(self.hot_k, self.hot_v, self.hot_page_table), mirror_page_size=self.shape.page_size)
        Z.select_fused(hs, q, self.host_k, self.host_v, self.page_table, self.bounds, self.num_summaries,
                       self.seq_len, self.close_items, self.mean_keys, p.top_k, p.c, p.sink, p.window, self.flags,
                       self.index, self.count, self.sel_workspace, partial=self.partial,
                       agreeability=self.agreeability, alpha_out=self.alpha, topk_out=self.topk,
                       dev_status=self.status, update=self.update)
        Z.tier_fetch(hs, self.host_k, self.host_v, self.page_table, self.hot_k, self.hot_v, self.hot_page_table,
                     self.hot_owner, self.hot_stamp, self.index, self.count, self.tier_ws, self.status,
                     seq_len=self.seq_len)  # (look-ahead: the next token's page)
        Z.sparse_decode_attn_lse(self.shape, q, self.hot_k, self.hot_v, self.hot_page_table, self.index, self.count,
                                 self.out, self.lse, self.workspace, dev_status=self.status,
                                 seq_len=self.seq_len if early else None, sink=p.sink, window=p.window,
                                 chained=self.chained)  # (the next token's row copy may overlap its end)
        self._warm = True
        return self.out


class LayerPipelinedTierStep(ZoomrStep):
    """The paper's own system, as P:105-109 describes it:
    the whole cache in (pinned) host memory; each step, after the selection,
    "for each layer of the model, the required KV cache slices are transferred
    to the GPU" and "the KVs for the next layer are prefetched" while the layer
    attends.  Per group of `layers_per_slice` layers:

        copy stream     zoomr_tier_gather_slice (rows of I_f, host -> HBM slice)
        compute stream  a5 on the slice (identity page table, index 0..|I_f|-1)

    with two slice buffers (peak residency: the slice being attended + the one
    being prefetched), events ordering every reuse.  The new
    token's K/V reach the host cache through zoomr_append_kv (write-through,
    TierDecodeLoop) -- in this step-level class the cache is given.  Batch 1,
    the paper's setting (q / out of a layer group are then contiguous views).
    pipelined=False runs the same launches back to back on one stream (the
    serial schedule SPEC's simulator compares against).
    """

    def __init__(self, shape: Z.Shape, max_summaries: int, index_capacity: int, params: StepParams,
                 host_k: torch.Tensor, host_v: torch.Tensor, page_table: torch.Tensor, layers_per_slice: int = 1,
                 slice_page_size: int = 64, device="cuda"):
        super().__init__(shape, 1, max_summaries, index_capacity, params, device, early_known=False)
        if not (host_k.is_pinned() and host_v.is_pinned()):
            raise TypeError("the host tier needs pinned host tensors")
        L, Hq, Hkv, d = shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
        if L % layers_per_slice:
            raise ValueError("layers_per_slice must divide the layer count")
        dev = self.out.device
        self.host_k, self.host_v, self.page_table = host_k, host_v, page_table
        self.Lg, self.Ps = layers_per_slice, slice_page_size
        spp = (index_capacity + slice_page_size - 1) // slice_page_size
        self.slices = [(torch.zeros(self.Lg, spp, Hkv, slice_page_size, d, dtype=torch.bfloat16, device=dev),
                        torch.zeros(self.Lg, spp, Hkv, slice_page_size, d, dtype=torch.bfloat16, device=dev))
                       for _ in range(2)]
        self.slice_pt = torch.arange(spp, dtype=torch.int32, device=dev).view(1, spp)
        self.iota = torch.arange(index_capacity, dtype=torch.int32, device=dev).view(1, index_capacity)
        self.slice_shape = Z.Shape(self.Lg, Hq, Hkv, d, slice_page_size)
        self.slice_ws = [torch.zeros(max(Z.attn_workspace_bytes(self.slice_shape, 1), 1), dtype=torch.uint8,
                                     device=dev) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=dev)
        ng = L // self.Lg
        self.ev_ready = [torch.cuda.Event() for _ in range(ng)]
        self.ev_free = [torch.cuda.Event() for _ in range(ng)]

    def hbm_bytes(self) -> int:
        """HBM the tier needs besides q / out: the two slices + the mean-key cache + index."""
        return sum(t.numel() * t.element_size() for pair in self.slices for t in pair) + \
            self.mean_keys.numel() * 4 + self.index.numel() * 4

    def select(self, q, seg, close_items=None):
        bounds, nsum, seq_len = seg
        p = self.params
        Z.select_fused(self.shape, q, self.host_k, self.host_v, self.page_table, bounds, nsum, seq_len,
                       close_items if close_items is not None and close_items.numel() else None, self.mean_keys,
                       p.top_k, p.c, p.sink, p.window, self.flags, self.index, self.count, self.sel_workspace,
                       partial=self.partial, agreeability=self.agreeability, dev_status=self.status)

    def gather(self, g, stream=None):
        sk, sv = self.slices[g % 2]
        Z.tier_gather_slice(self.shape, self.host_k, self.host_v, self.page_table, self.index, self.count,
                            g * self.Lg, self.Lg, sk, sv, dev_status=self.status, stream=stream)

    def attend_group(self, q, g, stream=None):
        sk, sv = self.slices[g % 2]
        a, b = g * self.Lg, (g + 1) * self.Lg
        Z.sparse_decode_attn(self.slice_shape, q[:, a:b], sk, sv, self.slice_pt, self.iota, self.count,
                             self.out[:, a:b], self.slice_ws[g % 2], dev_status=self.status, stream=stream)

    def run(self, q, seg, update_selection: bool = True, close_items=None, pipelined: bool = True):
        bounds, nsum, seq_len = seg
        p = self.params
        if q.shape[0] != 1 or not q.is_contiguous():
            raise ValueError("the layer-pipelined tier runs batch 1 (the paper's setting)")
        if update_selection:
            self.select(q, seg, close_items)
        else:
            Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count, self.status)
        ng = self.shape.num_layers // self.Lg
        if not pipelined:
            for g in range(ng):
                self.gather(g)
                self.attend_group(q, g)
            return self.out
        comp, cp = torch.cuda.current_stream(), self.copy_stream
        cp.wait_stream(comp)  # I_f is known
        for g in range(ng):
            with torch.cuda.stream(cp):
                if g >= 2:
                    cp.wait_event(self.ev_free[g - 2])  # slot g % 2: group g-2 has been attended
                self.gather(g, stream=cp)
                self.ev_ready[g].record(cp)
            comp.wait_event(self.ev_ready[g])
            self.attend_group(q, g, stream=comp)
            self.ev_free[g].record(comp)
        comp.wait_stream(cp)
        return self.out

    def launches_per_step(self, *args, **kwargs) -> int:
        return 1 + 2 * (self.shape.num_layers // self.Lg)
