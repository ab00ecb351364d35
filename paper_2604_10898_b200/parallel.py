"""Multi-GPU partitioning of the ZoomR step.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Two ways
to split the work, matching BASELINE.json's configs:

* batch sharding (configs[2]) -- sequences are independent problems: rank r
  owns sequences [r*B/N, (r+1)*B/N) with their own KV pages, mean keys and
  selection, and runs the unmodified single-GPU step.  No collective on the
  data path ("weak" scaling when the per-rank batch is fixed).

* KV-head sharding (configs[3], one long sequence) -- rank r owns KV heads
  [r*H_kv/N, (r+1)*H_kv/N) and their G query heads for every layer, so a1, a2
  (its local voters) and a5 stay local.  The consensus needs every voter:
  ONE all-reduce(SUM) of the per-summary partial (votes, A) precedes a3, after
  which every rank runs a3/a4 on identical inputs and obtains identical flags
  and I_f without a broadcast.  `partial` is int64 (votes, and A as the
  fixed-point sum of round(alpha * 2^32)), so the reduced value is bit-identical
  to the single-GPU one whatever the reduction order.

* token sharding (H_kv < #GPUs, e.g. Qwen2.5-7B's 4 KV
  heads on 8 GPUs) -- rank r holds the tokens t with owner[b][t] == r
  (`token_owner_map`: every summary S_i whole on one rank, because a1 reads
  all of its key rows; every other token in position chunks, round robin).
  The mean-key cache is replicated (a1 on the summaries a rank owns, then an
  all-reduce(SUM) of the cache: every entry has exactly one non-zero
  contribution, so the sum is exact); a2..a4 run replicated and give every
  rank the same I_f; a5 runs over the rank's part of I_f with its log-sum-exp
  (`zoomr_shard_index`, `zoomr_sparse_decode_attn_lse`); one all-gather of
  (out, lse, count) and `zoomr_merge_attn` give every rank the full output.

Host logic only: the kernels are the libzoomr ones.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

import torch

from . import zoomr as Z
from .step import StepParams, ZoomrStep


def shard_range(n: int, rank: int, world: int):
    """Contiguous balanced split of range(n): [start, stop) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


@dataclass(frozen=True)
class HeadShard:
    kv_start: int
    kv_stop: int
    q_start: int
    q_stop: int

    @property
    def num_kv(self) -> int:
        return self.kv_stop - self.kv_start

    @property
    def num_q(self) -> int:
        return self.q_stop - self.q_start


def shard_heads(num_q_heads: int, num_kv_heads: int, rank: int, world: int) -> HeadShard:
    """KV heads split across ranks; query head h follows KV head h // G (reading Q6)."""
    if num_kv_heads % world:
        raise ValueError(f"KV-head sharding needs world ({world}) | H_kv ({num_kv_heads})")
    G = num_q_heads // num_kv_heads
    k0, k1 = shard_range(num_kv_heads, rank, world)
    return HeadShard(k0, k1, k0 * G, k1 * G)


def local_shape(shape: Z.Shape, shard: HeadShard) -> Z.Shape:
    return Z.Shape(shape.num_layers, shard.num_q, shard.num_kv, shape.head_dim, shape.page_size)


def slice_heads(k_pool: torch.Tensor, v_pool: torch.Tensor, q: torch.Tensor, shard: HeadShard):
    """Rank-local views of a full pool / query set (used to build shards from one
    generated context; a real deployment allocates only its own heads)."""
    kp = k_pool[:, :, shard.kv_start:shard.kv_stop].contiguous()
    vp = v_pool[:, :, shard.kv_start:shard.kv_stop].contiguous()
    qq = q[:, :, shard.q_start:shard.q_stop].contiguous()
    return kp, vp, qq


def nccl_allreduce_sum(group=None):
    """The head-sharded exchange: sum `partial` (int64 [B][2][N_max]) over ranks in place."""
    import torch.distributed as dist

    def _ar(partial: torch.Tensor):
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return _ar


class HeadShardedStep(ZoomrStep):
    """ZoomrStep over this rank's KV heads; `run` inserts the all-reduce between a2 and a3."""

    def __init__(self, shape: Z.Shape, shard: HeadShard, batch: int, max_summaries: int,
                 index_capacity: int, params: StepParams, device="cuda", group=None,
                 debug_outputs: bool = False):
        super().__init__(local_shape(shape, shard), batch, max_summaries, index_capacity, params, device,
                         debug_outputs)
        self.global_shape, self.shard = shape, shard
        self._ar = nccl_allreduce_sum(group)

    def run(self, q, kv, seg, update_selection=True, close_items=None, allreduce=None, fused=True):
        """fused (default): zoomr_select_front -> all-reduce -> zoomr_select_tail -> a5;
        fused=False: the five separate calls with the all-reduce between a2 and a3."""
        return super().run(q, kv, seg, update_selection, close_items, allreduce or self._ar, fused=fused)


# ---------------------------------------------------------------- token sharding --
def token_owner_map(bounds, num_summaries, world: int, stride: int, chunk: int = 64) -> np.ndarray:
    """uint8 [B][stride]: the rank that holds each token position.

    A token outside every summary goes to rank (t // chunk) % world; a summary
    S_i = [s0, s1) goes whole to the rank of its first token, (s0 // chunk) %
    world, so that a1 finds all of its key rows on one rank.  Stateless in t:
    a decode step appends token t to the same rank (the rank of an open
    summary's first token while one is open)."""
    if not 1 <= world <= 255:
        raise ValueError("token sharding supports 1..255 ranks")
    bounds = np.asarray(bounds).reshape(len(num_summaries), -1, 4)
    B = bounds.shape[0]
    own = ((np.arange(stride) // chunk) % world).astype(np.uint8)
    out = np.broadcast_to(own, (B, stride)).copy()
    for b in range(B):
        for i in range(int(num_summaries[b])):
            s0, s1 = int(bounds[b, i, 2]), int(bounds[b, i, 3])
            out[b, s0:s1] = (s0 // chunk) % world
    return out


def gather_exchange(group=None):
    """The token-sharded exchange: all-gather (out, lse, count) of every rank."""
    import torch.distributed as dist

    def _ex(out, lse, count, part_out, part_lse, part_count):
        dist.all_gather(list(part_out.unbind(0)), out, group=group)
        dist.all_gather(list(part_lse.unbind(0)), lse, group=group)
        dist.all_gather(list(part_count.unbind(0)), count, group=group)
    return _ex


def allreduce_mean_keys(group=None):
    import torch.distributed as dist

    def _ar(mk):
        dist.all_reduce(mk, op=dist.ReduceOp.SUM, group=group)
    return _ar


class TokenShardedStep(ZoomrStep):
    """ZoomR step over this rank's tokens (full heads): replicated selection,
    split-K attention over the rank's part of I_f, one all-gather, the merge."""

    def __init__(self, shape: Z.Shape, rank: int, world: int, batch: int, max_summaries: int,
                 index_capacity: int, params: StepParams, device="cuda", group=None,
                 debug_outputs: bool = False,
                 exchange: Optional[Callable] = None, reduce_mean_keys: Optional[Callable] = None):
        super().__init__(shape, batch, max_summaries, index_capacity, params, device, debug_outputs,
                         early_known=False)
        self.rank, self.world = rank, world
        dev = self.out.device
        L, Hq, d = shape.num_layers, shape.num_q_heads, shape.head_dim
        self.mk_local = torch.zeros_like(self.mean_keys)  # this rank's summaries only, zeros elsewhere
        self.local_index = torch.zeros_like(self.index)
        self.local_count = torch.zeros_like(self.count)
        self.out_local = torch.zeros_like(self.out)
        self.lse_local = torch.zeros(batch, L, Hq, dtype=torch.float32, device=dev)
        self.part_out = torch.zeros(world, batch, L, Hq, d, dtype=torch.float32, device=dev)
        self.part_lse = torch.zeros(world, batch, L, Hq, dtype=torch.float32, device=dev)
        self.part_count = torch.zeros(world, batch, dtype=torch.int32, device=dev)
        self.lse = torch.zeros(batch, L, Hq, dtype=torch.float32, device=dev)
        self._ex = exchange or gather_exchange(group)
        self._ar_mk = reduce_mean_keys or allreduce_mean_keys(group)

    def update_mean_keys(self, kv, seg, items: Optional[torch.Tensor]):
        """a1 for the closed summaries this rank owns (items may be empty), then the
        replication of the cache.  Collective: every rank calls it at every close."""
        if items is not None and items.numel():
            k_pool, v_pool, page_table = kv
            bounds, nsum, seq_len = seg
            Z.update_mean_keys(self.shape, k_pool, v_pool, page_table, bounds, nsum, seq_len, items,
                               self.mk_local, self.status)
        self.mean_keys.copy_(self.mk_local)
        self._ar_mk(self.mean_keys)

    def run(self, q, kv, seg, owner, update_selection: bool = True):
        """Enqueue one step (a2..a5, the exchange, the merge); the caller ran
        update_mean_keys for the summaries closed since the last step."""
        self.run_local(q, kv, seg, owner, update_selection)
        return self.combine()

    def run_local(self, q, kv, seg, owner, update_selection: bool = True):
        """The rank-local part: replicated a2..a4, then a5 over this rank's tokens."""
        k_pool, v_pool, page_table = kv
        bounds, nsum, seq_len = seg
        p = self.params
        if update_selection:  # a2..a4 in one launch (no a1: the cache is already replicated)
            Z.select_fused(self.shape, q, k_pool, v_pool, page_table, bounds, nsum, seq_len, None,
                           self.mean_keys, p.top_k, p.c, p.sink, p.window, self.flags, self.index, self.count,
                           self.sel_workspace, partial=self.partial, agreeability=self.agreeability,
                           alpha_out=self.alpha, topk_out=self.topk, dev_status=self.status)
        else:
            Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count,
                          self.status)
        self.attend_local(q, kv, owner)

    def combine(self):
        """The exchange of (out, lse, count) and the merge into self.out / self.lse."""
        self._ex(self.out_local, self.lse_local, self.local_count, self.part_out, self.part_lse, self.part_count)
        Z.merge_attn(self.shape, self.part_out, self.part_lse, self.out, part_count=self.part_count, lse=self.lse)
        return self.out

    def attend_local(self, q, kv, owner):
        """This rank's part of I_f: restriction + a5 with log-sum-exp."""
        k_pool, v_pool, page_table = kv
        Z.shard_index(self.index, self.count, owner, self.rank, self.local_index, self.local_count, self.status)
        Z.sparse_decode_attn_lse(self.shape, q, k_pool, v_pool, page_table, self.local_index, self.local_count,
                                 self.out_local, self.lse_local, self.workspace, dev_status=self.status)
