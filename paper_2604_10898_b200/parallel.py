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

Host logic only: the kernels are the libzoomr ones.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

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

    def run(self, q, kv, seg, update_selection=True, close_items=None, allreduce=None, fused=False):
        return super().run(q, kv, seg, update_selection, close_items, allreduce or self._ar, fused=False)
