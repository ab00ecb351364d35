"""The paper's comparison policies on the same kernels:

* StreamingLLM: I_f = sink u recent window, no summaries --
  ZoomR's N_t = 0 path; at a matched budget the window grows to
  budget - sink ("set the equivalent budget");
* SumR ("a simplified variant of ZoomR"): every closed summary kept,
  nothing zoomed -- all flags 1.

Both skip a1-a3: the step is a4 (zoomr_build_index with fixed flags) + a5.

* H2O ("a dynamic approach that selects tokens based on importance scores
  at each generation step"; rule of SPEC h2o_step): the retained set
  is the sink, the window and the budget - |sink u window| previously retained
  tokens with the largest cumulative attention received (readings H1, H2 in
  DESIGN.md 8c).  Step = zoomr_h2o_select + a5 with logits +
  zoomr_h2o_accumulate (which also hands the set to the next step).

Host logic only (which flags, which window); the work is the libzoomr kernels."""
from __future__ import annotations

import torch

from . import zoomr as Z
from .step import StepParams, ZoomrStep

POLICIES = ("streamingllm", "sumr", "h2o")


class PolicyStep(ZoomrStep):
    def __init__(self, policy: str, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int,
                 params: StepParams, budget: int = 0, device="cuda", max_positions: int = 0):
        if policy not in POLICIES:
            raise ValueError(f"policy must be one of {POLICIES}")
        if policy == "streamingllm" and budget > 0:  # matched budget: the window takes what the sink leaves
            params = StepParams(params.top_k, params.c, params.sink, max(1, budget - params.sink))
        if policy == "h2o":
            if budget < 1:
                raise ValueError("h2o needs a budget")
            # |I| <= max(budget, sink + window): the index (and the logits) need no more
            index_capacity = min(index_capacity, max(budget, params.sink + params.window))
        super().__init__(shape, batch, max_summaries, index_capacity, params, device, early_known=False)
        self.policy, self.budget = policy, budget
        if policy == "h2o":
            L, Hq = shape.num_layers, shape.num_q_heads
            dev = self.out.device
            npos = max_positions or index_capacity
            self.score = torch.zeros(batch, npos, dtype=torch.float32, device=dev)  # cumulative attention received
            self.prev_index = torch.zeros_like(self.index)
            self.prev_count = torch.zeros_like(self.count)
            self.lse = torch.zeros(batch, L, Hq, dtype=torch.float32, device=dev)
            self.logits = torch.zeros(batch, L, Hq, index_capacity, dtype=torch.float32, device=dev)

    def start_h2o(self, seg):
        """Initial retained set: sink u the most recent tokens up to the budget (StreamingLLM at the
        budget; a4 with every flag 0), cumulative scores zero."""
        bounds, nsum, seq_len = seg
        p = self.params
        self.score.zero_()
        self.flags.zero_()
        Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, max(1, self.budget - p.sink), self.prev_index,
                      self.prev_count, self.status)

    def prepare(self, num_summaries: torch.Tensor):
        """Fixed flags: all closed summaries kept (SumR) or none (StreamingLLM)."""
        self.flags.zero_()
        if self.policy == "sumr":
            n = self.flags.shape[1]
            keep = torch.arange(n, device=self.flags.device)[None, :] < num_summaries.long()[:, None]
            self.flags.copy_(keep.to(torch.uint8))

    def run(self, q, kv, seg, *args, **kwargs):
        k_pool, v_pool, page_table = kv
        bounds, nsum, seq_len = seg
        p = self.params
        if self.policy == "h2o":
            Z.h2o_select(self.prev_index, self.prev_count, self.score, seq_len, p.sink, p.window, self.budget,
                         self.index, self.count, self.status)
            Z.sparse_decode_attn_logits(self.shape, q, k_pool, v_pool, page_table, self.index, self.count, self.out,
                                        self.lse, self.logits, self.workspace, dev_status=self.status)
            Z.h2o_accumulate(self.shape, self.index, self.count, self.logits, self.lse, self.score,
                             index_copy=self.prev_index, count_copy=self.prev_count, dev_status=self.status)
            return self.out
        Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count, self.status)
        self.attend(q, kv, seq_len)
        return self.out

    def launches_per_step(self, *args, **kwargs) -> int:
        return 3 if self.policy == "h2o" else 2
