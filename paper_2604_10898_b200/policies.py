"""The paper's comparison policies on the same kernels:

* StreamingLLM: I_f = sink u recent window, no summaries --
  ZoomR's N_t = 0 path; at a matched budget the window grows to
  budget - sink ("set the equivalent budget");
* SumR ("a simplified variant of ZoomR"): every closed summary kept,
  nothing zoomed -- all flags 1.

Both skip a1-a3: the step is a4 (zoomr_build_index with fixed flags) + a5.
Host logic only (which flags, which window); the work is the libzoomr kernels."""
from __future__ import annotations

import torch

from . import zoomr as Z
from .step import StepParams, ZoomrStep

POLICIES = ("streamingllm", "sumr")


class PolicyStep(ZoomrStep):
    def __init__(self, policy: str, shape: Z.Shape, batch: int, max_summaries: int, index_capacity: int,
                 params: StepParams, budget: int = 0, device="cuda"):
        if policy not in POLICIES:
            raise ValueError(f"policy must be one of {POLICIES}")
        if policy == "streamingllm" and budget > 0:  # matched budget: the window takes what the sink leaves
            params = StepParams(params.top_k, params.c, params.sink, max(1, budget - params.sink))
        super().__init__(shape, batch, max_summaries, index_capacity, params, device)
        self.policy = policy

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
        Z.build_index(bounds, nsum, seq_len, self.flags, p.sink, p.window, self.index, self.count, self.status)
        self.attend(q, kv, seq_len)
        return self.out

    def launches_per_step(self, *args, **kwargs) -> int:
        return 2
