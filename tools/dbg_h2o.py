"""Per-kernel times of one H2O step at the bench workload (8b16k, budget = ZoomR's mean |I_f|)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.policies import PolicyStep
from paper_2604_10898_b200.step import StepParams

cfg = S.config_by_name(sys.argv[1] if len(sys.argv) > 1 else "8b16k")
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 2820
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
kv = (inp.k_pool, inp.v_pool, inp.page_table)
seg = (inp.bounds, inp.num_summaries, inp.seq_len)
ps = PolicyStep("h2o", shape, 1, inp.bounds.shape[1], cfg.T, prm, budget=budget, max_positions=cfg.T)
ps.start_h2o(seg)
ps.run(inp.q, kv, seg)
REP = 20


def t(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(REP):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (10 * REP), 2)


p = ps.params
res = {
    "select": t(lambda: Z.h2o_select(ps.prev_index, ps.prev_count, ps.score, inp.seq_len, p.sink, p.window, budget,
                                     ps.index, ps.count, ps.status)),
    "a5_logits": t(lambda: Z.sparse_decode_attn_logits(shape, inp.q, *kv, ps.index, ps.count, ps.out, ps.lse,
                                                       ps.logits, ps.workspace, dev_status=ps.status)),
    "a5_plain_index_only": t(lambda: Z.sparse_decode_attn(shape, inp.q, *kv, ps.index, ps.count, ps.out,
                                                          ps.workspace, dev_status=ps.status)),
    "accumulate": t(lambda: Z.h2o_accumulate(shape, ps.index, ps.count, ps.logits, ps.lse, ps.score,
                                             index_copy=ps.prev_index, count_copy=ps.prev_count,
                                             dev_status=ps.status)),
    "step": t(lambda: ps.run(inp.q, kv, seg)),
}
# eviction pressure: a smaller budget than the previous set forces the radix select
ps2 = PolicyStep("h2o", shape, 1, inp.bounds.shape[1], cfg.T, prm, budget=budget, max_positions=cfg.T)
ps2.start_h2o(seg)
ps2.score.uniform_()
res["select_evict_half"] = t(lambda: Z.h2o_select(ps2.prev_index, ps2.prev_count, ps2.score, inp.seq_len, p.sink,
                                                  p.window, budget // 2 + 300, ps2.index, ps2.count, ps2.status))
ps.check_status()
ps2.check_status()
print(res)
