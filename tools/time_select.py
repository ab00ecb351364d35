"""GPU time of one zoomr_select_fused launch (graph of 20 launches), 8b16k."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep
cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
if os.environ.get("NO_A1"):
    newest = None
f = lambda: Z.select_fused(shape, inp.q, inp.k_pool, inp.v_pool, inp.page_table, inp.bounds, inp.num_summaries,
                           inp.seq_len, newest, st.mean_keys, cfg.top_k, cfg.c, cfg.sink, cfg.window, st.flags, st.index,
                           st.count, st.sel_workspace, partial=st.partial, agreeability=st.agreeability)
f(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20): f()
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): g.replay()
e1.record(); torch.cuda.synchronize()
print(os.environ.get("ZOOMR_FUSED_STOP", "0"), "no_a1" if newest is None else "a1", round(e0.elapsed_time(e1) * 1e3 / 400, 2), "us/select")
