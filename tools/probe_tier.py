"""Per-launch GPU times of the host tier's warm step (8B-16K, 16-token hot pages):
tier_fetch (plan + copy, nothing missing), a5 with lse on the hot pool, and the
same a5 on the all-HBM pool, each as the mean of a graph of 20 launches."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S  # noqa: E402
from paper_2604_10898_b200 import zoomr as Z  # noqa: E402
from paper_2604_10898_b200.step import StepParams, ZoomrStep  # noqa: E402
from paper_2604_10898_b200.tier import HostTierStep  # noqa: E402

cfg = S.CONFIGS["8b16k"]
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
kv = (inp.k_pool, inp.v_pool, inp.page_table)
seg = (inp.bounds, inp.num_summaries, inp.seq_len)
ref = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, prm)
ref.update_mean_keys(kv, seg, ref.all_items(inp.num_summaries))
ref.run(inp.q, kv, seg)
hk, hv = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
Ph = int(os.environ.get("PH", "16"))
st = HostTierStep(shape, 1, inp.bounds.shape[1], cfg.T, prm, hk, hv, inp.page_table, 1024 * (64 // Ph), hot_page_size=Ph)
st.mean_keys.copy_(ref.mean_keys)
st.run(inp.q, seg)
st.run(inp.q, seg)
torch.cuda.synchronize()


def t_us(fn, n=20):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


hs = st.host_shape
res = {"Ph": Ph}
res["tier_fetch_us"] = t_us(lambda: Z.tier_fetch(hs, hk, hv, inp.page_table, st.hot_k, st.hot_v, st.hot_page_table,
                                                  st.hot_owner, st.hot_stamp, st.index, st.count, st.tier_ws, st.status))
res["a5_lse_hot_us"] = t_us(lambda: Z.sparse_decode_attn_lse(st.shape, inp.q, st.hot_k, st.hot_v, st.hot_page_table,
                                                             st.index, st.count, st.out, st.lse, st.workspace))
res["a5_index_only_hot_us"] = t_us(lambda: Z.sparse_decode_attn(st.shape, inp.q, st.hot_k, st.hot_v,
                                                                st.hot_page_table, st.index, st.count, st.out,
                                                                st.workspace))
res["a5_early_hbm_us"] = t_us(lambda: ref.attend(inp.q, kv, inp.seq_len))
res["select_us"] = t_us(lambda: st.run(inp.q, seg) if False else Z.select_fused(
    hs, inp.q, hk, hv, inp.page_table, *seg, None, st.mean_keys, cfg.top_k, cfg.c, cfg.sink, cfg.window, st.flags,
    st.index, st.count, st.sel_workspace, partial=st.partial, dev_status=st.status))
res["tier_step_us"] = t_us(lambda: st.run(inp.q, seg))
res["hbm_step_us"] = t_us(lambda: ref.run(inp.q, kv, seg))
st.check_status()
print(json.dumps(res))
