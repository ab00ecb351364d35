"""Per-stage times of one token-sharded rank (8 simulated ranks, 8b16k): fused
select (a2..a4), shard_index, a5 with lse, merge -- each graph-captured REP times."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
from paper_2604_10898_b200.step import StepParams, ZoomrStep

name = sys.argv[1] if len(sys.argv) > 1 else "8b16k"
cfg = S.config_by_name(name)
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
kv = (inp.k_pool, inp.v_pool, inp.page_table)
seg = (inp.bounds, inp.num_summaries, inp.seq_len)
ref = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, prm)
ref.update_mean_keys(kv, seg, ref.all_items(inp.num_summaries))
W = 8
own = torch.from_numpy(token_owner_map(inp.bounds.cpu().numpy(), inp.num_summaries.cpu().numpy(), W,
                                       int(inp.seq_len.max()), 64)).cuda()
st = TokenShardedStep(shape, 0, W, 1, inp.bounds.shape[1], cfg.T, prm, exchange=lambda *a: None,
                      reduce_mean_keys=lambda m: None)
st.mean_keys.copy_(ref.mean_keys)
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
    return e0.elapsed_time(e1) * 1e3 / (10 * REP)


p = st.params
sel = lambda: Z.select_fused(shape, inp.q, *kv, *seg, None, st.mean_keys, p.top_k, p.c, p.sink, p.window, st.flags,
                             st.index, st.count, st.sel_workspace, partial=st.partial, dev_status=st.status)
shard = lambda: Z.shard_index(st.index, st.count, own, 0, st.local_index, st.local_count, st.status)
a5l = lambda: Z.sparse_decode_attn_lse(shape, inp.q, *kv, st.local_index, st.local_count, st.out_local, st.lse_local,
                                       st.workspace, dev_status=st.status)
a5full = lambda: Z.sparse_decode_attn(shape, inp.q, *kv, st.index, st.count, st.out, st.workspace,
                                      dev_status=st.status)
merge = lambda: Z.merge_attn(shape, st.part_out, st.part_lse, st.out, part_count=st.part_count, lse=st.lse)
res = {k: round(t(f), 2) for k, f in [("select_fused_a2a4", sel), ("shard_index", shard), ("a5_lse_rank0", a5l),
                                       ("a5_full_index", a5full), ("merge", merge)]}
res["all_local"] = round(t(lambda: (sel(), shard(), a5l())), 2)
res["rank0_share"] = int(st.local_count[0]) / int(st.count[0])
st.check_status()
print(res)
