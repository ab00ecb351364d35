"""Algorithm 1's decode loop over HBM vs over the host tier (8B-16K), as bench.py
sets them up: µs per token as a graph of N_TOK tokens each, and (EAGER=1, for an
ncu launch list) a few eager tokens of each loop.

  python tools/probe_loops.py                       graph timings (JSON line)
  EAGER=1 ncu --metrics gpu__time_duration.sum ... python tools/probe_loops.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S  # noqa: E402
from paper_2604_10898_b200 import zoomr as Z  # noqa: E402
from paper_2604_10898_b200.step import DecodeLoop, StepParams, ZoomrStep  # noqa: E402
from paper_2604_10898_b200.tier import TierDecodeLoop  # noqa: E402

cfg = S.CONFIGS["8b16k"]
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
kv = (inp.k_pool, inp.v_pool, inp.page_table)
seg = (inp.bounds, inp.num_summaries, inp.seq_len)
ref = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, prm)
ref.update_mean_keys(kv, seg, ref.all_items(inp.num_summaries))
ref.run(inp.q, kv, seg)
torch.cuda.synchronize()
B = 1
N_TOK = int(os.environ.get("N_TOK", "256"))
start = inp.seq_len - N_TOK
kin = torch.randn(B, cfg.L, cfg.Hkv, cfg.d, device="cuda").bfloat16()
vin = torch.randn_like(kin)
toks = torch.tensor([[200 if (i % 35) == 34 else 7] * B for i in range(N_TOK)], dtype=torch.int32, device="cuda")
host_k, host_v = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
ph = int(os.environ.get("PH", "16"))
variants = {
    "hbm_chained": lambda: DecodeLoop(shape, B, inp.bounds.shape[1], cfg.T, prm, 1000, 1001, [200]),
    "hbm_plain": lambda: DecodeLoop(shape, B, inp.bounds.shape[1], cfg.T, prm, 1000, 1001, [200], chained=False,
                                    fused_a0=False),
    "tier": lambda: TierDecodeLoop(shape, B, inp.bounds.shape[1], cfg.T, prm, host_k, host_v, inp.page_table,
                                   int(inp.k_pool.shape[1]) * (cfg.page // ph), 1000, 1001, [200],
                                   hot_page_size=ph),
}
only = os.environ.get("ONLY")
# diagnosis only: SKIP=fetch drops the tier fetch from the loop (valid only once every page
# the replayed tokens touch is resident, i.e. from the second pass of the graph on)
skip = set(filter(None, os.environ.get("SKIP", "").split(",")))
if "fetch" in skip:
    import paper_2604_10898_b200.tier as T_
    T_.Z.tier_fetch = lambda *a, **k: None
res = {}
for name, mk in variants.items():
    if only and name not in only.split(","):
        continue
    lp = mk()
    lp.mean_keys.copy_(ref.mean_keys)
    lp.start_from(inp.bounds, inp.num_summaries, start)
    tier = isinstance(lp, TierDecodeLoop)

    def step(i):
        if tier:
            lp.decode_step(kin, vin, inp.q, toks[i])
        else:
            lp.decode_step(kv, kin, vin, inp.q, toks[i])
    if os.environ.get("EAGER"):
        for i in range(int(os.environ.get("EAGER_TOK", "12"))):
            step(i)
        torch.cuda.synchronize()
        lp.check_status()
        continue
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(N_TOK):
            step(i)

    def run():
        lp.start_from(inp.bounds, inp.num_summaries, start)
        lp.flags.copy_(ref.flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / N_TOK
    run()
    res[name] = min(run() for _ in range(3))
    lp.check_status()
    del g, lp
    torch.cuda.empty_cache()
print(json.dumps(res))
