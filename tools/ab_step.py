"""A/B of step variants on 8b16k: time one graph-captured step (select + a5)."""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep

def run(variant, R=4, K=200):
    cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    gs = []
    for r in range(R):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
        st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window), **variant)
        kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
        gs.append((st.capture(inp.q, kv, seg, close_items=newest), inp, st))
    for i in range(20): gs[i % R][0].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K): gs[i % R][0].replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K

VARIANTS = {"phys": dict(use_phys=True), "nophys": dict(use_phys=False),
            "early": dict(early_known=True), "late": dict(early_known=False)}
for name in os.environ.get("VARS", "nophys,phys").split(","):
    v = VARIANTS[name]
    print(name, round(run(v), 2), "us/step", flush=True)
