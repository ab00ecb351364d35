"""A few eager decode steps of one workload (fused select + a5 with early rows), for
ncu / quick checks:  WL=8b16k STEPS=6 python tools/step_once.py"""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S  # noqa: E402
from paper_2604_10898_b200 import zoomr as Z  # noqa: E402
from paper_2604_10898_b200.step import StepParams, ZoomrStep  # noqa: E402

cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
if os.environ.get("HKV"):
    cfg = dataclasses.replace(cfg, Hkv=int(os.environ["HKV"]), Hq=int(os.environ["HQ"]))
inp = S.generate(cfg, device="cuda")
st = ZoomrStep(Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page), 1, inp.bounds.shape[1], cfg.T,
               StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
kv = (inp.k_pool, inp.v_pool, inp.page_table)
seg = (inp.bounds, inp.num_summaries, inp.seq_len)
st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
for _ in range(int(os.environ.get("STEPS", "6"))):
    st.run(inp.q, kv, seg, close_items=newest)
torch.cuda.synchronize()
st.check_status()
print("ok", int(st.count[0]))
