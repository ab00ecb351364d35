import ctypes as C, sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep
cfg = S.CONFIGS["8b16k"]
inp = S.generate(cfg, device="cuda")
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
for rep in range(4):
    st.run(inp.q, kv, seg)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 64)()
    Z.lib().zoomr_debug_attn_timeline(buf)
    t = list(buf)
    base = min(x for x in t if x)
    names = ["start", "after_wait", "roles", "first_issue/first_wait", "first_done/first_data", "last_issue/loop_end", "flush_end"]
    for who, lab in [(0, "cta0 math"), (1, "cta0 prod"), (2, "cta77 math"), (3, "cta77 prod")]:
        print(lab, [round((t[who * 16 + k] - base) / 1000, 2) if t[who * 16 + k] else None for k in range(12)])
    print()
