"""A/B: 4 x R decode steps captured in one graph, chained (ZoomrStep.chained:
zoomr_select_fused_chained runs a1/a2 while the previous step's
zoomr_sparse_decode_attn_chained finishes) vs the plain launches.  Outputs
must be bit-identical.   WL=8b16k|qwen7b16k python tools/ab_select_pdl.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep
cfg = S.CONFIGS[os.environ.get("WL", "8b16k")]
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
R = 4
sets = []
for r in range(R):
    inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
    st = ZoomrStep(shape, inp.q.shape[0], inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[b, int(inp.num_summaries[b]) - 1] for b in range(inp.q.shape[0])], dtype=torch.int32,
                          device="cuda")
    st.run(inp.q, kv, seg, close_items=newest)
    sets.append((inp, st, kv, seg, newest))
torch.cuda.synchronize()


def timeit(fn, n):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


res = {}
for name, flag in [("default", False), ("chained", True), ("default2", False), ("chained2", True)]:
    for _, st, *_ in sets:
        st.chained = flag
    gR = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gR):
        for rep in range(4):
            for inp, st, kv, seg, newest in sets:
                st.run(inp.q, kv, seg, close_items=newest)
    for _, st, *_ in sets:
        st.out.zero_(); st.index.zero_(); st.count.zero_()
    us = timeit(lambda: gR.replay(), 30) / (4 * R)
    torch.cuda.synchronize()
    outs = [(st.out.clone(), st.index.clone(), st.count.clone(), int(st.status.item())) for _, st, *_ in sets]
    res[name] = outs
    print(f"{name:10s}: {us:.2f} us/step ({4 * R} steps per graph)", flush=True)
ref = res["default"]
for name, outs in res.items():
    same = all(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2]) and a[3] == b[3] == 0
               for a, b in zip(ref, outs))
    print(name, "bit-identical to default:", same)
