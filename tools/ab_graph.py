"""Step time with 1 step per graph replay vs several steps captured in one graph."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep
cfg = S.CONFIGS["8b16k"]
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
R = 4
sets = []
for r in range(R):
    inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
    st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
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
g1 = []
for inp, st, kv, seg, newest in sets:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st.run(inp.q, kv, seg, close_items=newest)
    g1.append(g)
i = [0]
def one():
    g1[i[0] % R].replay(); i[0] += 1
print("1 step/graph :", round(timeit(one, 200), 2), "us/step")
gR = torch.cuda.CUDAGraph()
with torch.cuda.graph(gR):
    for inp, st, kv, seg, newest in sets:
        st.run(inp.q, kv, seg, close_items=newest)
print(f"{R} steps/graph:", round(timeit(lambda: gR.replay(), 50) / R, 2), "us/step")
