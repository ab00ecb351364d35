"""Probe: per-kernel GPU times of one workload (current build), for quick A/B.

usage: WL=70b64k HKV=1 HQ=8 python tools/probe_a5.py
Prints a5 alone (index-only, early rows), the fused select, the separate
a1..a4 launches and the step, each as the mean of a graph of 20 launches over
4 rotating input sets, with a5's GB/s against the measured HBM peak."""
import dataclasses
import json
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
if os.environ.get("BATCH"):
    cfg = dataclasses.replace(cfg, batch=int(os.environ["BATCH"]))
R = int(os.environ.get("ROT", "4"))
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
sets = []
for r in range(R):
    inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
    st = ZoomrStep(shape, inp.q.shape[0], inp.bounds.shape[1], cfg.T, prm,
                   early_known=os.environ.get("EARLY", "1") == "1")
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    st.run(inp.q, kv, seg, close_items=newest)
    sets.append(dict(inp=inp, st=st, kv=kv, seg=seg, newest=newest))
torch.cuda.synchronize()


def graph_of(fn, n=20):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(n):
            fn(i)
    return g


def t_us(fn, n=20, reps=5):
    g = graph_of(fn, n)
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        v = e0.elapsed_time(e1) * 1e3 / n
        best = v if best is None else min(best, v)
    return best


def X(i):
    return sets[i % R]


res = {"cfg": cfg.name, "L": cfg.L, "Hq": cfg.Hq, "Hkv": cfg.Hkv, "batch": cfg.batch}
res["index_count"] = [int(c) for c in sets[0]["st"].count.cpu()]
res["a5_index_only_us"] = t_us(lambda i: X(i)["st"].attend(X(i)["inp"].q, X(i)["kv"], None) if False else
                                Z.sparse_decode_attn(shape, X(i)["inp"].q, *X(i)["kv"], X(i)["st"].index,
                                                     X(i)["st"].count, X(i)["st"].out, X(i)["st"].workspace))
res["a5_early_us"] = t_us(lambda i: X(i)["st"].attend(X(i)["inp"].q, X(i)["kv"], X(i)["inp"].seq_len))
res["select_fused_us"] = t_us(lambda i: Z.select_fused(
    shape, X(i)["inp"].q, *X(i)["kv"], *X(i)["seg"], X(i)["newest"], X(i)["st"].mean_keys, cfg.top_k, cfg.c,
    cfg.sink, cfg.window, X(i)["st"].flags, X(i)["st"].index, X(i)["st"].count, X(i)["st"].sel_workspace,
    partial=X(i)["st"].partial, agreeability=X(i)["st"].agreeability, dev_status=X(i)["st"].status))
res["step_fused_us"] = t_us(lambda i: X(i)["st"].run(X(i)["inp"].q, X(i)["kv"], X(i)["seg"], close_items=X(i)["newest"]))
res["step_separate_us"] = t_us(lambda i: X(i)["st"].run(X(i)["inp"].q, X(i)["kv"], X(i)["seg"],
                                                        close_items=X(i)["newest"], fused=False))
def single_replay_us(fn, n=100):
    """One step per graph replay, n replays back to back (the bench's headline timing)."""
    gs = [graph_of(lambda i, r=r: fn(r), 1) for r in range(R)]
    for i in range(8):
        gs[i % R].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        gs[i % R].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


res["step_single_replay_us"] = single_replay_us(lambda i: X(i)["st"].run(X(i)["inp"].q, X(i)["kv"], X(i)["seg"],
                                                                          close_items=X(i)["newest"]))
res["step_held_us"] = t_us(lambda i: X(i)["st"].run(X(i)["inp"].q, X(i)["kv"], X(i)["seg"], update_selection=False))
for s_ in sets:
    s_["st"].check_status()
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]
a5_bytes = sum(c * cfg.L * cfg.Hkv * cfg.d * 4 for c in res["index_count"])
res["a5_bytes"] = a5_bytes
res["a5_index_only_frac"] = a5_bytes / (res["a5_index_only_us"] * 1e-6) / 1e9 / hbm
res["a5_early_frac"] = a5_bytes / (res["a5_early_us"] * 1e-6) / 1e9 / hbm
print(json.dumps(res))
