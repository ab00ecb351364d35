"""Where the fused select's time goes: time zoomr_select_fused alone (graph of 20
launches, inputs rotated) with the experiment build cut short at each phase
(ZOOMR_FUSED_STOP = 1 after the ticket, 2 after the collect, 3 after a3, 0 full).
  python -c "from paper_2604_10898_b200 import _build; _build.build(out='ablibs/lib_exp.so', defines=['ZOOMR_EXPERIMENTS'])"
  ZOOMR_LIB_OVERRIDE=$PWD/ablibs/lib_exp.so WL=8b16k python tools/select_phases.py"""
import dataclasses
import json
import os
import subprocess
import sys

if os.environ.get("_PHASE_CHILD"):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import zoomr_synth as S
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
    if os.environ.get("HKV"):
        cfg = dataclasses.replace(cfg, Hkv=int(os.environ["HKV"]), Hq=int(os.environ["HQ"]))
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    sets = []
    for r in range(4):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
        st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
        sets.append((inp, st, kv, seg, newest))

    def one(i, close=True):
        inp, st, kv, seg, newest = sets[i % 4]
        Z.select_fused(shape, inp.q, *kv, *seg, newest if close else None, st.mean_keys, cfg.top_k, cfg.c, cfg.sink,
                       cfg.window, st.flags, st.index, st.count, st.sel_workspace, partial=st.partial,
                       agreeability=st.agreeability, dev_status=st.status)
    res = {}
    for close in (True, False):
        one(0, close)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(20):
                one(i, close)
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 20)
        res["with_a1" if close else "no_a1"] = best
    print(json.dumps(res))
else:
    out = {}
    for stop in (1, 2, 3, 0):
        env = dict(os.environ, _PHASE_CHILD="1", ZOOMR_FUSED_STOP=str(stop))
        r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
        out[f"stop{stop}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    print(json.dumps({"wl": os.environ.get("WL", "8b16k"), **out}))
