"""K5 (a5 sparse decode attention) alone: time vs |I_f|, to separate the fixed
per-launch cost (ramp-up, merge tail) from the streaming rate.  GPU only.

  python tools/k5_sweep.py [--workload 8b16k] [--counts 256,512,1024,2048,2816]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S  # noqa: E402
from paper_2604_10898_b200 import zoomr as Z  # noqa: E402
from paper_2604_10898_b200.step import StepParams, ZoomrStep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="8b16k")
    ap.add_argument("--counts", default="128,256,512,1024,1536,2048,2816")
    ap.add_argument("--rotate", type=int, default=2)
    ap.add_argument("--rep", type=int, default=20)
    args = ap.parse_args()
    cfg = S.CONFIGS[args.workload]
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    sets = []
    for r in range(args.rotate):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 31 * r, query_mode="diffuse")
        st = ZoomrStep(shape, inp.q.shape[0], inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink,
                                                                                         cfg.window))
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        st.run(inp.q, kv, seg)
        sets.append((inp, st))
    torch.cuda.synchronize()
    full = [int(st.count[0]) for _, st in sets]
    rows = []
    for n in [int(x) for x in args.counts.split(",")]:
        graphs = []
        for inp, st in sets:
            st.count.fill_(min(n, full[0]))
            g = torch.cuda.CUDAGraph()
            Z.sparse_decode_attn(shape, inp.q, inp.k_pool, inp.v_pool, inp.page_table, st.index, st.count, st.out,
                                 st.workspace)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                for _ in range(args.rep):
                    Z.sparse_decode_attn(shape, inp.q, inp.k_pool, inp.v_pool, inp.page_table, st.index, st.count,
                                         st.out, st.workspace)
            graphs.append(g)
        for g in graphs:
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(10):
            graphs[it % len(graphs)].replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (10 * args.rep)
        nbytes = n * cfg.L * cfg.Hkv * cfg.d * 4
        rows.append({"count": n, "us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1)})
        print(json.dumps(rows[-1]), flush=True)
    # affine fit t = t0 + bytes / BW
    import numpy as np
    x = np.array([r["count"] * cfg.L * cfg.Hkv * cfg.d * 4 for r in rows], dtype=float)
    y = np.array([r["us"] for r in rows])
    A = np.vstack([np.ones_like(x), x]).T
    (t0, slope), *_ = np.linalg.lstsq(A, y, rcond=None)
    print(json.dumps({"fit_fixed_us": round(float(t0), 2), "fit_stream_GBps": round(1e-3 / slope, 1)}))


if __name__ == "__main__":
    main()
