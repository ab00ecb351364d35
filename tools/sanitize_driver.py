"""Small workloads through every libzoomr kernel, for compute-sanitizer
(tools/sanitize.sh runs it under memcheck, racecheck, synccheck, initcheck).

Covers: the separate a1..a5 calls and the fused select (tiny, and random small
layouts with d = 128 so that a5 takes its TMA / mbarrier path), a5's early rows
and index-only modes, one ZoomrStep(chained=True) captured three times back to
back in one graph, Algorithm 1's device decode loop, the token-sharded pieces
(restriction, a5 + lse, merge), H2O, and the host-memory tier.  Checks results
loosely (the parity tests are elsewhere): the point is the sanitizer's report."""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S  # noqa: E402
from paper_2604_10898_b200 import zoomr as Z  # noqa: E402
from paper_2604_10898_b200.step import DecodeLoop, StepParams, ZoomrStep  # noqa: E402


def small(name, **kw):
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=128, T=1024, n_pairs=12, LR=60, LS=12, sink=4, window=96,
                c=3, top_k=2, page=32, seed=41)
    base.update(kw)
    return S.Config(**base)


def make(cfg, seed=None, chained=False, early=True):
    inp = S.generate(cfg, device="cuda", seed=seed)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    st = ZoomrStep(shape, inp.q.shape[0], inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink,
                                                                                  cfg.window),
                   debug_outputs=True, chained=chained, early_known=early)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[b, max(int(n) - 1, -1)] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    return inp, st, kv, seg, shape, newest


def main():
    which = sys.argv[1:] or ["steps", "chained", "loop", "shard", "h2o", "tier"]
    torch.manual_seed(0)
    if "steps" in which:
        for cfg in (S.CONFIGS["tiny"], small("b3_jit", batch=3, jitter=True), small("g7", Hq=14),
                    small("d64", d=64, batch=2)):
            for fused in (True, False):
                for early in (True, False):
                    inp, st, kv, seg, shape, newest = make(cfg, early=early)
                    st.run(inp.q, kv, seg, close_items=newest, fused=fused)
                    torch.cuda.synchronize()
                    st.check_status()
                    assert torch.isfinite(st.out).all()
        print("steps ok", flush=True)
    if "chained" in which:
        inp, st, kv, seg, shape, newest = make(small("chain", batch=2), chained=True)
        st.run(inp.q, kv, seg, close_items=newest)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            st.run(inp.q, kv, seg, close_items=newest)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(3):
                st.run(inp.q, kv, seg, close_items=newest)
            st.attend(inp.q, kv, inp.seq_len)  # a5 right behind a chained a5 (detected: index-only)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        st.check_status()
        print("chained ok", flush=True)
    if "loop" in which:
        cfg = small("loop", T=1024)
        inp = S.generate(cfg, device="cuda")
        shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
        lp = DecodeLoop(shape, 1, 64, cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window), 1000, 1001, [200])
        lp.start(700)
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        toks = [7] * 20 + [1000] + [7] * 6 + [1001] + [7] * 10 + [200] + [7] * 5
        for t in toks:
            kin = torch.randn(1, cfg.L, cfg.Hkv, cfg.d, device="cuda").bfloat16()
            lp.decode_step(kv, kin, torch.randn_like(kin), inp.q, torch.tensor([t], dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        lp.check_status()
        print("loop ok", int(lp.num_summaries[0]), flush=True)
    if "shard" in which:
        from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
        cfg = small("shard", batch=2)
        inp = S.generate(cfg, device="cuda")
        shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
        world = 3
        own = token_owner_map(inp.bounds.cpu().numpy(), inp.num_summaries.cpu().numpy(), world,
                              int(inp.page_table.shape[1]) * cfg.page, 64)
        owner = torch.from_numpy(own).cuda()
        steps = []

        def ex(out, lse, count, po, pl, pc):
            for r, t in enumerate(steps):
                po[r].copy_(t.out_local)
                pl[r].copy_(t.lse_local)
                pc[r].copy_(t.local_count)
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        for r in range(world):
            t = TokenShardedStep(shape, r, world, 2, inp.bounds.shape[1], cfg.T,
                                 StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window), exchange=ex,
                                 reduce_mean_keys=lambda mk: None)
            t.mk_local.zero_()
            t.update_mean_keys(kv, seg, t.all_items(inp.num_summaries))
            steps.append(t)
        for t in steps:
            t.run_local(inp.q, kv, seg, owner)
        steps[0].combine()
        torch.cuda.synchronize()
        for t in steps:
            t.check_status()
        print("shard ok", flush=True)
    if "h2o" in which:
        from paper_2604_10898_b200.policies import PolicyStep
        cfg = small("h2o", batch=2)
        inp = S.generate(cfg, device="cuda")
        shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        for pol in ("streamingllm", "sumr", "h2o"):
            ps = PolicyStep(pol, shape, 2, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink,
                                                                                 cfg.window),
                            budget=300, max_positions=cfg.T)
            ps.prepare(inp.num_summaries)
            if pol == "h2o":
                ps.start_h2o(seg)
            for _ in range(3):
                ps.run(inp.q, kv, seg, update_selection=False)
            torch.cuda.synchronize()
            ps.check_status()
        print("h2o ok", flush=True)
    if "tier" in which:
        from paper_2604_10898_b200.tier import HostTierStep
        cfg = small("tier", batch=2)
        inp = S.generate(cfg, device="cuda")
        shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
        hk, hv = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
        st = HostTierStep(shape, 2, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window),
                          hk, hv, inp.page_table, 64)
        st.update_mean_keys((inp.k_pool, inp.v_pool, inp.page_table), (inp.bounds, inp.num_summaries, inp.seq_len),
                            st.all_items(inp.num_summaries))
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        for _ in range(2):
            st.run(inp.q, seg)
        torch.cuda.synchronize()
        st.check_status()
        print("tier ok", flush=True)


if __name__ == "__main__":
    main()
