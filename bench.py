#!/usr/bin/env python
"""bench.py -- ZoomR select + sparse-decode step on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload 8b16k]

One "step" = one pass of the whole hot path over one batch of synthetic input:
a1 mean-key update of the newest closed summary, a2 scoring + per-head top-k +
vote aggregation, a3 global top-c, a4 index build, a5 sparse decode attention
over I_f, for every layer and head (selection every step, U = 1).
N = 1 runs BASELINE configs[1] (Llama-3-8B shape, 16K context, batch 1).  N > 1
(launched by torchrun, one rank per GPU, NCCL) runs the same per-rank workload
on every rank with no data-path collective ("scaling": "weak"); the step time
is the max over ranks of the device-timed region.

Prints ONE JSON line on rank 0 (bench contract in the task statement).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "select+sparse-decode step µs and seqs/s at 1/2/4/8 B200; % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="8b16k")
    ap.add_argument("--query", default="planted", choices=["planted", "diffuse"])
    ap.add_argument("--rotate", type=int, default=4, help="independent input sets cycled per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-loop", action="store_true", help="skip the decode-loop measurement")
    ap.add_argument("--no-early", action="store_true",
                    help="A/B only: a5 waits for I_f before attending I_p / I_w")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-c3", action="store_true", help="skip the configs[2] batch-64 section")
    ap.add_argument("--no-heads", action="store_true", help="skip the configs[3] head-sharded section")
    ap.add_argument("--batch-per-gpu", type=int, default=0,
                    help="sequences per rank (default: the workload's batch split over the ranks)")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers --
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(cfg, counts, n_sum, closures=1):
    """SURVEY 8(d) bytes_step, per rank, U = 1.

    a5: |I_f| * L*H_kv*d*2*2 (K and V rows) + q read + fp32 out write + index read
    a4: |I_f| * 4 index write
    a2: N_t * L*H_kv*d*4 fp32 mean keys + q
    a1: |S| * L*H_kv*d*2 + L*H_kv*d*4 for the newest closed summary
    """
    L, Hq, Hkv, d = cfg.L, cfg.Hq, cfg.Hkv, cfg.d
    a5 = sum(c * L * Hkv * d * 4 + L * Hq * d * 2 + L * Hq * d * 4 + c * 4 for c in counts)
    a4 = sum(c * 4 for c in counts)
    a2 = sum(n * L * Hkv * d * 4 + L * Hq * d * 2 for n in n_sum)
    a1 = closures * (cfg.LS * L * Hkv * d * 2 + L * Hkv * d * 4)
    return {"a5": a5, "a4": a4, "a2": a2, "a1": a1, "total": a5 + a4 + a2 + a1}


def workload_config(cfg, args, world, batch_per_gpu, n_summaries):
    """The `config` of the JSON line -- workload parameters only, identical for both arms
    (the run-dependent figures, e.g. the realised |I_f|, are keys of their own)."""
    return {"workload": cfg.name, "batch_per_gpu": batch_per_gpu, "global_batch": batch_per_gpu * world,
            "T": cfg.T, "L": cfg.L, "H_q": cfg.Hq, "H_kv": cfg.Hkv, "d": cfg.d, "n_summaries": n_summaries,
            "c": cfg.c, "top_k": cfg.top_k, "sink": cfg.sink, "window": cfg.window,
            "update_every": max(1, cfg.update_every), "query": args.query,
            "parallelism": f"batch-shard x{world}" if world > 1 else "single",
            "l2": f"inputs larger than L2: {max(1, args.rotate)} independent input sets rotated per step"}


def init_dist(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def per_step_us(fn, K, W):
    """Per-step GPU times (us) from a CUDA event pair around each step (a separate
    pass from the headline timing, so the extra event records do not touch it)."""
    for i in range(W):
        fn(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        ev[i][0].record()
        fn(i)
        ev[i][1].record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) * 1e3 for a, b in ev]


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = (len(xs) - 1) * q
    lo, hi = int(k), min(int(k) + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (k - lo)


def pcts(xs):
    return {"p10": pct(xs, 0.1), "p50": pct(xs, 0.5), "p90": pct(xs, 0.9)}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# --------------------------------------------------------------- CPU oracle --
def oracle_inputs(inp, b=0):
    from zoomr_synth import bf16_bits, logical_rows
    K = bf16_bits(logical_rows(inp, b, "k"))
    V = bf16_bits(logical_rows(inp, b, "v"))
    q = bf16_bits(inp.q[b])
    n = int(inp.num_summaries[b])
    seg = inp.bounds[b, :n].cpu().numpy()
    return q, K, V, seg


def oracle_full_step(cfg, x, threads=0):
    """One full oracle step (O1-O7: a1-a5 over every layer and head) of one sequence."""
    import oracle
    q, K, V, seg = x
    return oracle.step(q, K, V, seg, cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.top_k, cfg.c, cfg.sink, cfg.window,
                       threads=threads)


def oracle_time(inp, seconds, threads=0):
    """Time the CPU oracle (as it stands) on rank 0: full steps of sequence 0, for
    about `seconds` (the cpu_baseline leg; the reference arm times the same
    function step by step)."""
    import oracle
    oracle.build()
    cfg = inp.cfg
    x = oracle_inputs(inp)
    nth = oracle.num_threads(threads)
    steps, t0 = 0, time.perf_counter()
    while True:
        oracle_full_step(cfg, x, threads)
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return steps, el, nth


def oracle_tiny_single_thread():
    """configs[0] (tiny) on ONE host thread: best of 3 full oracle steps, us."""
    import zoomr_synth as S
    inp = S.generate(S.CONFIGS["tiny"], device="cpu")
    x = oracle_inputs(inp)
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        oracle_full_step(inp.cfg, x, threads=1)
        el = (time.perf_counter() - t0) * 1e6
        best = el if best is None else min(best, el)
    return best


def run_reference(args):
    """Reference arm = the CPU oracle as it stands (there is no reference
    implementation to install: /root/reference holds only the paper and a spec).
    Each step is one FULL oracle step (O1-O7: the whole selection and the
    attention of every layer and head) of one sequence of the workload -- the
    same function the cpu_baseline leg of our arm times.  Under torchrun only
    rank 0 runs it."""
    rank, world, local = init_dist(args.gpus)
    if rank != 0:
        return
    import zoomr_synth as S
    import oracle
    oracle.build()
    cfg = S.config_by_name(args.workload)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    inp = S.generate(cfg, device=dev, batch=1, query_mode=args.query)
    x = oracle_inputs(inp)
    for _ in range(args.warmup):
        r = oracle_full_step(cfg, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle_full_step(cfg, x)
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    val = 1.0 / step_s
    cores = oracle.num_threads(0)
    sample = (f"per step: one full oracle step (a1-a5, all {cfg.L}x{cfg.Hq} heads) of one {cfg.name} sequence "
              f"(zoomr_oracle_step, fp64, OpenMP over (layer, head)); seqs/s = 1 / mean step time")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "seqs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(cfg, args, args.gpus, 1, int(inp.num_summaries[0])),
        "index_count": int(len(r["index"])),
        "step_ms_pcts": {k: v * 1e3 for k, v in pcts(times).items()},
        "cpu_baseline": {"value": val, "unit": "seqs/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": val, "unit": "seqs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm ----
def token_shard_section(shape, prm, s0, cfg, K, world_sim=8):
    import numpy as np
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
    inp, kv, seg = s0["inp"], s0["kv"], s0["seg"]
    Bseq = inp.q.shape[0]
    own_np = token_owner_map(inp.bounds.cpu().numpy(), inp.num_summaries.cpu().numpy(), world_sim,
                             int(inp.seq_len.max()), 64)
    owner = torch.from_numpy(own_np).cuda()
    steps = []

    def exchange(out, lse, count, po, pl, pc):
        for r, t in enumerate(steps):
            po[r].copy_(t.out_local)
            pl[r].copy_(t.lse_local)
            pc[r].copy_(t.local_count)
    for r in range(world_sim):
        t = TokenShardedStep(shape, r, world_sim, Bseq, inp.bounds.shape[1], cfg.T, prm, exchange=exchange,
                             reduce_mean_keys=lambda mk: None)
        t.mean_keys.copy_(s0["st"].mean_keys)  # the replicated cache
        steps.append(t)
    graphs = []
    for t in steps:
        t.run_local(inp.q, kv, seg, owner)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            t.run_local(inp.q, kv, seg, owner)
        graphs.append(g)
    steps[0].combine()
    torch.cuda.synchronize()
    gm = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gm):
        Z.merge_attn(shape, steps[0].part_out, steps[0].part_lse, steps[0].out, part_count=steps[0].part_count,
                     lse=steps[0].lse)

    def t_us(g):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / K
    per_rank = [t_us(g) for g in graphs]
    merge = t_us(gm)
    s0["g"].replay()  # the unsharded step on the same (possibly decode-loop-appended) cache
    torch.cuda.synchronize()
    err = float((steps[0].out - s0["st"].out).abs().max())
    for t in steps:
        t.check_status()
    L, Hq, d = cfg.L, cfg.Hq, cfg.d
    return {"ranks": world_sim, "rank_step_us_max": max(per_rank), "rank_step_us_mean": sum(per_rank) / world_sim,
            "merge_us": merge, "rank_index_share": [round(int(t.local_count.sum()) / max(1, int(t.count.sum())), 3)
                                                    for t in steps],
            "exchange_bytes_per_rank": Bseq * L * Hq * (d + 1) * 4 + Bseq * 4,
            "max_abs_diff_vs_unsharded": err,
            "note": "ranks simulated one after another on one GPU; each rank: a2+a3+a4 (replicated) + "
                    "shard_index + a5 with lse over its part of I_f; NVLink all-gather not included"}


def c3_section(rank, world, K, W, hbm):
    """BASELINE configs[2]: Llama-3-8B shape, 32K context, batch 64, batch-sharded
    over the ranks (64 / N sequences each, no collective).  When a rank's share of
    the KV does not fit its HBM (N = 1: 275 GB), logical pages alias onto a smaller
    physical pool by a seeded hash: the bytes read per step are
    unchanged, and the pool (~1000x L2) gives no cross-sequence L2 reuse."""
    import zoomr_synth as S
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import shard_range
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    cfg = S.CONFIGS["8b32k"]
    lo, hi = shard_range(cfg.batch, rank, world)
    nb = hi - lo
    page_bytes = 2 * cfg.L * cfg.Hkv * cfg.page * cfg.d * 2
    need_pages = nb * cfg.pages_per_seq
    free = torch.cuda.mem_get_info()[0]
    budget = free - (24 << 30)  # mean keys, index, workspaces, generator temporaries
    phys = None if need_pages * page_bytes <= budget else max(1, int(budget // page_bytes))
    inp = S.generate(cfg, device="cuda", seed=cfg.seed + 1000 * rank, batch=nb, phys_pages=phys)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    st = ZoomrStep(shape, nb, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    g = st.capture(inp.q, kv, seg, close_items=newest)
    ga = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga):
        st.attend(inp.q, kv, inp.seq_len)
    g.replay()
    torch.cuda.synchronize()
    st.check_status()
    Kc = max(5, min(K, 30))
    barrier(world)
    ts = per_step_us(lambda i: g.replay(), Kc, max(2, min(W, 5)))
    ta = per_step_us(lambda i: ga.replay(), Kc, 2)
    st.check_status()
    counts = [int(c) for c in st.count.cpu()]
    nsum = [int(n) for n in inp.num_summaries.cpu()]
    by = algorithmic_bytes(cfg, counts, nsum, closures=nb)
    step_us = statistics.median(ts)
    step_max = max_over_ranks(step_us, world)
    a5_us = statistics.median(ta)
    res = {"workload": "8b32k (configs[2])", "global_batch": cfg.batch, "ranks": world, "batch_per_rank": nb,
           "aliased_phys_pages": phys, "logical_pages": need_pages,
           "kv_gb_per_rank": (phys or need_pages) * page_bytes / 1e9,
           "step_us_median": step_us, "step_us_pcts": pcts(ts), "step_us_max_over_ranks": step_max,
           "seqs_per_s": cfg.batch / (step_max * 1e-6),
           "bytes_per_step": by["total"], "step_frac_of_hbm_peak": by["total"] / (step_us * 1e-6) / 1e9 / hbm,
           "a5_us_median": a5_us, "a5_frac_of_hbm_peak": by["a5"] / (a5_us * 1e-6) / 1e9 / hbm,
           "index_count_mean": sum(counts) / len(counts), "timing": "median of per-replay CUDA events, "
           f"{Kc} replays; seqs/s = 64 / max over ranks"}
    del st, inp, g, ga
    torch.cuda.empty_cache()
    return res


def head_sharded_section(rank, world, K, W, hbm):
    """BASELINE configs[3]: Llama-3-70B shape, 64K context, batch 1, KV-head-sharded
    (SURVEY 8(e).2): each rank owns 8 / N KV heads and their query heads for all 80
    layers; a1, a2 and a5 are local; ONE NCCL all-reduce(SUM) of the int64
    `partial` (votes, fixed-point A) sits between a2 and a3, captured in the CUDA
    graph with the step.  At N = 1 this is a dry run of rank 0 of an 8-way split
    over a 1-rank NCCL communicator (the all-reduce kernel runs, but no NVLink
    transfer).  Reported with and without the all-reduce, at U = 1 / 16 / 64."""
    import socket
    import torch.distributed as dist
    import zoomr_synth as S
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import nccl_allreduce_sum
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    full = S.CONFIGS["70b64k"]
    n_sh = 8 if world == 1 else world
    if full.Hkv % n_sh:
        return {"skipped": f"{n_sh} ranks do not divide H_kv = {full.Hkv}"}
    own_group = False
    if world == 1 and not dist.is_initialized():
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        own_group = True
    # the rank's heads, generated at that size (same distribution as a slice of the full model)
    cfg = dataclasses.replace(full, Hq=full.Hq // n_sh, Hkv=full.Hkv // n_sh)
    inp = S.generate(cfg, device="cuda", seed=full.seed + 100 * rank)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
    ar = nccl_allreduce_sum()
    NS = 10  # steps per graph: a decode loop enqueues steps back to back (no per-step launch gap)

    def multi(**kw):
        return st.capture(inp.q, kv, seg, close_items=newest, steps=NS, **kw)
    # select_front -> all-reduce -> select_tail -> a5 (the product path, HeadShardedStep.run)
    g_ar = multi(allreduce=ar)
    g_no = multi(allreduce=lambda t: None)     # the same launches without the exchange
    g_sep = multi(allreduce=ar, fused=False)   # a1 / a2 / all-reduce / a3 / a4 / a5 separately
    g_light = st.capture(inp.q, kv, seg, update_selection=False, steps=NS)
    g_ar.replay()
    torch.cuda.synchronize()
    st.check_status()
    Kc = max(5, min(K, 30))
    barrier(world)
    t_ar = [x / NS for x in per_step_us(lambda i: g_ar.replay(), Kc, max(3, min(W, 10)))]
    t_no = [x / NS for x in per_step_us(lambda i: g_no.replay(), Kc, 3)]
    t_sep = [x / NS for x in per_step_us(lambda i: g_sep.replay(), Kc, 3)]
    t_li = [x / NS for x in per_step_us(lambda i: g_light.replay(), Kc, 3)]
    st.check_status()
    m_ar, m_no, m_li = statistics.median(t_ar), statistics.median(t_no), statistics.median(t_li)
    m_ar_max = max_over_ranks(m_ar, world)
    cnt = int(st.count[0])
    by = algorithmic_bytes(cfg, [cnt], [int(inp.num_summaries[0])])
    res = {"workload": "70b64k (configs[3])", "shards": n_sh, "ranks_executed": world,
           "heads_per_rank": {"H_kv": cfg.Hkv, "H_q": cfg.Hq, "L": cfg.L},
           "communicator": "NCCL, world 1 (dry run: the all-reduce kernel, no transfer)" if world == 1
           else f"NCCL, world {world}",
           "allreduce_bytes": int(st.partial.numel() * 8), "index_count": cnt,
           "step_us_U1_with_allreduce": m_ar, "step_us_U1_with_allreduce_pcts": pcts(t_ar),
           "step_us_U1_with_allreduce_max_over_ranks": m_ar_max,
           "step_us_U1_without_allreduce": m_no, "allreduce_us": m_ar - m_no,
           "step_us_U1_separate_launches": statistics.median(t_sep),
           "step_us_held_selection": m_li,
           "step_us_U16": (m_ar + 15 * m_li) / 16, "step_us_U64": (m_ar + 63 * m_li) / 64,
           "seqs_per_s_U1": 1e6 / m_ar_max,
           "bytes_per_step_per_rank": by["total"],
           "step_frac_of_hbm_peak_U1": by["total"] / (m_ar * 1e-6) / 1e9 / hbm,
           "path": "zoomr_select_front (a1 + a2) -> NCCL all-reduce of partial -> zoomr_select_tail (a3 + a4) -> "
                   "a5 with early rows; timed as graphs of 10 back-to-back steps (median of per-replay events / 10); "
                   "U = 16 / 64 = one update step + U-1 held-selection steps (a4 + a5)"}
    del st, inp, g_ar, g_no, g_sep, g_light
    torch.cuda.empty_cache()
    if own_group:
        dist.destroy_process_group()
    return res


def layer_pipelined_section(shape, prm, s0, cfg, host_k, host_v, cache_bytes):
    from oracle.transfer import simulate_transfer_schedule
    from paper_2604_10898_b200.tier import LayerPipelinedTierStep
    inp = s0["inp"]
    seg = s0["seg"]
    out = {}

    def g_time(fn, n=3):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        best = None
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e3
            best = t if best is None else min(best, t)
        return best
    for lg in (1, 4):
        # slices sized for |I_f| <= 4096 rows (C2's largest |I_f| is 2836): a step with more reports CAPACITY
        st = LayerPipelinedTierStep(shape, inp.bounds.shape[1], 4096, prm, host_k, host_v, inp.page_table,
                                    layers_per_slice=lg)
        st.mean_keys.copy_(s0["st"].mean_keys)
        st.run(inp.q, seg)
        torch.cuda.synchronize()
        st.check_status()
        ng = cfg.L // lg
        t_sel = g_time(lambda: st.select(inp.q, seg))
        t_in = [g_time(lambda g=g: st.gather(g)) for g in range(ng)]
        t_c = [g_time(lambda g=g: st.attend_group(inp.q, g)) for g in range(ng)]
        t_pipe = g_time(lambda: st.run(inp.q, seg))
        t_serial = g_time(lambda: st.run(inp.q, seg, pipelined=False))
        sim = simulate_transfer_schedule(t_in, t_c)
        cnt = int(st.count[0])
        slice_bytes = cnt * lg * cfg.Hkv * cfg.d * 2 * 2
        st.check_status()
        out[f"layers_per_slice_{lg}"] = {
            "step_us_pipelined": t_pipe, "step_us_serial": t_serial, "select_us": t_sel,
            "gather_us_per_group_mean": sum(t_in) / ng, "attend_us_per_group_mean": sum(t_c) / ng,
            "model_total_us": t_sel + sim["total_time"], "model_serial_us": t_sel + sim["serial_time"],
            "model_vs_measured_pipelined": (t_sel + sim["total_time"]) / t_pipe,
            "model_peak_resident_slices": sim["peak_resident_layers"],
            "host_link_gbs": slice_bytes / (sum(t_in) / ng * 1e-6) / 1e9,
            "hbm_bytes": st.hbm_bytes(), "hbm_saving": cache_bytes / st.hbm_bytes(), "index_count": cnt}
        del st
    out["note"] = ("the paper's system: each step reloads I_f's rows layer group by layer group from pinned host "
                   "memory (SM-driven zero-copy gather) into one of two HBM slices while the previous group attends; "
                   "model = select + SPEC simulate_transfer_schedule(measured per-group gather, attend times)")
    return out


def host_tier_section(shape, prm, s0, cfg, K, hot_page_sizes=(64, 16)):
    """NEXT-2: the cache in pinned host memory, an HBM hot pool caching its pages."""
    from paper_2604_10898_b200.tier import HostTierStep
    inp = s0["inp"]
    B = inp.q.shape[0]
    host_k, host_v = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
    seg = s0["seg"]
    cache_bytes = host_k.numel() * 4  # K and V

    def ev_time(fn, n=1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n  # us

    def make(ph, hot_pages):
        st = HostTierStep(shape, B, inp.bounds.shape[1], cfg.T, prm, host_k, host_v, inp.page_table, hot_pages,
                          hot_page_size=ph)
        st.mean_keys.copy_(s0["st"].mean_keys)
        return st
    qa = inp.q
    g = torch.Generator(device="cuda").manual_seed(5)
    qb = (torch.randn(qa.shape, device="cuda", generator=g)).bfloat16()  # another query: other zoomed segments
    res = {}
    for ph in hot_page_sizes:
        if cfg.page % ph:
            continue
        page_bytes = 2 * cfg.L * cfg.Hkv * ph * cfg.d * 2  # K and V, every layer
        all_pages = int(inp.k_pool.shape[1]) * (cfg.page // ph)
        st = make(ph, all_pages)
        cold = []
        for _ in range(3):
            st.hot_page_table.fill_(-1)
            st.hot_owner.fill_(-1)
            st.hot_stamp.fill_(-1)
            cold.append(ev_time(lambda: st.run(qa, seg)))
            st.check_status()
        n_cold = st.fetched_pages()
        warm = ev_time(lambda: st.run(qa, seg), K)
        cold_us = sorted(cold)[1]
        # churn: the two queries alternate on a pool 8 pages larger than one step's pages
        del st
        tight = n_cold + 8
        st = make(ph, tight)
        st.run(qa, seg)
        st.run(qb, seg)
        torch.cuda.synchronize()
        i = [0]

        def alt():
            st.run(qa if i[0] % 2 == 0 else qb, seg)
            i[0] += 1
        churn = ev_time(alt, 20)
        sw = []
        for q_ in (qa, qb):
            st.run(q_, seg)
            torch.cuda.synchronize()
            sw.append(st.fetched_pages())
        st.check_status()
        del st
        res[f"hot_page_{ph}"] = {
            "cold_pages": n_cold, "cold_bytes": n_cold * page_bytes, "hbm_saving": cache_bytes / (n_cold * page_bytes),
            "cold_step_us": cold_us, "cold_fetch_gbs": n_cold * page_bytes / ((cold_us - warm) * 1e-6) / 1e9,
            "warm_step_us": warm, "alternating_pool_pages": tight, "alternating_us_per_step": churn,
            "alternating_pages_per_switch": sw}
    # Algorithm 1's decode loop over the tier: 256 tokens in one graph, a sentence boundary
    # every 35 tokens, write-through append to the host cache; hot pages of the host page
    # size (the loop's default) and of 16 tokens (1/4 of the HBM per touched page)
    from paper_2604_10898_b200.tier import TierDecodeLoop
    n_tok = 256
    start = inp.seq_len - n_tok
    kin = torch.randn(B, cfg.L, cfg.Hkv, cfg.d, device="cuda").bfloat16()
    vin = torch.randn_like(kin)
    toks = torch.tensor([[200 if (i % 35) == 34 else 7] * B for i in range(n_tok)], dtype=torch.int32,
                        device="cuda")
    for ph, key in ((cfg.page, "decode_loop_us_per_token"), (16, "decode_loop_us_per_token_hot16")):
        if cfg.page % ph:
            continue
        lp = TierDecodeLoop(shape, B, inp.bounds.shape[1], cfg.T, prm, host_k, host_v, inp.page_table,
                            int(inp.k_pool.shape[1]) * (cfg.page // ph), 1000, 1001, [200], hot_page_size=ph)
        lp.mean_keys.copy_(s0["st"].mean_keys)
        lp.start_from(inp.bounds, inp.num_summaries, start)
        gl_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gl_):
            for i in range(n_tok):
                lp.decode_step(kin, vin, qa, toks[i])

        def loop_run():
            lp.seq_len.copy_(start)
            return ev_time(gl_.replay) / n_tok
        loop_run()  # first pass: cold fetches
        res[key] = loop_run()
        lp.check_status()
        del lp, gl_
    # the paper's own transfer schedule: per step, the rows of I_f of each layer
    # group gathered host -> HBM slice on a copy stream while the previous group attends,
    # two slices resident; checked against SPEC's transfer-schedule model (oracle/transfer.py)
    # fed with the per-group transfer and compute times measured here
    if B == 1:
        res["paper_layer_pipelined"] = layer_pipelined_section(shape, prm, s0, cfg, host_k, host_v, cache_bytes)
    hb = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    db = torch.empty_like(hb, device="cuda")
    res["host_link_memcpy_gbs"] = hb.numel() / (ev_time(lambda: db.copy_(hb, non_blocking=True), 5) * 1e-6) / 1e9
    res["host_cache_bytes"] = cache_bytes
    res["note"] = ("cache in pinned host memory; per step: fused select + tier fetch (plan + copy of the missing "
                   "hot pages over the host link) + a5 on the HBM hot pool; hbm_saving = cache bytes / hot bytes "
                   "one step needs; alternating: two queries with different zoomed segments on a pool of one "
                   "step's pages + 8")
    return res


def run_ours(args):
    rank, world, local = init_dist(args.gpus)
    import zoomr_synth as S
    from paper_2604_10898_b200 import _build
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    if not torch.cuda.is_available():
        raise SystemExit("bench.py (ours) needs a CUDA device")
    _build.build()
    cfg = S.config_by_name(args.workload)
    # batch sharding: the workload's batch is split over the ranks (configs[2]: 64 sequences
    # over 1..8 GPUs), or --batch-per-gpu fixes the per-rank share
    from paper_2604_10898_b200.parallel import shard_range
    lo, hi = shard_range(cfg.batch, rank, world)
    per_rank = args.batch_per_gpu or max(1, hi - lo)
    if per_rank != cfg.batch:
        cfg = dataclasses.replace(cfg, batch=per_rank)
    # a rank's share that does not fit its HBM (e.g. configs[2] at N < 8): one input set
    # instead of `rotate` (a step then reads far more than L2 anyway), then logical pages
    # aliased onto a smaller physical pool (seeded hash; bytes per step unchanged)
    page_bytes = 2 * cfg.L * cfg.Hkv * cfg.page * cfg.d * 2
    budget = 0.80 * torch.cuda.get_device_properties(local).total_memory
    R = max(1, args.rotate)
    set_bytes = cfg.batch * cfg.pages_per_seq * page_bytes
    phys_pages = None
    if set_bytes * R > budget:
        R = 1
        args.rotate = 1
        if set_bytes > budget:
            phys_pages = int(budget // page_bytes)
    U = max(1, cfg.update_every)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
    sets = []
    for r in range(R):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 1000 * rank + 17 * r, query_mode=args.query,
                         phys_pages=phys_pages)
        st = ZoomrStep(shape, inp.q.shape[0], inp.bounds.shape[1], cfg.T, prm, early_known=not args.no_early)
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))  # initial cache (untimed)
        # the newest closed summary of every sequence: re-derived every step (a1 amortized)
        newest = torch.tensor([[b, int(inp.num_summaries[b]) - 1] for b in range(inp.q.shape[0])],
                              dtype=torch.int32, device="cuda")
        g = st.capture(inp.q, kv, seg, update_selection=True, close_items=newest)
        # selection held between updates (U > 1): a4 + a5 only (reading Q14)
        gl = st.capture(inp.q, kv, seg, update_selection=False) if U > 1 else None
        # a5 alone (for the kernel roofline), same buffers
        phys = st.index_phys if st.use_phys else None
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga):
            st.attend(inp.q, kv, inp.seq_len)
        g.replay()  # leave the full selection's flags / index in place
        sets.append(dict(inp=inp, st=st, g=g, gl=gl, ga=ga, kv=kv, seg=seg, newest=newest, phys=phys))
    torch.cuda.synchronize()
    for s in sets:
        s["st"].check_status()
    # a5 alone for the roofline: 2 x R launches per graph replay (the R input sets in
    # turn, > L2), so the average per launch is the kernel's, not a graph launch's
    # (one a5 per replay adds ~2-3 us of replay overhead per launch: `launch_us_single_replay`)
    A5_REP = 2
    ga_multi = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga_multi):
        for _ in range(A5_REP):
            for s in sets:
                s["st"].attend(s["inp"].q, s["kv"], s["inp"].seq_len)
    ga_multi.replay()
    torch.cuda.synchronize()
    full_launch = sets[0]["st"].launches_per_step(update_selection=True, close=True)
    light_launch = sets[0]["st"].launches_per_step(update_selection=False)
    counts = [[int(c) for c in s["st"].count.cpu()] for s in sets]
    nsum = [[int(n) for n in s["inp"].num_summaries.cpu()] for s in sets]
    per_set_bytes = [algorithmic_bytes(cfg, counts[i], nsum[i]) for i in range(R)]
    light_set_bytes = [algorithmic_bytes(cfg, counts[i], [0] * len(nsum[i]), closures=0) for i in range(R)]

    def is_full(i):  # step i uses set i % R; each set updates its selection every U of its steps
        return (i // R) % U == 0

    def step_fn(i):
        s = sets[i % R]
        (s["g"] if is_full(i) else s["gl"]).replay()

    def timed(fn, K, W):
        for i in range(W):
            fn(i)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(K):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
        return e0.elapsed_time(e1) / 1e3  # s

    K, W = args.steps, max(3, args.warmup)
    clk = ClockSampler(local).__enter__()
    time.sleep(1.0)  # let nvidia-smi start sampling before the timed region
    t_step = timed(step_fn, K, W)
    if len(clk.rows) < 3:  # short run: keep the GPU busy with timed-equivalent replays while sampling
        for _ in range(3):
            timed(step_fn, K, 0)
    clk.__exit__()
    t_step_max = max_over_ranks(t_step, world)
    step_times = per_step_us(step_fn, K, W)  # p10 / p50 / p90 (separate pass)
    t_attn_single = timed(lambda i: sets[i % R]["ga"].replay(), K, W)
    n_multi_a5 = max(1, K // (A5_REP * R))
    t_attn = timed(lambda i: ga_multi.replay(), n_multi_a5, W) / (n_multi_a5 * A5_REP * R) * K  # K launches' worth
    bytes_mean = sum((per_set_bytes if is_full(i) else light_set_bytes)[i % R]["total"] for i in range(K)) / K
    a5_mean = sum(per_set_bytes[i % R]["a5"] for i in range(K)) / K
    Bseq = sets[0]["inp"].q.shape[0]

    # e2e through the public API: pinned host q in, fp32 out back to host, every step
    qh = [s["inp"].q.cpu().pin_memory() for s in sets]
    oh = [torch.empty_like(s["st"].out, device="cpu").pin_memory() for s in sets]

    def e2e_step(i):
        s = sets[i % R]
        s["inp"].q.copy_(qh[i % R], non_blocking=True)
        (s["g"] if is_full(i) else s["gl"]).replay()
        oh[i % R].copy_(s["st"].out, non_blocking=True)
    t_e2e_serial = max_over_ranks(timed(e2e_step, K, W), world)

    # the same, pipelined as a serving loop would run it: step i+1's q goes up on a
    # copy stream while step i computes, and step i's output comes down on another
    # copy stream while step i+1 computes (events order every buffer reuse; the R
    # input sets are the buffers).  Every step still moves its q in and its out back.
    cs = torch.cuda.current_stream()
    s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_pipelined(K_, W_):
        q_ready = [torch.cuda.Event() for _ in range(R)]
        out_done = [torch.cuda.Event() for _ in range(R)]
        out_read = [torch.cuda.Event() for _ in range(R)]
        for r in range(R):  # recorded once so that the first waits are satisfied
            out_done[r].record(cs)
            out_read[r].record(cs)

        def up(i):
            r = i % R
            with torch.cuda.stream(s_up):
                s_up.wait_event(out_done[r])  # the step that last read this q has finished
                sets[r]["inp"].q.copy_(qh[r], non_blocking=True)
                q_ready[r].record(s_up)

        def run(n):
            up(0)
            for i in range(n):
                r = i % R
                if i + 1 < n:
                    up(i + 1)
                cs.wait_event(q_ready[r])
                cs.wait_event(out_read[r])  # this set's previous output has reached the host
                (sets[r]["g"] if is_full(i) else sets[r]["gl"]).replay()
                out_done[r].record(cs)
                with torch.cuda.stream(s_down):
                    s_down.wait_event(out_done[r])
                    oh[r].copy_(sets[r]["st"].out, non_blocking=True)
                    out_read[r].record(s_down)
            cs.wait_stream(s_down)
        run(W_)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        run(K_)
        e1.record(cs)
        torch.cuda.synchronize()
        barrier(world)
        return e0.elapsed_time(e1) / 1e3
    t_e2e = max_over_ranks(e2e_pipelined(K, W), world)
    h2d = sets[0]["inp"].q.numel() * 2
    d2h = sets[0]["st"].out.numel() * 4

    # Steps enqueued back to back (a serving loop capturing several steps per
    # graph): R x 4 full steps in one graph, plain launches vs the chained ones
    # (zoomr_select_fused_chained runs a1/a2 while the previous step's a5
    # finishes).  Informational: `value` stays one step per graph replay.
    chained = None
    if U == 1:
        def multi_graph(flag):
            for s in sets:
                s["st"].chained = flag
            gm_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gm_):
                for _ in range(4):
                    for s in sets:
                        s["st"].run(s["inp"].q, s["kv"], s["seg"], close_items=s["newest"])
            for s in sets:
                s["st"].chained = False
            return gm_
        g_plain, g_chain = multi_graph(False), multi_graph(True)
        n_multi = max(1, K // (4 * R))
        t_plain = max_over_ranks(timed(lambda i: g_plain.replay(), n_multi, 2), world) / (n_multi * 4 * R)
        t_chain = max_over_ranks(timed(lambda i: g_chain.replay(), n_multi, 2), world) / (n_multi * 4 * R)
        for s in sets:
            s["g"].replay()  # leave each set's one-step state in place
        torch.cuda.synchronize()
        for s in sets:
            s["st"].check_status()
        chained = {"steps_per_graph": 4 * R, "plain_us_per_step": t_plain * 1e6, "chained_us_per_step": t_chain * 1e6,
                   "chained_seqs_per_s": world * Bseq / t_chain,
                   "note": "zoomr_select_fused_chained + zoomr_sparse_decode_attn_chained: a1/a2 of step t+1 "
                           "overlap the end of step t's a5 (PDL); outputs bit-identical (tests/test_gpu_paths.py)"}

    # Algorithm 1's whole decode step on the device (append, segment tracking,
    # selection update at semantic boundaries only, I_f rebuild, attention):
    # one graph replay per token over the last 256 positions of a context,
    # a sentence boundary every 35 tokens -- informational, not `value`.
    decode_loop = None
    if world == 1 and not args.no_loop:
        from paper_2604_10898_b200.step import DecodeLoop
        s0 = sets[0]
        inp0 = s0["inp"]
        n_tok = 256
        start = inp0.seq_len - n_tok
        nmax0 = inp0.bounds.shape[1]
        extra = 8  # room for the summaries that close during the stretch
        # the closed summaries must end before the appended stretch (the bench context keeps its
        # open tail > 256 tokens, so they do)
        bpad = torch.zeros(Bseq, nmax0 + extra, 4, dtype=torch.int32, device="cuda")
        bpad[:, :nmax0] = inp0.bounds
        kin = torch.randn(Bseq, cfg.L, cfg.Hkv, cfg.d, device="cuda").bfloat16()
        vin = torch.randn_like(kin)
        # the token stream: regular text with a sentence boundary every 35 tokens,
        # and every LR+LS tokens a summary (begin delimiter, LS-2 summary tokens, end
        # delimiter): each end closes a summary (a1 on closure, N_t grows), so
        # selection updates see N_t = 120, 121, ...
        toks = []
        for i in range(n_tok):
            r = i % (cfg.LR + cfg.LS)
            if r == cfg.LR:
                toks.append(1000)
            elif r == cfg.LR + cfg.LS - 1:
                toks.append(1001)
            elif (i % 35) == 34:
                toks.append(200)
            else:
                toks.append(7)
        tok_dev = torch.tensor([[t] * Bseq for t in toks], dtype=torch.int32, device="cuda")
        def loop_time(**kw):
            lp = DecodeLoop(shape, Bseq, nmax0 + extra, cfg.T, prm, 1000, 1001, [200], **kw)
            lp.mean_keys[:, :, :, :nmax0].copy_(s0["st"].mean_keys)
            lp.start_from(bpad, inp0.num_summaries, start)
            gl_ = torch.cuda.CUDAGraph()  # all n_tok decode steps in one graph
            with torch.cuda.graph(gl_):
                for i in range(n_tok):
                    lp.decode_step(s0["kv"], kin, vin, inp0.q, tok_dev[i])

            def loop_run():
                lp.start_from(bpad, inp0.num_summaries, start)  # T, N_t, segment table, tracker: as at the start
                lp.flags[:, :nmax0].copy_(s0["st"].flags)  # the selection before the stretch (held to a boundary)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gl_.replay()
                e1.record()
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) * 1e3 / n_tok
            loop_run()
            us = loop_run()
            lp.check_status()
            return lp, us
        lp, us = loop_time()
        n_closed = int(lp.num_summaries[0]) - int(inp0.num_summaries[0])
        del lp
        _, us_sep = loop_time(chained=False, fused_a0=False)
        decode_loop = {"us_per_token": us, "tokens": n_tok, "selection_updates": sum(t == 200 for t in toks),
                       "summaries_closed": n_closed, "launches_per_token": 4,
                       "separate_us_per_token": us_sep,
                       "note": "zoomr_append_track (row copy + tracking kernel, PDL behind the chained a5) + fused "
                       "select (a1 at summary closures, a2/a3 at sentence boundaries only) + chained a5; the "
                       "256 steps captured in one CUDA graph.  separate_us_per_token: append + advance, track, select, "
                       "plain a5 as 5 plain launches (the round-1 loop)"}
    # the paper's comparison policies on the same kernels (NEXT-3), informational:
    # StreamingLLM at ZoomR's budget (mean |I_f|), SumR (all summaries kept): a4 + a5 per step;
    # H2O at the same budget: eviction by cumulative attention + a5 with logits + accumulation
    policies = None
    if world == 1 and not args.no_loop:
        from paper_2604_10898_b200.policies import PolicyStep
        budget = int(round(sum(sum(c) for c in counts) / sum(len(c) for c in counts)))
        policies = {}
        for pol in ("streamingllm", "sumr", "h2o"):
            gs, cnt_pol = [], []
            for s_ in sets:
                ps = PolicyStep(pol, shape, Bseq, s_["inp"].bounds.shape[1], cfg.T, prm, budget=budget,
                                max_positions=cfg.T)
                ps.prepare(s_["inp"].num_summaries)
                if pol == "h2o":
                    ps.start_h2o(s_["seg"])
                gp = ps.capture(s_["inp"].q, s_["kv"], s_["seg"], update_selection=False)
                gs.append((gp, ps))
            for i in range(W):
                gs[i % R][0].replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(K):
                gs[i % R][0].replay()
            e1.record()
            torch.cuda.synchronize()
            for gp, ps in gs:
                ps.check_status()
            policies[pol] = {"us_per_step": e0.elapsed_time(e1) * 1e3 / K,
                             "index_count_mean": float(sum(int(ps.count.float().mean()) for _, ps in gs) / R)}
        policies["budget"] = budget
    # token-sharded split-K (NEXT-4), informational: 8 ranks simulated one after
    # another on this GPU, each rank's local step (replicated a2..a4, its part of
    # I_f through a5 with log-sum-exp) timed alone, then the merge; the
    # all-gather of (out, lse, count) between GPUs is not part of these numbers
    token_sharded = None
    if world == 1 and not args.no_loop:
        token_sharded = token_shard_section(shape, prm, sets[0], cfg, K)
    host_tier = None
    if world == 1 and not args.no_loop and sets[0]["inp"].k_pool.numel() * 4 <= (8 << 30):  # pins the cache
        host_tier = host_tier_section(shape, prm, sets[0], cfg, K)
    # per-stage breakdown (informational): each stage alone, graph-replayed
    stages = {}
    s0 = sets[0]
    st, inp = s0["st"], s0["inp"]
    REP = 20  # launches per graph: the per-stage figure is GPU time, not CPU launch overhead

    def cap(fn):
        gg = torch.cuda.CUDAGraph()
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(gg):
            for _ in range(REP):
                fn()
        return gg
    st_graphs = {
        "a1_a4_fused_select": cap(lambda: Z.select_fused(
            shape, inp.q, inp.k_pool, inp.v_pool, inp.page_table, inp.bounds, inp.num_summaries, inp.seq_len,
            s0["newest"], st.mean_keys, cfg.top_k, cfg.c, cfg.sink, cfg.window, st.flags, st.index, st.count,
            st.sel_workspace, partial=st.partial, agreeability=st.agreeability, dev_status=st.status,
            index_phys=s0["phys"])),
        "a1_mean_keys": cap(lambda: st.update_mean_keys(s0["kv"], s0["seg"], s0["newest"])),
        "a2_score": cap(lambda: Z.score(shape, inp.q, st.mean_keys, inp.num_summaries, cfg.top_k, st.partial,
                                        dev_status=st.status)),
        "a3_select_topc": cap(lambda: Z.select_topc(st.partial, inp.num_summaries, cfg.c, st.flags,
                                                    st.agreeability, st.status)),
        "a4_build_index": cap(lambda: Z.build_index(inp.bounds, inp.num_summaries, inp.seq_len, st.flags,
                                                    cfg.sink, cfg.window, st.index, st.count, st.status)),
    }
    for k, gg in st_graphs.items():
        stages[k] = round(timed(lambda i: gg.replay(), 10, 2) / (10 * REP) * 1e6, 2)
    stages["a5_sparse_attn"] = round(t_attn / K * 1e6, 2)
    torch.cuda.synchronize()
    for s in sets:
        s["st"].check_status()

    hbm, peak_src = peaks()
    # configs[2] (batch 64, batch-sharded, aliased pages when a rank's share does not
    # fit) and configs[3] (70B-64K KV-head-sharded with the NCCL all-reduce in the
    # graph; a 1-rank dry run at N = 1) -- sections of the same line
    c3 = None if args.no_c3 else c3_section(rank, world, K, W, hbm)
    head_sharded = None if args.no_heads else head_sharded_section(rank, world, K, W, hbm)
    step_s = t_step_max / K
    value = world * Bseq * K / t_step_max
    attn_s = t_attn / K
    achieved = a5_mean / attn_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(cfg.name, {}).get("a5_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": "seqs/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": workload_config(cfg, args, world, Bseq, nsum[0][0]),
        "index_count_mean": sum(sum(c) for c in counts) / sum(len(c) for c in counts),
        "kv_pages_per_set": {"logical": cfg.batch * cfg.pages_per_seq,
                             "physical": phys_pages or cfg.batch * cfg.pages_per_seq},
        "step_us": step_s * 1e6,
        "step_us_pcts": pcts(step_times),
        "step_roofline": {"bytes_per_step": bytes_mean, "achieved_gbs": bytes_mean / step_s / 1e9,
                          "frac": bytes_mean / step_s / 1e9 / hbm},
        "roofline": {"kernel": "a5 zoomr_sparse_decode_attn", "bound": "hbm", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": a5_mean,
                     "launch_us": attn_s * 1e6, "launch_us_single_replay": t_attn_single / K * 1e6,
                     "timing": f"CUDA events over {n_multi_a5} replays of a graph of {A5_REP * R} a5 launches "
                               f"(the {R} input sets in turn, early rows as in the step), average per launch"},
        "stages_us": stages,
        "decode_loop": decode_loop,
        "chained": chained,
        "policies": policies,
        "token_sharded": token_sharded,
        "host_tier": host_tier,
        "c3": c3,
        "head_sharded": head_sharded,
        "e2e": {"value": world * Bseq * K / t_e2e, "unit": "seqs/s", "pipelined": True,
                "serial_value": world * Bseq * K / t_e2e_serial, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": sum(full_launch if is_full(i) else light_launch for i in range(K)),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        steps, el, nth = oracle_time(sets[0]["inp"], args.cpu_seconds)
        line["cpu_baseline"] = {"value": steps * Bseq / el, "unit": "seqs/s", "cores": nth, "kind": "oracle",
                                "sample": f"{steps} full oracle steps (a1-a5, all {cfg.L}x{cfg.Hq} heads) of "
                                          f"one {cfg.name} sequence, {el:.1f} s",
                                "cpu_model": cpu_model(), "tiny_single_thread_us": oracle_tiny_single_thread()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
