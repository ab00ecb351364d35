"""Full-size GPU parity (BASELINE configs[2..4] and the Qwen shape): the whole
selection over every voter, and every (layer, head) attention output (70B-64K,
8B-32K, the configs[4] L_R = 64 point, Qwen-7B-16K); the KV-head-sharded exchange
simulated on one GPU (one a2 per head shard, partials summed in rank order).
The real exchange through parallel.py's collectives runs in
tests/test_gpu_multiproc.py (2 processes, gloo on CUDA tensors)."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import zoomr_synth as S
from tests import parity as PY

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    from paper_2604_10898_b200 import _build
    _build.build()


def _run(inp, fused=True, capacity=None):
    st = PY.make_step(inp, capacity=capacity)
    PY.run_full(inp, st, fused=fused)
    return st


def test_70b64k_full_size_every_head():
    """configs[3] unsharded at full size (|I_f| up to 6236, 80 layers: the 70B stream-K
    split with ~2.9x the segments and more merges): all 80 x 64 attention outputs."""
    inp = S.generate(S.CONFIGS["70b64k"], device="cuda")
    st = _run(inp, capacity=16384)
    rep = PY.check_sequence_sampled(inp, st, 0, {})
    assert rep["attn_outputs_checked"] == 80 * 64
    print(rep)
    del st, inp
    torch.cuda.empty_cache()


def test_8b32k_batch_subset():
    cfg = dataclasses.replace(S.CONFIGS["8b32k"], batch=3)
    inp = S.generate(cfg, device="cuda")
    st = _run(inp, capacity=8192)
    rep = {}
    for b in range(3):
        PY.check_sequence_sampled(inp, st, b, rep)  # every (layer, head) of every sequence
    print(rep)


def test_8b32k_jitter_layout():
    cfg = dataclasses.replace(S.CONFIGS["8b32k"], batch=2, jitter=True)
    inp = S.generate(cfg, device="cuda")
    st = _run(inp, capacity=8192, fused=False)
    rep = {}
    for b in range(2):
        PY.check_sequence_sampled(inp, st, b, rep, layers=[5], qheads=[3, 17])


@pytest.mark.parametrize("cfg_name,world", [("8b16k", 8), ("8b16k", 2), ("tiny", 2)])
def test_head_sharded_exchange_simulated(cfg_name, world):
    """a2 per KV-head shard + sum of int64 partials == unsharded a2, bit for bit;
    hence identical flags / I_f on every rank, and per-shard a5 == unsharded a5."""
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import HeadShardedStep, local_shape, shard_heads, slice_heads
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    cfg = S.CONFIGS[cfg_name]
    inp = S.generate(cfg, device="cuda")
    full = PY.make_step(inp, capacity=cfg.T)
    PY.run_full(inp, full, fused=False)
    torch.cuda.synchronize()
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    steps, parts = [], []
    for r in range(world):
        sh = shard_heads(cfg.Hq, cfg.Hkv, r, world)
        kp, vp, qq = slice_heads(inp.k_pool, inp.v_pool, inp.q, sh)
        st = ZoomrStep(local_shape(shape, sh), 1, inp.bounds.shape[1], cfg.T, prm)
        kv = (kp, vp, inp.page_table)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        Z.score(st.shape, qq, st.mean_keys, inp.num_summaries, cfg.top_k, st.partial, dev_status=st.status)
        steps.append((st, kv, qq, sh))
        parts.append(st.partial.clone())
    total = torch.zeros_like(parts[0])
    for p in parts:  # the all-reduce(SUM), in rank order
        total += p
    assert torch.equal(total, full.partial)
    for st, kv, qq, sh in steps:  # every rank: a3, a4 on identical inputs, then local a5
        st.partial.copy_(total)
        Z.select_topc(st.partial, inp.num_summaries, cfg.c, st.flags, st.agreeability, st.status)
        Z.build_index(inp.bounds, inp.num_summaries, inp.seq_len, st.flags, cfg.sink, cfg.window, st.index, st.count,
                      st.status)
        Z.sparse_decode_attn(st.shape, qq, kv[0], kv[1], kv[2], st.index, st.count, st.out, st.workspace,
                             dev_status=st.status)
        torch.cuda.synchronize()
        st.check_status()
        assert torch.equal(st.flags, full.flags) and torch.equal(st.count, full.count)
        assert torch.equal(st.index, full.index)
        torch.testing.assert_close(st.out, full.out[:, :, sh.q_start:sh.q_stop], atol=2e-6, rtol=0)


@pytest.mark.parametrize("LR,c", [(64, 8), (1024, 32)])
def test_stress_128k_sampled(LR, c):
    """configs[4]: 128K context on the 8B shape (N_t = 1631 at L_R = 64: the vote-histogram
    top-c path and a 10k+ entry index set; L_R = 1024: 33k+ token zoomed segments)."""
    cfg = S.stress_config(LR, c)
    inp = S.generate(cfg, device="cuda")
    st = _run(inp, capacity=cfg.T)
    # every (layer, head) at the L_R = 64 point (N_t = 1631); sampled at L_R = 1024 (|I_f| ~ 34K rows)
    rep = PY.check_sequence_sampled(inp, st, 0, {}, **({} if LR == 64 else dict(layers=[0, 17], qheads=[1, 30])))
    print(cfg.name, rep.get("index_counts"), rep.get("attn_max_abs_err"))
    del st, inp
    torch.cuda.empty_cache()


def test_update_interval_holds_flags():
    """U > 1 (reading Q11/Q14): between selection updates a4 re-derives the window from
    the current T with the held flags; compare with the oracle's index for the held flags."""
    cfg = S.CONFIGS["tiny"]
    inp = S.generate(cfg, device="cuda", seed=3)
    st = PY.make_step(inp)
    PY.run_full(inp, st)
    flags = st.flags.clone()
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    inp.seq_len.fill_(cfg.T - 7)  # an earlier step: the window slides back, flags are held
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.run(inp.q, kv, seg, update_selection=False)
    torch.cuda.synchronize()
    assert torch.equal(st.flags, flags)
    seg_h = PY.seg_host(inp, 0)
    idx_ref = oracle.build_index(seg_h, flags[0, :len(seg_h)].cpu().numpy(), cfg.T - 7, cfg.sink, cfg.window)
    cnt = int(st.count[0])
    assert np.array_equal(st.index[0, :cnt].cpu().numpy(), idx_ref)


def test_qwen_shape_g7_full_size_sampled():
    """NEXT-4: the Qwen2.5-7B grouping (28 query / 4 KV heads, G = 7) at 16K, full size."""
    inp = S.generate(S.CONFIGS["qwen7b16k"], device="cuda")
    st = _run(inp, capacity=8192)
    rep = {}
    PY.check_sequence_sampled(inp, st, 0, rep)  # every (layer, head)
    print(rep)


def test_many_wave_select_grids_qwen_batch3():
    """A grid of more than one wave of 256-thread CTAs takes the select's small-CTA
    instantiation (64 threads, eight per SM): G = 7 at batch 3 (3 x 113 CTAs) -- a1
    bit-exact, votes exact, flags / I_f exact, sampled attention within the rule."""
    cfg = dataclasses.replace(S.CONFIGS["qwen7b16k"], batch=3, seed=77)
    inp = S.generate(cfg, device="cuda")
    st = _run(inp, capacity=8192)
    rep = {}
    for b in range(3):
        PY.check_sequence_sampled(inp, st, b, rep, layers=[0, 27], qheads=[0, 13, 27])
    print(rep)
