"""GPU parity of the token-sharded split-K path.

R ranks are simulated one after another on one GPU (no rank waits on another):
each owns the tokens of `token_owner_map`, computes the mean keys of its own
summaries, runs the replicated selection and a5 over its part of I_f with the
log-sum-exp (zoomr_shard_index, zoomr_sparse_decode_attn_lse); the "exchange"
copies every rank's (out, lse, count) into the part buffers and
zoomr_merge_attn combines them.  Checked against the oracle: the replicated
mean keys and I_f bit-exactly, every rank's part of I_f exactly, each rank's
output and lse (O7, O8 over that part), and the merged output and lse over I_f.

Marked `gpu`: run on a B200 with the built libzoomr.so."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import zoomr_synth as S
from tests import parity as PY

pytestmark = pytest.mark.gpu

ATOL_OUT = 2e-3   # north_star's attention tolerance
ATOL_LSE = 1e-4   # fp32 logits (|z| <~ 10) and fp32 sums: ~1e-5 expected


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    from paper_2604_10898_b200 import _build
    _build.build()


def _small(name, **kw):
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=128, T=2048, n_pairs=24, LR=60, LS=12, sink=4, window=96,
                c=3, top_k=2, page=32, seed=51, batch=2)
    base.update(kw)
    return S.Config(**base)


def _simulate(inp, world, owner_np=None, chunk=64):
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    cfg = inp.cfg
    B = inp.q.shape[0]
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    stride = int(inp.seq_len.max().item())
    if owner_np is None:
        owner_np = token_owner_map(inp.bounds.cpu().numpy(), inp.num_summaries.cpu().numpy(), world, stride, chunk)
    owner = torch.from_numpy(owner_np).to("cuda")
    params = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
    steps = []

    def exchange(out, lse, count, po, pl, pc):  # what the all-gather delivers
        for r, s in enumerate(steps):
            po[r].copy_(s.out_local)
            pl[r].copy_(s.lse_local)
            pc[r].copy_(s.local_count)

    def no_reduce(mk):
        pass

    for r in range(world):
        steps.append(TokenShardedStep(shape, r, world, B, inp.bounds.shape[1], cfg.T, params, device="cuda",
                                      debug_outputs=True, exchange=exchange, reduce_mean_keys=no_reduce))
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    # a1 on the summaries each rank owns (ownership of a summary = of its first token)
    items = ZoomrStep.all_items(inp.num_summaries).cpu().numpy()
    for r, st in enumerate(steps):
        mine = [(b, i) for b, i in items if owner_np[b, int(inp.bounds[b, i, 2])] == r]
        t = torch.tensor(mine, dtype=torch.int32, device="cuda").reshape(-1, 2)
        st.update_mean_keys(kv, seg, t)
    total = sum(st.mk_local for st in steps)  # what the all-reduce(SUM) delivers
    for st in steps:
        st.mean_keys.copy_(total)
    for st in steps:
        st.run_local(inp.q, kv, seg, owner)
    for st in steps:
        st.combine()
    torch.cuda.synchronize()
    for st in steps:
        st.check_status()
    return steps, owner_np


def _check(inp, steps, owner_np):
    cfg = inp.cfg
    L, Hq, Hkv, d = cfg.L, cfg.Hq, cfg.Hkv, cfg.d
    ref = PY.make_step(inp)
    PY.run_full(inp, ref, fused=False)
    for st in steps[1:]:
        assert torch.equal(st.out, steps[0].out) and torch.equal(st.lse, steps[0].lse)  # same on every rank
    for st in steps:
        assert torch.equal(st.mean_keys, ref.mean_keys)  # replicated cache, bit-exact
        assert torch.equal(st.count, ref.count)
        for b in range(inp.q.shape[0]):
            n = int(ref.count[b])
            assert torch.equal(st.index[b, :n], ref.index[b, :n])
    for b in range(inp.q.shape[0]):
        K, V = PY.host_kv(inp, b)
        q = PY.bf16_bits(inp.q[b])
        idx = ref.index[b, : int(ref.count[b])].cpu().numpy()
        for r, st in enumerate(steps):
            want = idx[owner_np[b, idx] == r]
            n = int(st.local_count[b])
            assert n == len(want)
            np.testing.assert_array_equal(st.local_index[b, :n].cpu().numpy(), want)
            if n:
                o = oracle.sparse_decode_attn(q, K, V, want, L, Hq, Hkv, d)
                np.testing.assert_allclose(st.out_local[b].cpu().numpy(), o, rtol=0, atol=ATOL_OUT)
                lse = oracle.log_partition(q, K, want, L, Hq, Hkv, d)
                np.testing.assert_allclose(st.lse_local[b].cpu().numpy(), lse, rtol=0, atol=ATOL_LSE)
        o = oracle.sparse_decode_attn(q, K, V, idx, L, Hq, Hkv, d)
        np.testing.assert_allclose(steps[0].out[b].cpu().numpy(), o, rtol=0, atol=ATOL_OUT)
        lse = oracle.log_partition(q, K, idx, L, Hq, Hkv, d)
        np.testing.assert_allclose(steps[0].lse[b].cpu().numpy(), lse, rtol=0, atol=ATOL_LSE)
        # and the merged output agrees with the unsharded a5 to fp32 rounding
        torch.testing.assert_close(steps[0].out[b], ref.out[b], rtol=0, atol=2e-5)


@pytest.mark.parametrize("cfg,world", [
    (_small("g4_w2"), 2),
    (_small("g4_w3", page=16, seed=52), 3),
    (_small("g7_w8", Hq=14, Hkv=2, seed=53, batch=1), 8),   # Qwen grouping: H_kv = 2 < 8 ranks
    (_small("g1_d64_w4", Hq=2, Hkv=2, d=64, seed=54), 4),
], ids=lambda x: x.name if hasattr(x, "name") else str(x))
def test_token_sharded_step(cfg, world):
    inp = S.generate(cfg, device="cuda")
    steps, owner = _simulate(inp, world)
    _check(inp, steps, owner)


def test_rank_with_no_part_of_the_index():
    """Every token on rank 0 except one summary on rank 1 that is not selected
    for sequence 0 and a chunk of sequence 1: rank 1's part can be empty
    (count 0, its out/lse rows untouched and excluded by the merge)."""
    cfg = _small("empty_part", seed=55)
    inp = S.generate(cfg, device="cuda")
    T = int(inp.seq_len.max().item())
    owner = np.zeros((2, T), np.uint8)
    owner[1, 100:164] = 1
    steps, _ = _simulate(inp, 2, owner_np=owner)
    assert int(steps[1].local_count[0]) == 0
    _check(inp, steps, owner)


def test_merge_of_identical_parts_and_empty_sequences():
    """zoomr_merge_attn alone: R copies of one part merge to that part and lse + ln R;
    a sequence whose every part is empty gets out = 0 and lse = -inf."""
    from paper_2604_10898_b200 import zoomr as Z
    shape = Z.Shape(2, 4, 2, 64, 16)
    g = torch.Generator(device="cuda").manual_seed(5)
    R, B = 3, 2
    one = torch.randn(1, B, 2, 4, 64, device="cuda", generator=g)
    lse1 = torch.randn(1, B, 2, 4, device="cuda", generator=g)
    po, pl = one.expand(R, -1, -1, -1, -1).contiguous(), lse1.expand(R, -1, -1, -1).contiguous()
    cnt = torch.ones(R, B, dtype=torch.int32, device="cuda")
    cnt[:, 1] = 0
    out = torch.full((B, 2, 4, 64), float("nan"), device="cuda")
    lse = torch.full((B, 2, 4), float("nan"), device="cuda")
    Z.merge_attn(shape, po, pl, out, part_count=cnt, lse=lse)
    torch.cuda.synchronize()
    torch.testing.assert_close(out[0], one[0, 0], rtol=1e-6, atol=0)
    torch.testing.assert_close(lse[0], lse1[0, 0] + float(np.log(R)), rtol=0, atol=1e-5)
    assert torch.all(out[1] == 0) and torch.all(torch.isneginf(lse[1]))


def test_qwen_shape_full_size_sharded_equals_unsharded():
    """Full-size Qwen2.5-7B shape (28 layers, 28/4 heads, T = 16K) over 8 simulated
    ranks: the merged output equals the unsharded a5's to fp32 rounding (that
    one is checked against the oracle at full size in test_gpu_large)."""
    cfg = dataclasses.replace(S.CONFIGS["qwen7b16k"], batch=1)
    inp = S.generate(cfg, device="cuda", seed=9)
    steps, owner = _simulate(inp, 8)
    ref = PY.make_step(inp, debug=False, capacity=8192)
    PY.run_full(inp, ref, fused=True)
    n = int(ref.count[0])
    assert torch.equal(steps[3].index[0, :n], ref.index[0, :n])
    assert sum(int(s.local_count[0]) for s in steps) == n
    torch.testing.assert_close(steps[5].out, ref.out, rtol=0, atol=2e-5)
