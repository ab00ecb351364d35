"""GPU parity of the H2O comparison policy:
zoomr_h2o_select, a5 with logits, zoomr_h2o_accumulate, over several decode
steps with T growing (so tokens leave the window and get evicted), against the
oracle's O9 (selection taken on the GPU's fp32 scores, so the integer decision
is made in the same precision on both sides), O7/O8 (attention, lse) and the
oracle's per-step weights accumulated in fp64.

Marked `gpu`: run on a B200 with the built libzoomr.so."""
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


def _cfg(name, **kw):
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=128, T=1024, n_pairs=12, LR=50, LS=10, sink=4, window=64,
                c=3, top_k=2, page=32, seed=61, batch=2)
    base.update(kw)
    return S.Config(**base)


def _run(cfg, budget, steps, T0):
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.policies import PolicyStep
    from paper_2604_10898_b200.step import StepParams
    inp = S.generate(cfg, device="cuda")
    B = inp.q.shape[0]
    L, Hq, Hkv, d = cfg.L, cfg.Hq, cfg.Hkv, cfg.d
    shape = Z.Shape(L, Hq, Hkv, d, cfg.page)
    st = PolicyStep("h2o", shape, B, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window),
                    budget=budget, max_positions=cfg.T)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seq_len = torch.full((B,), T0, dtype=torch.int32, device="cuda")
    seg = (inp.bounds, torch.zeros_like(inp.num_summaries), seq_len)
    st.start_h2o(seg)
    g = torch.Generator(device="cuda").manual_seed(cfg.seed)
    host = [PY.host_kv(inp, b) for b in range(B)]
    score_ref = np.zeros((B, cfg.T))
    evicted_any = False
    for k in range(steps):
        q = (torch.randn(B, L, Hq, d, device="cuda", generator=g) * 1.5).bfloat16()
        score_before = st.score.clone()
        prev = [st.prev_index[b, : int(st.prev_count[b])].cpu().numpy() for b in range(B)]
        st.run(q, kv, seg)
        torch.cuda.synchronize()
        st.check_status()
        for b in range(B):
            T = int(seq_len[b])
            idx = st.index[b, : int(st.count[b])].cpu().numpy()
            # the selection, in the GPU's precision (its fp32 scores, exactly representable in fp64)
            want = oracle.h2o_select(prev[b], score_before[b, :T].double().cpu().numpy(), T, cfg.sink, cfg.window,
                                     budget)
            np.testing.assert_array_equal(idx, want)
            evicted_any |= len(set(prev[b]) - set(idx)) > 0
            K, V = host[b]
            qb = PY.bf16_bits(q[b])
            o = oracle.sparse_decode_attn(qb, K, V, idx, L, Hq, Hkv, d)
            np.testing.assert_allclose(st.out[b].cpu().numpy(), o, rtol=0, atol=2e-3)
            lse = oracle.log_partition(qb, K, idx, L, Hq, Hkv, d)
            np.testing.assert_allclose(st.lse[b].cpu().numpy(), lse, rtol=0, atol=1e-4)
            score_ref[b, idx] += oracle.h2o_weights(qb, K, idx, L, Hq, Hkv, d)
            np.testing.assert_allclose(st.score[b].cpu().numpy(), score_ref[b], rtol=0, atol=1e-5)
            # the set handed to the next step
            assert int(st.prev_count[b]) == len(idx)
            assert np.array_equal(st.prev_index[b, : len(idx)].cpu().numpy(), idx)
        seq_len += 1  # the next token (its K/V rows already exist in the synthetic cache)
    return evicted_any


@pytest.mark.parametrize("cfg,budget", [
    (_cfg("g4"), 160),
    (_cfg("g7_p16", Hq=14, Hkv=2, page=16, seed=62, batch=1), 100),
    (_cfg("g1_d64", Hq=2, Hkv=2, d=64, seed=63), 90),
], ids=lambda x: x.name if hasattr(x, "name") else str(x))
def test_h2o_steps_match_oracle(cfg, budget):
    assert _run(cfg, budget, steps=12, T0=cfg.T - 20)


def test_h2o_budget_at_least_T_is_full_attention():
    """with budget >= T nothing is evicted and H2O is full attention."""
    cfg = _cfg("full", T=512, batch=1)
    assert not _run(cfg, budget=600, steps=3, T0=400)


def test_h2o_budget_only_sink_and_window():
    """budget <= |sink u window|: every older token is evicted on the first step."""
    cfg = _cfg("tight", seed=64, batch=1)
    assert _run(cfg, budget=cfg.sink + cfg.window, steps=3, T0=cfg.T - 10)
