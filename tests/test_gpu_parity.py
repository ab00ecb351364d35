"""GPU parity: libzoomr (through the C-ABI) vs the fp64 CPU oracle, element by element.

Marked `gpu`: run on a B200 with the built libzoomr.so.
"""
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


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("seed", [1, 11, 12])
def test_tiny_end_to_end(seed, fused):
    inp = S.generate(S.CONFIGS["tiny"], device="cuda", seed=seed)
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    PY.check_sequence(inp, st, 0, rep)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("query", ["planted", "diffuse"])
def test_tiny_batched_variants(query, fused):
    import dataclasses
    cfg = dataclasses.replace(S.CONFIGS["tiny"], batch=5)
    inp = S.generate(cfg, device="cuda", seed=21, query_mode=query)
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    for b in range(5):
        PY.check_sequence(inp, st, b, rep)


@pytest.mark.parametrize("fused", [False, True])
def test_8b16k_end_to_end(fused):
    inp = S.generate(S.CONFIGS["8b16k"], device="cuda")
    st = PY.make_step(inp, capacity=8192)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    PY.check_sequence(inp, st, 0, rep)
    print(rep)


@pytest.mark.parametrize("cfg_name,batch", [("tiny", 3), ("8b16k", 1)])
def test_fused_equals_separate_calls(cfg_name, batch):
    """zoomr_select_fused and the four separate calls give bit-identical results."""
    import dataclasses
    cfg = dataclasses.replace(S.CONFIGS[cfg_name], batch=batch)
    inp = S.generate(cfg, device="cuda", seed=5)
    a, b = PY.make_step(inp), PY.make_step(inp)
    PY.run_full(inp, a, fused=False)
    PY.run_full(inp, b, fused=True)
    for name in ("mean_keys", "partial", "flags", "index", "count", "alpha", "topk", "agreeability"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert torch.equal(a.out, b.out)


def test_fused_repeated_steps_reset_workspace():
    """Tickets / arrival counters reset themselves: many graph replays stay correct."""
    inp = S.generate(S.CONFIGS["tiny"], device="cuda", seed=7)
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=True)
    ref_out, ref_idx = st.out.clone(), st.index.clone()
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    g = st.capture(inp.q, kv, seg, update_selection=True, close_items=None, fused=True)
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    st.check_status()
    assert torch.equal(st.out, ref_out) and torch.equal(st.index, ref_idx)


def _integerize_and_duplicate(inp, dup_pairs):
    """Parity-only variant: integer-valued keys/queries and duplicated
    summaries, so alphas tie EXACTLY on both sides and only the fixed tie-break
    (alpha desc, index asc; votes desc, A desc, index asc) decides."""
    cfg = inp.cfg
    P = cfg.page
    inp.k_pool.copy_(torch.round(inp.k_pool.float() * 2).to(torch.bfloat16))
    inp.q.copy_(torch.round(inp.q.float() * 8).to(torch.bfloat16))
    for b in range(inp.q.shape[0]):
        pt = inp.page_table[b].long()
        bd = inp.bounds[b].cpu().tolist()
        for (i, j) in dup_pairs:
            si, sj = bd[i][2], bd[j][2]
            n = bd[i][3] - bd[i][2]
            assert bd[j][3] - bd[j][2] == n
            for t in range(n):
                src, dst = si + t, sj + t
                inp.k_pool[:, pt[dst // P], :, dst % P] = inp.k_pool[:, pt[src // P], :, src % P]
    return inp


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("seed", [3, 4, 5, 6])
def test_exact_ties_follow_the_fixed_tie_break(seed, fused):
    import dataclasses
    cfg = dataclasses.replace(S.CONFIGS["tiny"], batch=2, c=3, top_k=3)
    inp = _integerize_and_duplicate(S.generate(cfg, device="cuda", seed=seed), [(1, 5), (2, 6), (0, 7)])
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    for b in range(2):
        PY.check_sequence(inp, st, b, rep)
    assert rep.get("excused_voters", 0) == 0 and rep.get("excused_cuts", 0) == 0


@pytest.mark.parametrize("fused", [False, True])
def test_many_summaries_histogram_topc(fused):
    """N_t above the block size: the vote-histogram threshold path of a3 (and a wide a4)."""
    cfg = S.Config("many", L=2, Hq=8, Hkv=2, d=32, T=8192, n_pairs=600, LR=8, LS=4, sink=16, window=64,
                   c=12, top_k=4, page=32, seed=9, off_target=0.6)
    inp = S.generate(cfg, device="cuda")
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    PY.check_sequence(inp, st, 0, rep)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("c,small_group", [(60, True), (300, False)])
def test_large_tie_group_at_the_topc_cut(c, small_group, fused):
    """N_t = 1600 with diffuse queries (V = 128 voters, k = 8): most voted summaries
    hold one or two votes, so the threshold bin of a3 holds a large tie group,
    ranked by (v desc, A desc, i asc).  c = 60 puts the cut in a group of a few
    hundred members; c = 300 puts it in the v = 1 group (> 512 members)."""
    cfg = S.Config("ties1600", L=4, Hq=32, Hkv=8, d=32, T=20480, n_pairs=1600, LR=8, LS=4, sink=16,
                   window=64, c=c, top_k=8, page=32, seed=21, query="diffuse", off_target=1.0)
    inp = S.generate(cfg, device="cuda")
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    PY.check_sequence(inp, st, 0, {})
    # the case asked for: size of the tie group at the cut (votes from the oracle-checked partial)
    v = st.partial[0, 0, :cfg.n_pairs].cpu()
    vs = torch.sort(v[v > 0], descending=True).values
    cut_v = int(vs[min(c, len(vs)) - 1])
    m = int((v == cut_v).sum())
    assert len(vs) > c and (m <= 512) == small_group, (len(vs), cut_v, m)


@pytest.mark.parametrize("fused", [False, True])
def test_degenerate_cases(fused):
    """c = 0 (SumR-like keep-all-voted), k > N_t, c > |I_all|, window >= T, sink > T."""
    import dataclasses
    base = S.CONFIGS["tiny"]
    for cfg in (dataclasses.replace(base, c=0), dataclasses.replace(base, top_k=20, c=30),
                dataclasses.replace(base, window=300, sink=300), dataclasses.replace(base, n_pairs=1)):
        inp = S.generate(cfg, device="cuda", seed=13)
        st = PY.make_step(inp)
        PY.run_full(inp, st, fused=fused)
        PY.check_sequence(inp, st, 0, {})


@pytest.mark.parametrize("variant", ["tiny_b5_jitter", "tiny_window_ge_T", "tiny_c0", "tiny_b320", "tiny_b320_nosum",
                                     "8b16k"])
def test_early_known_rows_equal_index_only(variant):
    """a5 with seq_len/sink/window (I_p and I_w attended before the wait, merged
    with the rest of I_f afterwards) vs a5 reading every row from the index:
    the same softmax over the same rows, only the merge order differs."""
    import dataclasses
    base = S.CONFIGS["tiny"]
    cfg = {"tiny_b5_jitter": dataclasses.replace(base, batch=5, jitter=True),
           "tiny_window_ge_T": dataclasses.replace(base, batch=2, window=300, sink=7),
           "tiny_c0": dataclasses.replace(base, c=0, sink=0),
           # more segments (640) than math warps: one warp's range spans >= 3 segments per phase
           "tiny_b320": dataclasses.replace(base, batch=320, window=96),
           # no summaries and sink + window = one tile: I_f is phase A only (no phase-B
           # parts), with warps holding two phase-A segments
           "tiny_b320_nosum": dataclasses.replace(base, batch=320, n_pairs=0, sink=4, window=28),
           "8b16k": S.CONFIGS["8b16k"]}[variant]
    inp = S.generate(cfg, device="cuda", seed=31)
    cap = 8192 if variant == "8b16k" else None
    a, b = PY.make_step(inp, capacity=cap), PY.make_step(inp, capacity=cap)
    b.early_known = False
    PY.run_full(inp, a, fused=True)
    PY.run_full(inp, b, fused=True)
    assert torch.equal(a.index, b.index) and torch.equal(a.count, b.count)
    assert (a.out - b.out).abs().max().item() <= 1e-5
    rep = {}
    B = inp.q.shape[0]
    for s in sorted({min(x, B - 1) for x in (0, 1, 2, B // 2, B - 1)}):
        PY.check_sequence(inp, a, s, rep)
