"""GPU parity of the less common paths through the C-ABI: other head dims and
group sizes, the page-resolved rows (index_phys), a5 launched alone and
back to back inside a CUDA graph, and the device status codes.

Marked `gpu`: run on a B200 with the built libzoomr.so."""
import dataclasses

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


def _small(name, **kw):
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=64, T=2048, n_pairs=24, LR=60, LS=12, sink=4, window=96,
                c=3, top_k=2, page=32, seed=41)
    base.update(kw)
    return S.Config(**base)


@pytest.mark.parametrize("cfg", [
    _small("d64_g4"),                                  # d = 64: one swizzled 64-column region, TMA boxes
    _small("d128_g1", d=128, Hq=2, Hkv=2),             # G = 1
    _small("d128_g8", d=128, Hq=16, Hkv=2),            # G = 8 (hi and lo in separate MMA n-tiles)
    _small("d32_g2", d=32, Hq=4, Hkv=2, batch=3),      # d = 32: rows by cp.async only
    _small("d128_g7", d=128, Hq=14, Hkv=2),            # G = 7 (Qwen2.5-7B grouping; MMA column 7 padded)
], ids=lambda c: c.name)
@pytest.mark.parametrize("fused", [False, True])
def test_head_dims_and_groups(cfg, fused):
    inp = S.generate(cfg, device="cuda")
    st = PY.make_step(inp)
    PY.run_full(inp, st, fused=fused)
    rep = {}
    for b in range(inp.q.shape[0]):
        PY.check_sequence(inp, st, b, rep)


@pytest.mark.parametrize("cfg_name", ["tiny", "8b16k"])
def test_page_resolved_rows_equal(cfg_name):
    """The fused select's index_phys (page-resolved rows) drives a5 to the same
    output as the page-table lookups, with and without the early rows."""
    cfg = dataclasses.replace(S.CONFIGS[cfg_name], batch=2 if cfg_name == "tiny" else 1)
    inp = S.generate(cfg, device="cuda", seed=8)
    cap = 8192 if cfg_name == "8b16k" else None
    a, b = PY.make_step(inp, capacity=cap), PY.make_step(inp, capacity=cap)
    b.use_phys = True
    for early in (True, False):
        a.early_known = b.early_known = early
        PY.run_full(inp, a, fused=True)
        PY.run_full(inp, b, fused=True)
        assert torch.equal(a.index, b.index) and torch.equal(a.count, b.count)
        assert torch.equal(a.out, b.out), early
    rep = {}
    PY.check_sequence(inp, b, 0, rep)


def test_attention_alone_back_to_back_in_a_graph():
    """a5 launched repeatedly in one CUDA graph (programmatic launch edges between
    consecutive a5 nodes): the self-resetting workspace keeps every launch exact."""
    inp = S.generate(S.CONFIGS["8b16k"], device="cuda", seed=3)
    st = PY.make_step(inp, capacity=8192)
    PY.run_full(inp, st, fused=True)
    ref = st.out.clone()
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    for early in (False, True):
        st.early_known = early
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(8):
                st.attend(inp.q, kv, inp.seq_len)
        for _ in range(3):
            st.out.zero_()
            g.replay()
        torch.cuda.synchronize()
        st.check_status()
        assert (st.out - ref).abs().max().item() <= 1e-5, early


def test_device_status_codes():
    """Data-dependent errors are recorded in the device status word (first wins):
    I_f longer than the index capacity -> CAPACITY (list truncated to the capacity)."""
    from paper_2604_10898_b200 import zoomr as Z
    inp = S.generate(S.CONFIGS["tiny"], device="cuda", seed=2)
    st = PY.make_step(inp, capacity=40)  # |I_f| of tiny is 82-106
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    st.run(inp.q, kv, seg, fused=True)
    torch.cuda.synchronize()
    assert int(st.status.item()) == Z.ERR_CAPACITY
    assert int(st.count[0]) == 40
    # an empty summary segment (s1 <= s0) -> EMPTY_SEGMENT
    st2 = PY.make_step(inp)
    bad = inp.bounds.clone()
    bad[0, 3, 3] = bad[0, 3, 2]
    st2.update_mean_keys(kv, (bad, inp.num_summaries, inp.seq_len), torch.tensor([[0, 3]], dtype=torch.int32,
                                                                                 device="cuda"))
    torch.cuda.synchronize()
    assert int(st2.status.item()) == Z.ERR_EMPTY_SEGMENT


@pytest.mark.parametrize("policy", ["streamingllm", "sumr"])
@pytest.mark.parametrize("cfg_name", ["tiny", "8b16k"])
def test_comparison_policies(policy, cfg_name):
    """StreamingLLM at a matched budget and SumR on the same kernels (a4 with fixed
    flags + a5) vs the oracle's index build and attention on the same flags."""
    import numpy as np
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.policies import PolicyStep
    from paper_2604_10898_b200.step import StepParams
    cfg = S.CONFIGS[cfg_name]
    inp = S.generate(cfg, device="cuda", seed=4)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    budget = 2 * cfg.window
    st = PolicyStep(policy, shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window),
                    budget=budget)
    st.prepare(inp.num_summaries)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.run(inp.q, kv, seg)
    torch.cuda.synchronize()
    st.check_status()
    sg = PY.seg_host(inp, 0)
    flags = np.ones(len(sg), np.uint8) if policy == "sumr" else np.zeros(len(sg), np.uint8)
    idx = oracle.build_index(sg, flags, cfg.T, st.params.sink, st.params.window)
    cnt = int(st.count[0])
    assert cnt == len(idx) and np.array_equal(st.index[0, :cnt].cpu().numpy(), idx)
    if policy == "streamingllm":
        assert cnt == min(budget, cfg.T)
    layers, heads = ([0], [0, cfg.Hq - 1]) if cfg_name == "8b16k" else (range(cfg.L), range(cfg.Hq))
    q = PY.bf16_bits(inp.q[0])
    out = st.out[0].cpu().numpy().astype(np.float64)
    G = cfg.Hq // cfg.Hkv
    for l in layers:
        Kr = PY.gather_tokens(inp, 0, idx, "k", layers=[l])
        Vr = PY.gather_tokens(inp, 0, idx, "v", layers=[l])
        for h in heads:
            o = oracle.attend_one(q[l, h], np.ascontiguousarray(Kr[:, 0, h // G]), np.ascontiguousarray(Vr[:, 0, h // G]),
                                  np.arange(len(idx)))
            assert np.abs(out[l, h] - o).max() <= 2e-3


@pytest.mark.parametrize("cfg", [
    _small("chain_b3", d=128, batch=3),
    _small("chain_g7", d=128, Hq=14, Hkv=2),
    dataclasses.replace(S.CONFIGS["8b16k"], seed=12),
], ids=lambda c: c.name)
def test_chained_steps_in_one_graph(cfg):
    """zoomr_select_fused_chained / zoomr_sparse_decode_attn_chained (ABI 8): several
    steps over independent input sets captured back to back in ONE graph, each
    select running a1/a2 while the previous step's a5 finishes.  Every step's
    outputs are bit-identical to the same step run alone (unchained), and the
    small cases are checked against the oracle."""
    from paper_2604_10898_b200 import zoomr as Z
    R = 3
    sets = []
    for r in range(R):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 5 * r)
        cap = 8192 if cfg.T > 4096 else None
        ref, st = PY.make_step(inp, capacity=cap), PY.make_step(inp, capacity=cap)
        st.chained = True
        PY.run_full(inp, ref, fused=True)  # unchained, eager
        kv = (inp.k_pool, inp.v_pool, inp.page_table)
        seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                              dtype=torch.int32, device="cuda")
        sets.append((inp, ref, st, kv, seg, newest))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (kernel attributes) outside the capture
        for inp, ref, st, kv, seg, newest in sets:
            st.run(inp.q, kv, seg, close_items=newest)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(3):
            for inp, ref, st, kv, seg, newest in sets:
                st.run(inp.q, kv, seg, close_items=newest)
    for _, _, st, *_ in sets:
        st.out.zero_()
        st.index.zero_()
        st.count.zero_()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    for inp, ref, st, kv, seg, newest in sets:
        st.check_status()
        ref.check_status()
        assert torch.equal(st.count, ref.count)
        for b in range(inp.q.shape[0]):
            n = int(st.count[b])
            assert torch.equal(st.index[b, :n], ref.index[b, :n])
        assert torch.equal(st.flags, ref.flags)
        assert torch.equal(st.out, ref.out)
        if cfg.T <= 4096:
            rep = {}
            for b in range(inp.q.shape[0]):
                PY.check_sequence(inp, st, b, rep)
    # a plain a5 enqueued right behind a chained one on the same workspace
    # attends index-only (the early rows would race the chained launch's merges)
    inp, ref, st, kv, seg, newest = sets[0]
    for _ in range(3):
        st.run(inp.q, kv, seg, close_items=newest)
        st.attend(inp.q, kv, inp.seq_len)
    torch.cuda.synchronize()
    st.check_status()
    assert (st.out - ref.out).abs().max().item() <= 1e-5
    assert "zoomr_select_fused_chained" in Z.EXPORTS


@pytest.mark.parametrize("cfg", [
    _small("chain1_b3", d=128, batch=3),
    dataclasses.replace(S.stress_config(64, 8), name="chain1_stress_LR64", seed=13),
    dataclasses.replace(S.CONFIGS["8b16k"], seed=14, batch=2),
], ids=lambda c: c.name)
def test_chained_same_object_back_to_back(cfg):
    """ONE ZoomrStep(chained=True) run N times back to back inside one graph (the
    serving-loop case: every select and a5 share one selection workspace and one
    attention workspace), the queries alternating between two sets so that
    consecutive steps select different summaries.  Each select(t+1) may start
    only after select(t) completed (a5(t) triggers after its wait): a vote or
    ticket of step t+1 landing while step t still aggregates would leave the
    self-resetting workspaces dirty and the outputs wrong.  Checked: the last
    step's outputs equal the same step run alone (unchained), and both
    workspaces are all-zero after every replay -- at the configs[4] point with
    the longest select tail (L_R = 64, N_t = 1631) and at batch > 1."""
    inp = S.generate(cfg, device="cuda")
    cap = 40000 if cfg.T > 4096 else None
    g2 = torch.Generator(device="cuda").manual_seed(cfg.seed + 99)
    q_b = (0.25 * torch.randn(inp.q.shape, device="cuda", generator=g2)).bfloat16()  # diffuse: other summaries
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    refs = {}
    for name, q in (("a", inp.q), ("b", q_b)):
        ref = PY.make_step(inp, debug=False, capacity=cap)
        ref.update_mean_keys(kv, seg, ref.all_items(inp.num_summaries))
        ref.run(q, kv, seg, close_items=newest)
        torch.cuda.synchronize()
        ref.check_status()
        refs[name] = ref
    st = PY.make_step(inp, debug=False, capacity=cap)
    st.chained = True
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.run(inp.q, kv, seg, close_items=newest)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    N = 8
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(N):
            st.run(inp.q if i % 2 == 0 else q_b, kv, seg, close_items=newest)
    last = refs["b"]  # N even: the last step used q_b
    for _ in range(4):
        st.out.zero_()
        g.replay()
        torch.cuda.synchronize()
        st.check_status()
        assert torch.equal(st.count, last.count)
        for b in range(inp.q.shape[0]):
            n = int(st.count[b])
            assert torch.equal(st.index[b, :n], last.index[b, :n])
        assert torch.equal(st.flags, last.flags)
        assert torch.equal(st.partial, last.partial)
        assert torch.equal(st.out, last.out)
        assert int(st.sel_workspace.count_nonzero()) == 0, "selection workspace left dirty"
        ws_cnt_bytes = inp.q.shape[0] * cfg.L * cfg.Hkv * 4
        assert int(st.workspace[-ws_cnt_bytes:].count_nonzero()) == 0, "a5 arrival counters left dirty"


def test_a5_behind_chained_a5_same_workspace():
    """The old caller rule (zoomr.h ABI 8: "the kernel following a chained a5 must
    not be a PDL-launched a5 using the same workspace") deliberately broken: a
    chained a5 followed directly by an a5 WITH the early rows (which write the
    workspace before their wait), on one workspace, alternating queries, 10
    times in one graph.  The library detects the order and runs the second a5
    index-only; every output equals the a5 run alone."""
    from paper_2604_10898_b200 import zoomr as Z
    cfg = dataclasses.replace(S.CONFIGS["8b16k"], seed=15)
    inp = S.generate(cfg, device="cuda")
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st = PY.make_step(inp, debug=False, capacity=8192)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    st.run(inp.q, kv, seg)
    g2 = torch.Generator(device="cuda").manual_seed(7)
    q_b = (0.25 * torch.randn(inp.q.shape, device="cuda", generator=g2)).bfloat16()
    outs = {}
    for name, q in (("a", inp.q), ("b", q_b)):
        o = torch.zeros_like(st.out)
        Z.sparse_decode_attn(st.shape, q, *kv, st.index, st.count, o, st.workspace, dev_status=st.status)
        outs[name] = o
    torch.cuda.synchronize()
    oa, ob = torch.zeros_like(st.out), torch.zeros_like(st.out)
    args = dict(dev_status=st.status)
    Z.sparse_decode_attn(st.shape, inp.q, *kv, st.index, st.count, oa, st.workspace, chained=True, **args)
    Z.sparse_decode_attn(st.shape, q_b, *kv, st.index, st.count, ob, st.workspace, seq_len=inp.seq_len,
                         sink=cfg.sink, window=cfg.window, **args)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            Z.sparse_decode_attn(st.shape, inp.q, *kv, st.index, st.count, oa, st.workspace, chained=True, **args)
            Z.sparse_decode_attn(st.shape, q_b, *kv, st.index, st.count, ob, st.workspace, seq_len=inp.seq_len,
                                 sink=cfg.sink, window=cfg.window, **args)
    for _ in range(3):
        oa.zero_()
        ob.zero_()
        g.replay()
        torch.cuda.synchronize()
        st.check_status()
        assert torch.equal(oa, outs["a"])
        assert torch.equal(ob, outs["b"])


@pytest.mark.parametrize("ranges", [[(0, 1), (1, 0)], [(0, 3), (3, 2), (5, 3)]], ids=["2_ranges", "3_ranges"])
def test_a5_layer_ranges(ranges):
    """a5 with layer_begin / layer_count: attending the layers in
    pieces gives the output of one all-layer launch (to fp32 rounding: the
    stream-K split, hence the summation order, depends on the launch's work),
    and a launch leaves the out rows of the other layers untouched."""
    from paper_2604_10898_b200 import zoomr as Z
    cfg = _small("layers", L=8, d=128, batch=2, Hq=8, Hkv=2)
    inp = S.generate(cfg, device="cuda")
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    st = PY.make_step(inp, debug=False)
    PY.run_full(inp, st, fused=True)
    full = st.out.clone()
    out = torch.full_like(full, 7.0)
    for lb, lc in ranges:
        Z.sparse_decode_attn(st.shape, inp.q, *kv, st.index, st.count, out, st.workspace, dev_status=st.status,
                             layer_begin=lb, layer_count=lc)
        torch.cuda.synchronize()
        hi = cfg.L if lc == 0 else lb + lc
        assert (out[:, lb:hi] - full[:, lb:hi]).abs().max().item() <= 1e-5
        assert bool((out[:, hi:] == 7.0).all())
    lse = torch.zeros(inp.q.shape[0], cfg.L, cfg.Hq, device="cuda")
    o2 = torch.zeros_like(full)
    Z.sparse_decode_attn_lse(st.shape, inp.q, *kv, st.index, st.count, o2, lse, st.workspace, layer_begin=2,
                             layer_count=3)
    torch.cuda.synchronize()
    assert (o2[:, 2:5] - full[:, 2:5]).abs().max().item() <= 1e-5
    assert bool((lse[:, :2] == 0).all()) and bool((lse[:, 5:] == 0).all()) and bool((lse[:, 2:5] != 0).all())
    with pytest.raises(Z.ZoomrError):
        Z.sparse_decode_attn(st.shape, inp.q, *kv, st.index, st.count, out, st.workspace, layer_begin=7,
                             layer_count=2)


@pytest.mark.parametrize("cfg", [
    _small("ft_b3", d=128, batch=3, jitter=True),
    _small("ft_g7", d=128, Hq=14, Hkv=2),
    dataclasses.replace(S.stress_config(64, 8), name="ft_stress_LR64", seed=16),
], ids=lambda c: c.name)
def test_select_front_tail_equal_separate_calls(cfg):
    """zoomr_select_front + zoomr_select_tail (ABI 9, the KV-head-sharded step's
    select around its all-reduce) == zoomr_score + zoomr_select_topc +
    zoomr_build_index, bit for bit (partial, flags, AG, I_f), with and without the
    front's a1 of the newest summaries, and with update[b] = 0 holding flags."""
    from paper_2604_10898_b200 import zoomr as Z
    inp = S.generate(cfg, device="cuda")
    cap = 40000 if cfg.T > 4096 else None
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    ref = PY.make_step(inp, capacity=cap)
    PY.run_full(inp, ref, fused=False)
    st = PY.make_step(inp, capacity=cap)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    for b, i in newest.tolist():
        st.mean_keys[b, :, :, i] = float("nan")  # the front's a1 must recompute them
    for rep in range(2):
        st.partial.fill_(-1)
        Z.select_front(st.shape, inp.q, *kv, *seg, newest if rep == 0 else None, st.mean_keys, cfg.top_k,
                       st.partial, st.sel_workspace, alpha_out=st.alpha, topk_out=st.topk, dev_status=st.status)
        Z.select_tail(st.shape, *seg, st.partial, cfg.c, cfg.sink, cfg.window, st.flags, st.index, st.count,
                      agreeability=st.agreeability, dev_status=st.status)
        torch.cuda.synchronize()
        st.check_status()
        assert torch.equal(st.partial, ref.partial)
        assert torch.equal(st.flags, ref.flags) and torch.equal(st.count, ref.count)
        assert torch.equal(st.agreeability, ref.agreeability)
        for b in range(inp.q.shape[0]):
            n = int(st.count[b])
            assert torch.equal(st.index[b, :n], ref.index[b, :n])
        assert int(st.sel_workspace.count_nonzero()) == 0
    # update[b] = 0: the front leaves partial[b] alone, the tail keeps flags[b] and rebuilds I_f
    if inp.q.shape[0] > 1:
        upd = torch.ones(inp.q.shape[0], dtype=torch.uint8, device="cuda")
        upd[0] = 0
        held = st.flags.clone()
        st.flags[1:].zero_()
        st.partial[0].fill_(-7)
        q2 = (0.25 * torch.randn(inp.q.shape, device="cuda")).bfloat16()
        Z.select_front(st.shape, q2, *kv, *seg, None, st.mean_keys, cfg.top_k, st.partial, st.sel_workspace,
                       dev_status=st.status, update=upd)
        Z.select_tail(st.shape, *seg, st.partial, cfg.c, cfg.sink, cfg.window, st.flags, st.index, st.count,
                      dev_status=st.status, update=upd)
        torch.cuda.synchronize()
        st.check_status()
        assert bool((st.partial[0] == -7).all())
        assert torch.equal(st.flags[0], held[0])
        n0 = int(st.count[0])
        assert torch.equal(st.index[0, :n0], ref.index[0, :n0])
