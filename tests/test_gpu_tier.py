"""GPU tests of the host-memory tier.

The cache lives in pinned host memory; zoomr_tier_fetch keeps the pages of
each step's I_f resident in an HBM hot pool (LRU among the pages the step does
not touch).  Checked over several steps with changing queries (so I_f and the
resident set churn): the output is bit-identical to the same a5 launch on an
all-HBM pool, the residency table equals a plain Python model of the stated
replacement rule, every resident page holds exactly its host page, the number
of copied pages is the model's, and an undersized hot pool reports CAPACITY.

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
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=128, T=2048, n_pairs=24, LR=60, LS=12, sink=4, window=96,
                c=3, top_k=2, page=32, seed=71, batch=2)
    base.update(kw)
    return S.Config(**base)


class LruModel:
    """The replacement rule of zoomr_tier_fetch (include/zoomr.h), written plainly."""

    def __init__(self, hot_pages):
        self.H, self.pt, self.owner, self.stamp, self.step = hot_pages, {}, [-1] * hot_pages, [-1] * hot_pages, 0

    def fetch(self, needed):
        self.step += 1
        missing = []
        for x in sorted(needed):
            if x in self.pt:
                self.stamp[self.pt[x]] = self.step
            else:
                missing.append(x)
        cand = [h for h in range(self.H) if self.stamp[h] < self.step]
        victims = sorted(sorted(cand, key=lambda h: (self.stamp[h], h))[: len(missing)])
        for x, h in zip(missing, victims):
            if self.owner[h] >= 0:
                del self.pt[self.owner[h]]
            self.owner[h], self.pt[x], self.stamp[h] = x, h, self.step
        return len(missing)


def _setup_steps(cfg, hot_pages, hot_page_size=0):
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import StepParams, ZoomrStep
    from paper_2604_10898_b200.tier import HostTierStep
    inp = S.generate(cfg, device="cuda")
    B = inp.q.shape[0]
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    ref = ZoomrStep(shape, B, inp.bounds.shape[1], cfg.T, prm, early_known=False)
    ref.update_mean_keys(kv, seg, ref.all_items(inp.num_summaries))
    host_k, host_v = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
    st = HostTierStep(shape, B, inp.bounds.shape[1], cfg.T, prm, host_k, host_v, inp.page_table, hot_pages,
                      hot_page_size=hot_page_size)
    st.mean_keys.copy_(ref.mean_keys)
    return inp, ref, st, kv, seg


@pytest.mark.parametrize("cfg,hot_pages,ph", [
    (_cfg("b2"), 90, 0),
    (_cfg("g7_p16", Hq=14, Hkv=2, page=16, seed=72), 170, 0),
    (_cfg("hot16_of_32", seed=73), 170, 16),   # hot pages smaller than host pages
    (_cfg("hot8_of_32_g1", Hq=2, Hkv=2, seed=74), 330, 8),
], ids=lambda x: x.name if hasattr(x, "name") else str(x))
def test_tier_steps_equal_hbm_and_follow_lru(cfg, hot_pages, ph):
    inp, ref, st, kv, seg = _setup_steps(cfg, hot_pages, ph)
    B, P = inp.q.shape[0], ph or cfg.page  # P: the hot page size
    R = cfg.page // P
    mp = inp.page_table.shape[1] * R
    model = LruModel(hot_pages)
    g = torch.Generator(device="cuda").manual_seed(cfg.seed)
    fetched = []
    for k in range(8):
        q = (torch.randn(inp.q.shape, device="cuda", generator=g) * (0.5 + 0.25 * k)).bfloat16()
        ref.run(q, kv, seg, fused=True)
        st.run(q, seg)
        torch.cuda.synchronize()
        ref.check_status()
        st.check_status()
        assert torch.equal(st.count, ref.count) and torch.equal(st.index, ref.index)
        assert torch.equal(st.out, ref.out)  # same rows, same tiles, same order: bit-identical
        needed = set()
        for b in range(B):
            idx = ref.index[b, : int(ref.count[b])].cpu().numpy()
            needed |= {b * mp + int(lp) for lp in np.unique(idx // P)}
        nf = model.fetch(needed)
        assert st.fetched_pages() == nf
        fetched.append(nf)
        hpt = st.hot_page_table.cpu().numpy().reshape(-1)
        want = np.full(B * mp, -1)
        for x, h in model.pt.items():
            want[x] = h
        np.testing.assert_array_equal(hpt, want)
        np.testing.assert_array_equal(st.hot_owner.cpu().numpy(), model.owner)
        # resident pages hold exactly their host rows (every layer, K and V)
        pt = inp.page_table.cpu().numpy()
        for x, h in model.pt.items():
            b, lph = divmod(x, mp)
            hp, sub = int(pt[b, lph // R]), lph % R
            for hot, pool in ((st.hot_k, inp.k_pool), (st.hot_v, inp.v_pool)):
                assert torch.equal(hot[:, h], pool[:, hp, :, sub * P:(sub + 1) * P])
    assert fetched[0] > 0 and sum(fetched[1:]) > 0  # cold start, then churn
    # and one step against the oracle, for good measure
    b = 0
    K, V = PY.host_kv(inp, b)
    idx = st.index[b, : int(st.count[b])].cpu().numpy()
    o = oracle.sparse_decode_attn(PY.bf16_bits(q[b]), K, V, idx, cfg.L, cfg.Hq, cfg.Hkv, cfg.d)
    np.testing.assert_allclose(st.out[b].cpu().numpy(), o, rtol=0, atol=2e-3)


def test_tier_repeated_step_fetches_nothing():
    inp, ref, st, kv, seg = _setup_steps(_cfg("same", batch=1), 64)
    st.run(inp.q, seg)
    torch.cuda.synchronize()
    first = st.fetched_pages()
    st.run(inp.q, seg)
    torch.cuda.synchronize()
    st.check_status()
    assert first > 0 and st.fetched_pages() == 0


def test_tier_pool_too_small_reports_capacity():
    from paper_2604_10898_b200 import zoomr as Z
    inp, ref, st, kv, seg = _setup_steps(_cfg("small", batch=1), 4)
    st.run(inp.q, seg)
    torch.cuda.synchronize()
    with pytest.raises(Z.ZoomrError):
        st.check_status()


@pytest.mark.parametrize("ph", [0, 8])
def test_tier_decode_loop_equals_hbm_decode_loop(ph):
    """Algorithm 1's decode loop over the host tier (write-through append, newest rows into the
    hot pool, a1 from the host cache, look-ahead fetch, a5 with early rows once warm) against the
    all-HBM DecodeLoop on the same token stream: segment table, flags, I_f and outputs identical
    at every step (outputs bit-identical from the tier's second step on), eagerly and as graph
    replays."""
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import DecodeLoop, StepParams
    from paper_2604_10898_b200.tier import TierDecodeLoop
    from tests.test_gpu_loop import BEGIN, BOUNDARY, END, token_stream
    B, L, Hq, Hkv, d, P = 2, 2, 8, 2, 64, 16
    n_p, steps, MS = 40, 120, 16
    T_max = n_p + steps
    prm = StepParams(2, 2, 4, 24)
    gen = torch.Generator(device="cpu").manual_seed(9)
    pages = (T_max + P - 1) // P
    k_pool = torch.randn(L, B * pages, Hkv, P, d, generator=gen).bfloat16()
    v_pool = torch.randn(L, B * pages, Hkv, P, d, generator=gen).bfloat16()
    page_table = torch.randperm(B * pages, generator=gen).int().view(B, pages).contiguous().cuda()
    shape = Z.Shape(L, Hq, Hkv, d, P)
    # both loops attend the sink / window rows before their wait (the tier from its second
    # step on, once the look-ahead fetch has made the next token's page resident)
    ref = DecodeLoop(shape, B, MS, T_max, prm, BEGIN, END, BOUNDARY, early_known=True)
    kv_dev = (k_pool.cuda(), v_pool.cuda(), page_table)
    tl = TierDecodeLoop(shape, B, MS, T_max, prm, k_pool.pin_memory(), v_pool.pin_memory(), page_table,
                        hot_pages=B * pages * (P // (ph or P)), begin_id=BEGIN, end_id=END, boundary_ids=BOUNDARY,
                        hot_page_size=ph)
    ref.start(n_p)
    tl.start(n_p)
    rng = np.random.default_rng(9)
    toks = torch.tensor([[t] * B for t in token_stream(rng, steps)], dtype=torch.int32, device="cuda")
    kin = torch.randn(steps, B, L, Hkv, d, device="cuda").bfloat16()
    vin = torch.randn(steps, B, L, Hkv, d, device="cuda").bfloat16()
    qs = torch.randn(steps, B, L, Hq, d, device="cuda").bfloat16()
    half = steps // 2
    for i in range(half):  # eager
        ref.decode_step(kv_dev, kin[i], vin[i], qs[i], toks[i])
        tl.decode_step(kin[i], vin[i], qs[i], toks[i])
        torch.cuda.synchronize()
        ref.check_status()
        tl.check_status()
        assert torch.equal(tl.seq_len, ref.seq_len) and torch.equal(tl.num_summaries, ref.num_summaries)
        assert torch.equal(tl.bounds, ref.bounds) and torch.equal(tl.flags, ref.flags)
        assert torch.equal(tl.count, ref.count) and torch.equal(tl.index, ref.index)
        if i == 0:  # the tier's first step attends index-only (cold hot pool): another split, fp32 rounding
            assert (tl.out - ref.out).abs().max().item() <= 1e-5
        else:
            assert torch.equal(tl.out, ref.out), i
    assert int(tl.num_summaries.min()) >= 1
    # the rest as graph replays (inputs copied into static buffers)
    sk, sv, sq, st_ = kin[0].clone(), vin[0].clone(), qs[0].clone(), toks[0].clone()
    graphs = []
    for loop, args in ((ref, (kv_dev, sk, sv, sq, st_)), (tl, (sk, sv, sq, st_))):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            loop.decode_step(*args)
        graphs.append(g)
    for i in range(half, steps):
        sk.copy_(kin[i]); sv.copy_(vin[i]); sq.copy_(qs[i]); st_.copy_(toks[i])
        graphs[0].replay()
        graphs[1].replay()
        torch.cuda.synchronize()
        ref.check_status()
        tl.check_status()
        assert torch.equal(tl.index, ref.index) and torch.equal(tl.out, ref.out), i
    # the host cache received every appended row (write-through)
    assert torch.equal(tl.host_k.cuda(), kv_dev[0]) and torch.equal(tl.host_v.cuda(), kv_dev[1])


@pytest.mark.parametrize("cfg,lg", [
    (_cfg("lp_small", L=4, batch=1), 1),
    (_cfg("lp_small2", L=4, batch=1, Hq=14, Hkv=2), 2),
    (S.CONFIGS["8b16k"], 1),
], ids=lambda x: getattr(x, "name", str(x)))
def test_layer_pipelined_tier_matches_hbm_and_oracle(cfg, lg):
    """The paper's layer-by-layer host tier (LayerPipelinedTierStep):
    per group of layers, the rows of I_f are gathered host -> HBM slice on a copy
    stream while the previous group attends, two slices resident.  The output
    equals the all-HBM step (fp32 rounding: another stream-K split) and the
    oracle (2e-3), pipelined and serial, eager and as a CUDA-graph replay; the
    slice holds exactly the host rows of I_f."""
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import StepParams
    from paper_2604_10898_b200.tier import LayerPipelinedTierStep
    inp = S.generate(cfg, device="cuda")
    cap = 8192 if cfg.T > 4096 else cfg.T
    ref = PY.make_step(inp, debug=False, capacity=cap)
    PY.run_full(inp, ref, fused=True)
    hk, hv = inp.k_pool.cpu().pin_memory(), inp.v_pool.cpu().pin_memory()
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    st = LayerPipelinedTierStep(shape, inp.bounds.shape[1], cap, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window),
                                hk, hv, inp.page_table, layers_per_slice=lg)
    st.mean_keys.copy_(ref.mean_keys)
    for pipelined in (True, False):
        st.out.zero_()
        st.run(inp.q, seg, pipelined=pipelined)
        torch.cuda.synchronize()
        st.check_status()
        assert torch.equal(st.count, ref.count) and torch.equal(st.flags, ref.flags)
        assert (st.out - ref.out).abs().max().item() <= 1e-5
    # the last group's slice holds the host rows of I_f (layer by layer, every head)
    n = int(st.count[0])
    idx = st.index[0, :n].long()
    g = cfg.L // lg - 1
    sk, _ = st.slices[g % 2]
    for ll in range(lg):
        l = g * lg + ll
        rows = sk[ll].permute(0, 2, 1, 3).reshape(-1, cfg.Hkv, cfg.d)[:n]  # slice row j -> [H_kv][d]
        pages, slots = inp.page_table[0].long()[idx // cfg.page], idx % cfg.page
        host_rows = inp.k_pool[l][pages, :, slots]  # [n][H_kv][d]
        assert torch.equal(rows, host_rows)
    # graph replay (both streams captured), then the oracle on sampled heads
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.run(inp.q, seg)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        st.run(inp.q, seg)
    st.out.zero_()
    gr.replay()
    torch.cuda.synchronize()
    assert (st.out - ref.out).abs().max().item() <= 1e-5
    if cfg.T <= 4096:
        K, V = PY.host_kv(inp, 0)
        o = oracle.sparse_decode_attn(S.bf16_bits(inp.q[0]), K, V, st.index[0, :n].cpu().numpy(), cfg.L, cfg.Hq,
                                      cfg.Hkv, cfg.d)
        assert np.abs(st.out[0].cpu().numpy().astype(np.float64) - o).max() <= PY.ATTN_TOL
