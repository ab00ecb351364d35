"""The device decode loop against the oracle's Algorithm-1
loop (oracle/loop.py), step by step on a scripted token stream with summary
delimiters and semantic boundaries: segment table, N_t, flags, I_f exact;
attention within the 2e-3 rule; votes exact at every selection update.
Eager launches and CUDA-graph replays of the same step.

Marked `gpu`: run on a B200 with the built libzoomr.so."""
import numpy as np
import pytest
import torch

import oracle
from oracle.loop import OracleLoop

pytestmark = pytest.mark.gpu

BEGIN, END, DOT = 1000, 1001, 200
BOUNDARY = (DOT, 201, 202)


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    from paper_2604_10898_b200 import _build
    _build.build()


def token_stream(rng, n):
    """Regular text with a boundary every ~7 tokens, a summary (begin, 3-6 tokens, end) every ~20."""
    toks, since_sum, in_sum, body = [], 0, False, 0
    while len(toks) < n:
        if in_sum:
            if body <= 0:
                toks.append(END)
                in_sum, since_sum = False, 0
            else:
                toks.append(DOT if rng.random() < 0.2 else int(rng.integers(3, 100)))
                body -= 1
        elif since_sum >= 14 and rng.random() < 0.25:
            toks.append(BEGIN)
            in_sum, body = True, int(rng.integers(3, 7))
        else:
            toks.append(DOT if rng.random() < 0.15 else int(rng.integers(3, 100)))
            since_sum += 1
    return toks


def bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("graph,chained,fused_a0", [(False, True, True), (True, True, True), (True, False, False),
                                                    (False, False, True)])
def test_decode_loop_matches_oracle_loop(graph, chained, fused_a0):
    """chained + fused_a0 (the default): zoomr_append_track launched with PDL behind the
    chained a5 of the previous step; otherwise plain launches / separate append + track."""
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import DecodeLoop, StepParams
    B, L, Hq, Hkv, d, P = 2, 2, 8, 2, 64, 16
    n_p, steps, MS = 24, 160, 16
    T_max = n_p + steps
    top_k, c, sink, window = 2, 2, 4, 24
    rng = np.random.default_rng(5)
    gen = torch.Generator(device="cpu").manual_seed(5)
    pages = (T_max + P - 1) // P
    k_pool = torch.zeros(L, B * pages, Hkv, P, d, dtype=torch.bfloat16)
    v_pool = torch.zeros_like(k_pool)
    # distinct physical pages per sequence
    perm = torch.randperm(B * pages, generator=gen).int()
    page_table = perm.view(B, pages).contiguous()
    prompt_k = torch.randn(B, n_p, L, Hkv, d, generator=gen).bfloat16()
    prompt_v = torch.randn(B, n_p, L, Hkv, d, generator=gen).bfloat16()
    for b in range(B):
        for t in range(n_p):
            pg, sl = int(page_table[b, t // P]), t % P
            k_pool[:, pg, :, sl] = prompt_k[b, t]
            v_pool[:, pg, :, sl] = prompt_v[b, t]
    kv = (k_pool.cuda(), v_pool.cuda(), page_table.cuda())
    shape = Z.Shape(L, Hq, Hkv, d, P)
    loop = DecodeLoop(shape, B, MS, T_max, StepParams(top_k, c, sink, window), BEGIN, END, BOUNDARY,
                      chained=chained, fused_a0=fused_a0)
    loop.start(n_p)
    refs = [OracleLoop(L, Hq, Hkv, d, top_k, c, sink, window, BEGIN, END, BOUNDARY,
                       list(bits(prompt_k[b])), list(bits(prompt_v[b]))) for b in range(B)]
    streams = [token_stream(np.random.default_rng(10 + b), steps) for b in range(B)]
    k_in = torch.zeros(B, L, Hkv, d, dtype=torch.bfloat16, device="cuda")
    v_in, q_in = torch.zeros_like(k_in), torch.zeros(B, L, Hq, d, dtype=torch.bfloat16, device="cuda")
    tok_in = torch.zeros(B, dtype=torch.int32, device="cuda")
    g = None
    n_updates = 0
    for t in range(steps):
        k_new = torch.randn(B, L, Hkv, d, generator=gen).bfloat16()
        v_new = torch.randn(B, L, Hkv, d, generator=gen).bfloat16()
        q = (0.25 * torch.randn(B, L, Hq, d, generator=gen)).bfloat16()
        toks = torch.tensor([streams[b][t] for b in range(B)], dtype=torch.int32)
        k_in.copy_(k_new)
        v_in.copy_(v_new)
        q_in.copy_(q)
        tok_in.copy_(toks)
        if graph:
            if g is None:  # capture the whole step once; replays read the input buffers
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    loop.decode_step(kv, k_in, v_in, q_in, tok_in)
            g.replay()
        else:
            loop.decode_step(kv, k_in, v_in, q_in, tok_in)
        torch.cuda.synchronize()
        loop.check_status()
        for b in range(B):
            r = refs[b].step(bits(k_new[b]), bits(v_new[b]), bits(q[b]), int(toks[b]))
            n = r["segs"].shape[0]
            assert int(loop.seq_len[b]) == refs[b].T
            assert int(loop.num_summaries[b]) == n, (t, b)
            assert np.array_equal(loop.bounds[b, :n].cpu().numpy(), r["segs"]), (t, b)
            assert np.array_equal(loop.flags[b, :n].cpu().numpy(), r["flags"]), (t, b)
            cnt = int(loop.count[b])
            assert cnt == len(r["index"]) and np.array_equal(loop.index[b, :cnt].cpu().numpy(), r["index"]), (t, b)
            err = np.abs(loop.out[b].cpu().numpy().astype(np.float64) - r["out"]).max()
            assert err <= 2e-3, (t, b, err)
            if r["update"] and n:
                n_updates += 1
                assert np.array_equal(loop.partial[b, 0, :n].cpu().numpy(), r["votes"]), (t, b)
    assert n_updates >= 10
    assert min(int(x) for x in loop.num_summaries.cpu()) >= 4


def test_chained_loop_graph_equals_plain_loop():
    """Many decode steps back to back in ONE graph (append_track of step t+1 overlapping the
    end of step t's chained a5): every output of every step bit-identical to the plain
    5-launch loop, and the final segment table / T equal."""
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.step import DecodeLoop, StepParams
    B, L, Hq, Hkv, d, P = 3, 2, 8, 2, 128, 32
    n_p, steps, MS = 300, 96, 16
    T_max = n_p + steps
    gen = torch.Generator(device="cpu").manual_seed(9)
    pages = (T_max + P - 1) // P
    k_pool = torch.randn(L, B * pages, Hkv, P, d, generator=gen).bfloat16().cuda()
    v_pool = torch.randn(L, B * pages, Hkv, P, d, generator=gen).bfloat16().cuda()
    page_table = torch.randperm(B * pages, generator=gen).int().view(B, pages).cuda()
    streams = [token_stream(np.random.default_rng(20 + b), steps) for b in range(B)]
    toks = torch.tensor([[streams[b][t] for b in range(B)] for t in range(steps)], dtype=torch.int32).cuda()
    k_new = torch.randn(steps, B, L, Hkv, d, generator=gen).bfloat16().cuda()
    v_new = torch.randn(steps, B, L, Hkv, d, generator=gen).bfloat16().cuda()
    q = (0.25 * torch.randn(steps, B, L, Hq, d, generator=gen)).bfloat16().cuda()
    shape = Z.Shape(L, Hq, Hkv, d, P)
    res = []
    for chained, fused_a0 in ((True, True), (False, False)):
        kv = (k_pool.clone(), v_pool.clone(), page_table)
        lp = DecodeLoop(shape, B, MS, T_max, StepParams(2, 2, 4, 64), BEGIN, END, BOUNDARY, chained=chained,
                        fused_a0=fused_a0)
        lp.start(n_p)
        outs = torch.zeros(steps, *lp.out.shape, device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for t in range(steps):
                lp.decode_step(kv, k_new[t], v_new[t], q[t], toks[t])
                outs[t].copy_(lp.out)
        lp.start(n_p)
        g.replay()
        torch.cuda.synchronize()
        lp.check_status()
        res.append(dict(outs=outs, seq_len=lp.seq_len.clone(), bounds=lp.bounds.clone(),
                        num_summaries=lp.num_summaries.clone(), flags=lp.flags.clone(), k=kv[0], v=kv[1]))
    a, b = res
    assert int(a["num_summaries"].min()) >= 2
    for k in ("seq_len", "bounds", "num_summaries", "flags", "k", "v"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(a["outs"], b["outs"])
