"""Guard-band checks of every libzoomr kernel's memory accesses.

compute-sanitizer is refused on this GPU pool (profiles/r02_sanitizer_refused.txt),
so out-of-bounds accesses are caught the way the pool's operators suggest, with
our own bounds checks: every device buffer a step touches -- its outputs and
workspaces AND its inputs (pools, queries, page table, segment table) -- is
re-allocated as the middle of a larger allocation whose bands before and after
hold a sentinel.  Output / workspace bands are 0xA5 bytes: an out-of-bounds
WRITE changes them.  Input bands are bf16 / fp32 NaN (0xFF bytes): an
out-of-bounds READ that reaches a result poisons it, so results must still be
finite and equal to the same step on unguarded buffers.  Covers the fused and
separate steps with and without the early rows, the chained steps in one
graph, the front / tail split, Algorithm 1's decode loop with a summary
closure, the token-sharded pieces, H2O and the host-memory tier."""
import dataclasses

import pytest
import torch

import zoomr_synth as S
from tests import parity as PY

pytestmark = pytest.mark.gpu

GUARD = 1 << 14  # bytes per band
OUT_BYTE = 0xA5
IN_BYTE = 0xFF


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10898_b200 import _build
    _build.build()


class Guards:
    def __init__(self):
        self.bands = []

    def wrap(self, t: torch.Tensor, fill: int) -> torch.Tensor:
        n = t.numel() * t.element_size()
        big = torch.full((n + 2 * GUARD,), fill, dtype=torch.uint8, device=t.device)
        inner = big[GUARD:GUARD + n].view(t.dtype).view(t.shape)
        inner.copy_(t)
        self.bands.append((big, n, fill))
        return inner

    def guard_obj(self, obj, fill=OUT_BYTE, skip=()):
        """Every CUDA tensor attribute of obj -> a guarded copy (same values)."""
        seen = {}
        for k, v in list(vars(obj).items()):
            if k in skip or not isinstance(v, torch.Tensor) or not v.is_cuda or v.numel() == 0:
                continue
            key = v.data_ptr()
            if key not in seen:
                seen[key] = self.wrap(v.contiguous(), fill)
            setattr(obj, k, seen[key])

    def check(self):
        torch.cuda.synchronize()
        for big, n, fill in self.bands:
            lo, hi = big[:GUARD], big[GUARD + n:]
            assert bool((lo == fill).all()) and bool((hi == fill).all()), "a guard band was overwritten"


def guarded_inputs(inp, g: Guards):
    out = dataclasses.replace(inp)
    for k in ("bounds", "num_summaries", "seq_len", "k_pool", "v_pool", "page_table", "q"):
        setattr(out, k, g.wrap(getattr(inp, k), IN_BYTE if k in ("k_pool", "v_pool", "q") else 0x7F))
    return out


def small(name, **kw):
    base = dict(name=name, L=2, Hq=8, Hkv=2, d=128, T=2048, n_pairs=24, LR=60, LS=12, sink=4, window=96,
                c=3, top_k=2, page=32, seed=61, batch=3, jitter=True)
    base.update(kw)
    return S.Config(**base)


def _newest(inp):
    return torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                        dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("cfg", [small("guard_g4"), small("guard_g7", Hq=14), small("guard_d64", d=64),
                                 S.CONFIGS["tiny"]], ids=lambda c: c.name)
def test_step_paths_stay_in_bounds(cfg):
    from paper_2604_10898_b200 import zoomr as Z
    raw = S.generate(cfg, device="cuda")
    ref = PY.make_step(raw, debug=False)
    PY.run_full(raw, ref, fused=True)
    g = Guards()
    inp = guarded_inputs(raw, g)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    for fused in (True, False):
        for early in (True, False):
            st = PY.make_step(inp, debug=True)
            st.early_known = early
            g.guard_obj(st)
            st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
            st.run(inp.q, kv, seg, close_items=_newest(inp), fused=fused)
            g.check()
            st.check_status()
            assert torch.isfinite(st.out).all()
            assert (st.out - ref.out).abs().max().item() <= 1e-5
            assert torch.equal(st.flags, ref.flags) and torch.equal(st.count, ref.count)
    # chained, back to back in one graph, and the front / tail split
    st = PY.make_step(inp, debug=False)
    st.chained = True
    g.guard_obj(st)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    newest = _newest(inp)
    st.run(inp.q, kv, seg, close_items=newest)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(3):
            st.run(inp.q, kv, seg, close_items=newest)
    gr.replay()
    g.check()
    assert (st.out - ref.out).abs().max().item() <= 1e-5
    Z.select_front(st.shape, inp.q, *kv, *seg, None, st.mean_keys, cfg.top_k, st.partial, st.sel_workspace,
                   dev_status=st.status)
    Z.select_tail(st.shape, *seg, st.partial, cfg.c, cfg.sink, cfg.window, st.flags, st.index, st.count,
                  agreeability=st.agreeability, dev_status=st.status)
    st.attend(inp.q, kv, inp.seq_len, phys=False)
    g.check()
    st.check_status()
    assert torch.equal(st.flags, ref.flags)


def test_decode_loop_policies_shard_tier_stay_in_bounds():
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
    from paper_2604_10898_b200.policies import PolicyStep
    from paper_2604_10898_b200.step import DecodeLoop, StepParams
    from paper_2604_10898_b200.tier import HostTierStep
    cfg = small("guard_misc", batch=2)
    raw = S.generate(cfg, device="cuda")
    g = Guards()
    inp = guarded_inputs(raw, g)
    shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
    prm = StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window)
    kv = (inp.k_pool, inp.v_pool, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    # Algorithm 1's device loop: 40 tokens with a summary closing and two boundaries
    lp = DecodeLoop(shape, 2, 32, cfg.T, prm, 1000, 1001, [200])
    g.guard_obj(lp)
    lp.start(1500)
    toks = [7] * 10 + [1000] + [7] * 5 + [1001] + [7] * 6 + [200] + [7] * 10 + [200] + [7] * 5
    for t in toks:
        k_new = torch.randn(2, cfg.L, cfg.Hkv, cfg.d, device="cuda").bfloat16()
        lp.decode_step(kv, g.wrap(k_new, IN_BYTE), g.wrap(torch.randn_like(k_new), IN_BYTE), inp.q,
                       g.wrap(torch.tensor([t, t], dtype=torch.int32, device="cuda"), 0x7F))
    g.check()
    lp.check_status()
    assert int(lp.num_summaries[0]) == 1 and torch.isfinite(lp.out).all()
    # comparison policies (a4 with fixed flags, H2O eviction + logits + accumulation)
    for pol in ("streamingllm", "sumr", "h2o"):
        ps = PolicyStep(pol, shape, 2, inp.bounds.shape[1], cfg.T, prm, budget=400, max_positions=cfg.T)
        g.guard_obj(ps)
        ps.prepare(inp.num_summaries)
        if pol == "h2o":
            ps.start_h2o(seg)
        for _ in range(3):
            ps.run(inp.q, kv, seg, update_selection=False)
        g.check()
        ps.check_status()
        assert torch.isfinite(ps.out).all()
    # token-sharded pieces: restriction, a5 + lse, merge
    world = 3
    own = token_owner_map(raw.bounds.cpu().numpy(), raw.num_summaries.cpu().numpy(), world,
                          int(raw.page_table.shape[1]) * cfg.page, 64)
    owner = g.wrap(torch.from_numpy(own).cuda(), 0x7F)
    steps = []

    def ex(out, lse, count, po, pl, pc):
        for r, t in enumerate(steps):
            po[r].copy_(t.out_local)
            pl[r].copy_(t.lse_local)
            pc[r].copy_(t.local_count)
    for r in range(world):
        t = TokenShardedStep(shape, r, world, 2, inp.bounds.shape[1], cfg.T, prm, exchange=ex,
                             reduce_mean_keys=lambda mk: None)
        g.guard_obj(t)
        t.update_mean_keys(kv, seg, t.all_items(inp.num_summaries))
        steps.append(t)
    for t in steps:
        t.run_local(inp.q, kv, seg, owner)
    steps[0].combine()
    g.check()
    for t in steps:
        t.check_status()
    assert torch.isfinite(steps[0].out).all()
    # host tier: plan + page copy + a5 on the hot pool (16-token hot pages)
    hk, hv = raw.k_pool.cpu().pin_memory(), raw.v_pool.cpu().pin_memory()
    ts = HostTierStep(shape, 2, inp.bounds.shape[1], cfg.T, prm, hk, hv, inp.page_table,
                      2 * int(raw.page_table.shape[1]) * 2, hot_page_size=16)
    g.guard_obj(ts, skip=("host_k", "host_v"))
    ts.mean_keys.copy_(steps[0].mean_keys)
    for _ in range(2):
        ts.run(inp.q, seg)
    g.check()
    ts.check_status()
    assert torch.isfinite(ts.out).all()
