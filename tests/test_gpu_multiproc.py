"""The sharded product paths run for real: 2 processes on cuda:0, gloo on CUDA tensors.

NCCL refuses two ranks on one device, gloo does not: each rank drives its own
libzoomr kernels on cuda:0 and exchanges through `parallel.py`'s own
collectives (the functions the NCCL deployment calls), so the code under test
is the product path end to end -- `HeadShardedStep.run` (a1, a2 over the rank's
heads, `nccl_allreduce_sum` of the int64 partial, a3, a4, a5) and
`TokenShardedStep` (a1 on the rank's own summaries + all-reduce of the
mean-key cache, replicated a2..a4, a5 with log-sum-exp over the rank's part of
I_f, the all-gather, `zoomr_merge_attn`).  The ranks' kernels never wait on
one another: every exchange is a host-mediated gloo collective.

Checked against the fp64 oracle run in the parent on the full (unsharded)
instance: every rank's flags and I_f bit-exact, votes exact, outputs within
2e-3 (the rank's heads for head sharding, every head after the merge for
token sharding), over several steps with changing queries.
"""
import dataclasses
import os
import socket
import tempfile

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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFGS = {
    "small_g4": S.Config("mp_small_g4", L=3, Hq=8, Hkv=2, d=128, T=2048, n_pairs=24, LR=60, LS=12, sink=4,
                         window=96, c=3, top_k=2, page=32, seed=51, batch=2),
    "small_g7": S.Config("mp_small_g7", L=2, Hq=14, Hkv=2, d=128, T=2048, n_pairs=24, LR=60, LS=12, sink=4,
                         window=96, c=3, top_k=2, page=32, seed=52, batch=2),
    "8b16k": dataclasses.replace(S.CONFIGS["8b16k"], seed=53),
}
STEPS = 3


def _queries(inp, step):
    """Step 0: the generator's planted query; later steps: other seeded queries."""
    if step == 0:
        return inp.q
    g = torch.Generator(device="cuda").manual_seed(1000 + step)
    return (0.25 * torch.randn(inp.q.shape, device="cuda", generator=g)).bfloat16()


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _head_worker(rank, world, port, name, outdir, fused=True):
    dist = _init(rank, world, port)
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import HeadShardedStep, shard_heads, slice_heads
    from paper_2604_10898_b200.step import StepParams
    cfg = CFGS[name]
    inp = S.generate(cfg, device="cuda")
    sh = shard_heads(cfg.Hq, cfg.Hkv, rank, world)
    kp, vp, _ = slice_heads(inp.k_pool, inp.v_pool, inp.q, sh)
    kv = (kp, vp, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st = HeadShardedStep(Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page), sh, inp.q.shape[0],
                         inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    newest = torch.tensor([[b, int(n) - 1] for b, n in enumerate(inp.num_summaries.cpu().tolist())],
                          dtype=torch.int32, device="cuda")
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    res = []
    for s in range(STEPS):
        q = _queries(inp, s)[:, :, sh.q_start:sh.q_stop].contiguous()
        st.run(q, kv, seg, close_items=newest, fused=fused)  # a1 (newest) a2 -> all-reduce -> a3 a4 a5
        torch.cuda.synchronize()
        st.check_status()
        res.append({k: getattr(st, k).cpu().clone() for k in ("partial", "flags", "index", "count", "out")})
    torch.save({"shard": (sh.q_start, sh.q_stop), "steps": res}, os.path.join(outdir, f"head{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _token_worker(rank, world, port, name, outdir):
    dist = _init(rank, world, port)
    from paper_2604_10898_b200 import zoomr as Z
    from paper_2604_10898_b200.parallel import TokenShardedStep, token_owner_map
    from paper_2604_10898_b200.step import StepParams
    cfg = CFGS[name]
    inp = S.generate(cfg, device="cuda")
    B, P = inp.q.shape[0], cfg.page
    stride = int(inp.page_table.shape[1]) * P
    own = token_owner_map(inp.bounds.cpu().numpy(), inp.num_summaries.cpu().numpy(), world, stride, chunk=64)
    owner = torch.from_numpy(own).cuda()
    # this rank holds only its tokens: every other row of the pools is NaN (a read would poison the result)
    kp, vp = inp.k_pool.clone(), inp.v_pool.clone()
    for b in range(B):
        t = torch.nonzero(owner[b] != rank).flatten()
        t = t[t < int(inp.page_table.shape[1]) * P]
        pages = inp.page_table[b].long()[t // P]
        kp[:, pages, :, t % P, :] = float("nan")
        vp[:, pages, :, t % P, :] = float("nan")
    kv = (kp, vp, inp.page_table)
    seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st = TokenShardedStep(Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, P), rank, world, B, inp.bounds.shape[1], cfg.T,
                          StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    mine = [(b, i) for b in range(B) for i in range(int(inp.num_summaries[b]))
            if own[b, int(inp.bounds[b, i, 2])] == rank]
    items = torch.tensor(mine if mine else [[0, 0]], dtype=torch.int32, device="cuda")[: len(mine)]
    st.update_mean_keys(kv, seg, items)  # a1 on this rank's summaries + all-reduce of the cache
    res = []
    for s in range(STEPS):
        st.run(_queries(inp, s), kv, seg, owner)  # replicated a2..a4, local a5 + lse, all-gather, merge
        torch.cuda.synchronize()
        st.check_status()
        res.append({k: getattr(st, k).cpu().clone() for k in ("flags", "index", "count", "out", "local_count")})
    torch.save({"mean_keys": st.mean_keys.cpu(), "steps": res}, os.path.join(outdir, f"token{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(fn, world, name, *extra):
    import torch.multiprocessing as mp
    d = tempfile.mkdtemp(prefix="zoomr_mp_")
    mp.spawn(fn, args=(world, _free_port(), name, d, *extra), nprocs=world, join=True)
    return d


def _oracle_steps(inp):
    """The oracle's full step on the unsharded instance, per sequence and step."""
    cfg = inp.cfg
    ref = []
    for s in range(STEPS):
        q = _queries(inp, s)
        per = []
        for b in range(inp.q.shape[0]):
            K, V = PY.host_kv(inp, b)
            per.append(oracle.step(S.bf16_bits(q[b]), K, V, PY.seg_host(inp, b), cfg.L, cfg.Hq, cfg.Hkv, cfg.d,
                                   cfg.top_k, cfg.c, cfg.sink, cfg.window))
        ref.append(per)
    return ref


@pytest.mark.parametrize("name,fused", [("small_g4", True), ("small_g4", False), ("8b16k", True)])
def test_head_sharded_step_two_processes(name, fused):
    """fused: zoomr_select_front -> all-reduce -> zoomr_select_tail -> a5 (the bench's
    path); not fused: a1, a2, all-reduce, a3, a4, a5 as separate calls."""
    world = 2
    d = _spawn(_head_worker, world, name, fused)
    inp = S.generate(CFGS[name], device="cuda")
    ref = _oracle_steps(inp)
    outs = [torch.load(os.path.join(d, f"head{r}.pt")) for r in range(world)]
    for s in range(STEPS):
        for r in range(world):
            x = outs[r]["steps"][s]
            assert torch.equal(x["partial"], outs[0]["steps"][s]["partial"])  # the all-reduced partial is replicated
            q0, q1 = outs[r]["shard"]
            for b in range(inp.q.shape[0]):
                o = ref[s][b]
                n = len(o["flags"])
                assert np.array_equal(x["partial"][b, 0, :n].numpy(), o["votes"]), "votes after the all-reduce"
                assert np.array_equal(x["flags"][b, :n].numpy(), o["flags"]), "flags"
                c = int(x["count"][b])
                assert np.array_equal(x["index"][b, :c].numpy(), o["index"]), "I_f"
                err = np.abs(x["out"][b].numpy().astype(np.float64) - o["out"][:, q0:q1]).max()
                assert err <= PY.ATTN_TOL, f"rank {r} step {s} seq {b}: attention err {err}"


@pytest.mark.parametrize("name,world", [("small_g7", 2), ("small_g4", 3)])
def test_token_sharded_step_processes(name, world):
    d = _spawn(_token_worker, world, name)
    inp = S.generate(CFGS[name], device="cuda")
    ref = _oracle_steps(inp)
    outs = [torch.load(os.path.join(d, f"token{r}.pt")) for r in range(world)]
    for r in range(world):  # the replicated mean-key cache: bit-exact to the oracle's fp64 means in fp32
        for b in range(inp.q.shape[0]):
            n = int(inp.num_summaries[b])
            mk = outs[r]["mean_keys"][b, :, :, :n].numpy()
            assert np.array_equal(mk, ref[0][b]["mean_keys"].astype(np.float32)), "replicated mean keys"
    for s in range(STEPS):
        for r in range(world):
            x = outs[r]["steps"][s]
            assert int(sum(outs[rr]["steps"][s]["local_count"].sum() for rr in range(world))) == \
                int(x["count"].sum()), "the ranks' parts partition I_f"
            for b in range(inp.q.shape[0]):
                o = ref[s][b]
                n = len(o["flags"])
                assert np.array_equal(x["flags"][b, :n].numpy(), o["flags"]), "flags"
                c = int(x["count"][b])
                assert np.array_equal(x["index"][b, :c].numpy(), o["index"]), "I_f"
                err = np.abs(x["out"][b].numpy().astype(np.float64) - o["out"]).max()
                assert err <= PY.ATTN_TOL, f"rank {r} step {s} seq {b}: merged attention err {err}"
