"""Seeded synthetic inputs for the ZoomR hot path ("input recipe").

Shared by the product path, the tests, the bench and the oracle's callers, and
by design holds NONE of the method's arithmetic (no mean keys, scores, votes,
selection, index sets or attention): it only draws random tensors with the
structure of the paper's workloads and lays them out in a paged KV pool.

Structure:
  * segment table: sink [0, s), then N_t pairs (R_i of L_R tokens, S_i of L_S
    tokens) back to back, then the open tail up to T;
  * keys: per (b, l, g, pair i) a centroid mu ~ N(0, I_d); every token of R_i
    and S_i is mu + 0.5 * eps (segment-local keys, P:37 citing ShadowKV;
    summaries restate their segment); sink and tail keys ~ N(0, I_d);
  * values ~ N(0, I_d);
  * queries "planted": each sequence picks m = c target pairs; a voter (l, h)
    is on-target with probability 1 - f: q = (0.25 / sqrt(m)) (sum_t mu_t + 0.5 eps),
    else it targets m random pairs ("diffuse" = f = 1 with q = 0.25 N(0, I));
  * everything rounded to bf16 once; the page table is a seeded permutation
    of physical pages so page boundaries are real.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional

import torch


@dataclass(frozen=True)
class Config:
    name: str
    L: int
    Hq: int
    Hkv: int
    d: int
    T: int
    n_pairs: int          # N_t closed summaries
    LR: int               # regular-segment length
    LS: int               # summary length
    sink: int = 4
    window: int = 512
    c: int = 4
    top_k: int = 2
    page: int = 64
    batch: int = 1
    seed: int = 0
    off_target: float = 0.25   # f
    query: str = "planted"     # or "diffuse"
    jitter: bool = False       # L_R ~ U[0.8, 1.2] L_R, L_S ~ U[0.8, 1.2] L_S per pair (C3 variant)
    update_every: int = 1      # U (selection update interval, BJ stress config)

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def pages_per_seq(self) -> int:
        return (self.T + self.page - 1) // self.page

    def kv_bytes_per_token(self) -> int:
        return self.L * self.Hkv * self.d * 2 * 2


def _pairs_fit(T, sink, LR, LS, tail_min):
    return max(0, (T - sink - tail_min) // (LR + LS))


# BASELINE.json configs; seeds C1=1 .. C4=4, C5 = 5 + grid index.
CONFIGS = {
    # configs[0]: tiny, CPU oracle in seconds
    "tiny": Config("tiny", L=1, Hq=4, Hkv=2, d=16, T=256, n_pairs=8, LR=23, LS=4, sink=4, window=32,
                   c=2, top_k=2, page=16, seed=1),
    # configs[1]: Llama-3-8B shape, 16K reasoning context, batch 1 (the N=1 bench workload)
    "8b16k": Config("8b16k", L=32, Hq=32, Hkv=8, d=128, T=16384, n_pairs=120, LR=116, LS=16, sink=4,
                    window=512, c=4, top_k=2, seed=2),
    # configs[2]: same shape, 32K, batch 64 (batch-sharded)
    "8b32k": Config("8b32k", L=32, Hq=32, Hkv=8, d=128, T=32768, n_pairs=119, LR=250, LS=20, sink=4,
                    window=512, c=4, top_k=2, batch=64, seed=3),
    # Qwen2.5-7B shape (28 layers, 28 query / 4 KV heads: G = 7), 16K, batch 1
    "qwen7b16k": Config("qwen7b16k", L=28, Hq=28, Hkv=4, d=128, T=16384, n_pairs=120, LR=116, LS=16, sink=4,
                        window=512, c=4, top_k=2, seed=6),
    # configs[3]: Llama-3-70B shape, 64K, batch 1 (KV-head-sharded over 8 GPUs)
    "70b64k": Config("70b64k", L=80, Hq=64, Hkv=8, d=128, T=65536, n_pairs=240, LR=250, LS=20,
                     sink=4, window=512, c=4, top_k=2, seed=4),
}


def stress_config(LR: int, c: int, update_every: int = 1, grid_index: int = 0) -> Config:
    """configs[4]: 128K stress point on the 8B shape (L_S = 16, N_t = floor((T-516)/(L_R+16)))."""
    T = 131072
    n = (T - 516) // (LR + 16)
    return Config(f"stress_LR{LR}_c{c}_U{update_every}", L=32, Hq=32, Hkv=8, d=128, T=T, n_pairs=n,
                  LR=LR, LS=16, sink=4, window=512, c=c, top_k=2, seed=5 + grid_index,
                  update_every=update_every)


def config_by_name(name: str) -> Config:
    """'tiny' | '8b16k' | '8b32k' | '70b64k' | 'stress_LR<L_R>_c<c>_U<U>' (configs[4] grid point)."""
    if name in CONFIGS:
        return CONFIGS[name]
    if name.startswith("stress"):
        kv = {}
        for part in name.split("_")[1:]:
            key = part.rstrip("0123456789")
            kv[key] = int(part[len(key):])
        return stress_config(kv.get("LR", 64), kv.get("c", 8), kv.get("U", 1))
    raise KeyError(name)


@dataclass
class Inputs:
    cfg: Config
    bounds: torch.Tensor        # int32 [B][N_max][4]
    num_summaries: torch.Tensor  # int32 [B]
    seq_len: torch.Tensor       # int32 [B]
    k_pool: torch.Tensor        # bf16 [L][pages][Hkv][P][d]
    v_pool: torch.Tensor
    page_table: torch.Tensor    # int32 [B][max_pages]
    q: torch.Tensor             # bf16 [B][L][Hq][d]
    targets: list = field(default_factory=list)  # planted target pairs per sequence

    @property
    def device(self):
        return self.k_pool.device


def layout(cfg: Config, gen: Optional[torch.Generator] = None):
    """Segment table of one sequence: list of (r0, r1, s0, s1)."""
    seg, p = [], cfg.sink
    for _ in range(cfg.n_pairs):
        lr, ls = cfg.LR, cfg.LS
        if cfg.jitter and gen is not None:
            lr = int(cfg.LR * (0.8 + 0.4 * torch.rand((), generator=gen).item()))
            ls = max(1, int(cfg.LS * (0.8 + 0.4 * torch.rand((), generator=gen).item())))
        if p + lr + ls > cfg.T - 1:
            break
        seg.append((p, p + lr, p + lr, p + lr + ls))
        p += lr + ls
    return seg


def generate(cfg: Config, device="cuda", seed: Optional[int] = None, batch: Optional[int] = None,
             phys_pages: Optional[int] = None, query_mode: Optional[str] = None) -> Inputs:
    """Draw one batch of seeded synthetic inputs.

    phys_pages: if smaller than batch * pages_per_seq, logical pages of different
    sequences alias onto the same physical pages (seeded hash) -- used only to
    time configs whose full KV exceeds one GPU's HBM; the bytes read per step
    are unchanged, but the planted structure no longer holds on aliased pages.
    """
    dev = torch.device(device)
    B = cfg.batch if batch is None else batch
    seed = cfg.seed if seed is None else seed
    qmode = query_mode or cfg.query
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    hgen = torch.Generator()
    hgen.manual_seed(seed)
    L, Hq, Hkv, d, P, T = cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page, cfg.T
    G = Hq // Hkv
    npg = cfg.pages_per_seq
    total_logical = B * npg
    nphys = total_logical if phys_pages is None else min(phys_pages, total_logical)

    segs = [layout(cfg, hgen) for _ in range(B)]
    nmax = max(1, max(len(s) for s in segs))
    bounds = torch.zeros(B, nmax, 4, dtype=torch.int32)
    for b, s in enumerate(segs):
        if s:
            bounds[b, :len(s)] = torch.tensor(s, dtype=torch.int32)
    num_summaries = torch.tensor([len(s) for s in segs], dtype=torch.int32)
    seq_len = torch.full((B,), T, dtype=torch.int32)

    # page table: seeded permutation of physical pages (aliasing if nphys < B*npg)
    perm = torch.randperm(total_logical, generator=hgen)
    page_table = (perm % nphys).to(torch.int32).view(B, npg)

    k_pool = torch.empty(L, nphys, Hkv, P, d, dtype=torch.bfloat16, device=dev)
    v_pool = torch.empty_like(k_pool)
    q = torch.empty(B, L, Hq, d, dtype=torch.bfloat16, device=dev)
    targets = []
    pt_dev = page_table.to(dev).long()
    Tp = npg * P
    for b in range(B):
        s = segs[b]
        n = len(s)
        # pair id per token (-1 = sink / tail)
        pair = torch.full((Tp,), -1, dtype=torch.long)
        for i, (r0, r1, s0, s1) in enumerate(s):
            pair[r0:s1] = i
        pair = pair.to(dev)
        in_pair = pair >= 0
        pidx = pair.clamp(min=0)
        mu_all = torch.randn(L, Hkv, max(n, 1), d, generator=gen, device=dev)
        for l in range(L):
            k = torch.randn(Tp, Hkv, d, generator=gen, device=dev)
            if n:
                mu_tok = mu_all[l][:, pidx].permute(1, 0, 2)  # [Tp][Hkv][d]
                k = torch.where(in_pair[:, None, None], mu_tok + 0.5 * k, k)
            v = torch.randn(Tp, Hkv, d, generator=gen, device=dev)
            kp = k.to(torch.bfloat16).view(npg, P, Hkv, d).permute(0, 2, 1, 3)
            vp = v.to(torch.bfloat16).view(npg, P, Hkv, d).permute(0, 2, 1, 3)
            k_pool[l].index_copy_(0, pt_dev[b], kp.contiguous())
            v_pool[l].index_copy_(0, pt_dev[b], vp.contiguous())
        # queries
        m = max(1, cfg.c)
        if qmode == "diffuse" or n == 0:
            qb = 0.25 * torch.randn(L, Hq, d, generator=gen, device=dev)
            targets.append([])
        else:
            m = min(m, n)
            tgt = torch.randperm(n, generator=hgen)[:m]
            targets.append(sorted(tgt.tolist()))
            noise = torch.randn(L, Hq, d, generator=gen, device=dev)
            mu_q = mu_all.repeat_interleave(G, dim=1)  # [L][Hq][n][d]
            on = mu_q[:, :, tgt.to(dev)].sum(2)
            rnd = torch.randint(0, n, (L, Hq, m), generator=gen, device=dev)
            off = torch.gather(mu_q, 2, rnd[..., None].expand(L, Hq, m, d)).sum(2)
            is_off = torch.rand(L, Hq, generator=gen, device=dev) < cfg.off_target
            base = torch.where(is_off[..., None], off, on)
            qb = (0.25 / math.sqrt(m)) * (base + 0.5 * noise)
        q[b] = qb.to(torch.bfloat16)
        del mu_all
    return Inputs(cfg=replace(cfg, batch=B), bounds=bounds.to(dev), num_summaries=num_summaries.to(dev),
                  seq_len=seq_len.to(dev), k_pool=k_pool, v_pool=v_pool,
                  page_table=page_table.to(dev), q=q, targets=targets)


def logical_rows(inp: Inputs, b: int, which: str = "k", layers=None, heads=None) -> torch.Tensor:
    """Gather sequence b's cache back into logical token order: [T][L'][H'][d] bf16.

    Plumbing (a page-table gather with torch indexing), used to hand the oracle
    exactly the bytes the pool holds."""
    pool = inp.k_pool if which == "k" else inp.v_pool
    cfg = inp.cfg
    dev = pool.device
    lay = torch.arange(cfg.L, device=dev) if layers is None else torch.as_tensor(list(layers), device=dev)
    hed = torch.arange(cfg.Hkv, device=dev) if heads is None else torch.as_tensor(list(heads), device=dev)
    pt = inp.page_table[b].long()
    sub = pool.index_select(0, lay).index_select(1, pt).index_select(2, hed)  # [L'][npg][H'][P][d]
    sub = sub.permute(1, 3, 0, 2, 4).reshape(-1, lay.numel(), hed.numel(), cfg.d)
    return sub[: int(inp.seq_len[b])]


def bf16_bits(t: torch.Tensor):
    """bf16 tensor -> numpy uint16 bit patterns (host copy)."""
    import numpy as np
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view(np.uint16)
