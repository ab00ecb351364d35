"""Test helpers: bf16 bit conversion and an independent pure-Python brute force.

The brute force below re-derives ZoomR's selection (Alg.1 @P:404-424)
with Python sets, sorted() and plain float loops -- deliberately a different
idiom from the C oracle -- so that a dropped term, a wrong index or a flipped
tie rule in either one shows up as a disagreement on tiny random instances
(SPEC acceptance criterion 2).
"""
from __future__ import annotations

import math

import numpy as np
import torch


def to_bf16_bits(x) -> np.ndarray:
    """float array -> uint16 bf16 bit patterns (round-to-nearest-even via torch)."""
    t = torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def bf16_bits_to_float(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def brute_selection(keys, q, seg, top_k, c, sink, window, T):
    """Pure-Python selection. keys: float [T][L][Hkv][d]; q: float [L][Hq][d].

    Returns (per_voter_sets list[set], votes dict, I_c set, I_s set, I_f sorted list).
    """
    T_, L, Hkv, d = len(keys), len(keys[0]), len(keys[0][0]), len(keys[0][0][0])
    Hq = len(q[0])
    G = Hq // Hkv
    n = len(seg)
    if n == 0:
        I_f = sorted(set(range(min(sink, T))) | set(range(max(0, T - window), T)))
        return [], {}, set(), set(), I_f
    # mean keys
    mk = {}
    for l in range(L):
        for g in range(Hkv):
            for i, (r0, r1, s0, s1) in enumerate(seg):
                rows = [keys[j][l][g] for j in range(s0, s1)]
                mk[l, g, i] = [sum(r[e] for r in rows) / len(rows) for e in range(d)]
    sets, votes, A = [], {}, {}
    for l in range(L):
        for h in range(Hq):
            al = [sum(q[l][h][e] * mk[l, h // G, i][e] for e in range(d)) for i in range(n)]
            chosen = sorted(range(n), key=lambda i: (-al[i], i))[:top_k]
            sets.append(set(chosen))
            for i in chosen:
                votes[i] = votes.get(i, 0) + 1
                A[i] = A.get(i, 0.0) + al[i]
    ranked = sorted(votes, key=lambda i: (-votes[i], -A[i], i))
    I_c = set(ranked[:c])
    I_s = set(ranked[c:])
    I_f = set(range(min(sink, T))) | set(range(max(0, T - window), T))
    for i in I_c:
        I_f |= set(range(seg[i][0], seg[i][1]))
    for i in I_s:
        I_f |= set(range(seg[i][2], seg[i][3]))
    return sets, votes, I_c, I_s, sorted(I_f)


def random_layout(rng, T, n_pairs, sink):
    """Random valid segment table: pairs (R_i, S_i) in order after the sink, some R_i empty."""
    cuts = sorted(rng.choice(np.arange(sink, T + 1), size=3 * n_pairs, replace=True).tolist())
    seg = []
    for i in range(n_pairs):
        r0, r1, s1 = cuts[3 * i], cuts[3 * i + 1], cuts[3 * i + 2]
        if s1 <= r1:  # summary must be non-empty
            continue
        if seg and r0 < seg[-1][3]:
            continue
        seg.append((r0, r1, r1, s1))
    return seg


def sdpa_fp64(q_vec, K_rows, V_rows):
    """torch's scaled_dot_product_attention in fp64 on CPU for one query row."""
    qt = torch.as_tensor(np.asarray(q_vec, dtype=np.float64)).view(1, 1, 1, -1)
    kt = torch.as_tensor(np.asarray(K_rows, dtype=np.float64)).view(1, 1, len(K_rows), -1)
    vt = torch.as_tensor(np.asarray(V_rows, dtype=np.float64)).view(1, 1, len(V_rows), -1)
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).view(-1).numpy()


SIGMA_SPEC = math.exp(1 / math.sqrt(2)) / (math.exp(1 / math.sqrt(2)) + 1.0)
