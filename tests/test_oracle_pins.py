"""Pins for the CPU oracle (oracle/zoomr_oracle.c) -- CPU only.

Each test pins an oracle function to something other than itself: a SPEC worked
example, a value the paper prints, a closed form, an invariant, a textbook or
library routine (torch SDPA in fp64), or an independent pure-Python brute force.
Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import math

import numpy as np
import pytest

import oracle
from tests.util import (SIGMA_SPEC, bf16_bits_to_float, brute_selection, random_layout, sdpa_fp64,
                        to_bf16_bits)


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


# ----------------------------------------------------------------- O1 -----
def _keys_1head(rows, T=None):
    """rows: list of d-vectors -> keys [T][1][1][d] bf16 bits."""
    a = np.asarray(rows, dtype=np.float32)
    return to_bf16_bits(a.reshape(a.shape[0], 1, 1, -1))


def test_mean_key_spec_examples():
    # S:109 single key [3,-1] -> [3,-1]
    mk = oracle.update_mean_keys(_keys_1head([[3, -1]]), [[0, 0, 0, 1]], 1, 1, 2)
    assert mk[0, 0, 0].tolist() == [3.0, -1.0]
    # S:110 keys [2,0],[0,2] -> [1,1]
    mk = oracle.update_mean_keys(_keys_1head([[2, 0], [0, 2]]), [[0, 0, 0, 2]], 1, 1, 2)
    assert mk[0, 0, 0].tolist() == [1.0, 1.0]
    # S:111 keys [1,0],[2,1],[3,5] -> [2,2]
    mk = oracle.update_mean_keys(_keys_1head([[1, 0], [2, 1], [3, 5]]), [[0, 0, 0, 3]], 1, 1, 2)
    assert mk[0, 0, 0].tolist() == [2.0, 2.0]


def test_mean_key_uses_exactly_the_summary_range():
    # tokens outside S_i are huge: an off-by-one range (s1 inclusive, r0 start) would show.
    rows = [[1000, 1000]] * 4 + [[2, 4], [4, 8]] + [[-1000, 500]] * 3
    seg = [[0, 4, 4, 6]]
    mk = oracle.update_mean_keys(_keys_1head(rows), seg, 1, 1, 2)
    assert mk[0, 0, 0].tolist() == [3.0, 6.0]


def test_mean_key_layer_head_addressing():
    # distinct constant per (layer, kv-head): mean must return that constant
    L, H, d, T = 3, 2, 4, 10
    k = np.zeros((T, L, H, d), np.float32)
    for l in range(L):
        for h in range(H):
            k[:, l, h, :] = 10 * l + h + np.arange(d) / 8
    mk = oracle.update_mean_keys(to_bf16_bits(k), [[0, 2, 2, 5], [5, 7, 7, 9]], L, H, d)
    for l in range(L):
        for h in range(H):
            for i in range(2):
                np.testing.assert_array_equal(mk[l, h, i], 10 * l + h + np.arange(d) / 8)


def test_mean_key_permutation_invariance_and_linearity():
    rng = np.random.default_rng(0)
    rows = rng.integers(-8, 8, size=(8, 4)).astype(np.float32)
    seg = [[0, 0, 0, 8]]
    m1 = oracle.update_mean_keys(_keys_1head(rows), seg, 1, 1, 4)
    m2 = oracle.update_mean_keys(_keys_1head(rows[::-1].copy()), seg, 1, 1, 4)
    m3 = oracle.update_mean_keys(_keys_1head(2 * rows), seg, 1, 1, 4)
    np.testing.assert_array_equal(m1, m2)
    np.testing.assert_array_equal(2 * m1, m3)


def test_segment_validation_errors():
    # EmptySegment, order, beyond T
    assert oracle.validate_segments([[0, 2, 2, 2]], 10) == oracle.ZO_ERR_EMPTY_SEGMENT
    assert oracle.validate_segments([[0, 3, 2, 4]], 10) == oracle.ZO_ERR_SEGMENT_ORDER
    assert oracle.validate_segments([[0, 2, 2, 4], [3, 5, 5, 6]], 10) == oracle.ZO_ERR_SEGMENT_ORDER
    assert oracle.validate_segments([[0, 2, 2, 11]], 10) == oracle.ZO_ERR_INDEX_RANGE
    assert oracle.validate_segments([[0, 2, 2, 4], [4, 4, 4, 6]], 10) == oracle.ZO_OK


# ----------------------------------------------------------------- O2 -----
def _score1(qv, kbars, k=1):
    """one layer, one head."""
    d = len(qv)
    q = to_bf16_bits(np.asarray(qv, np.float32).reshape(1, 1, d))
    mk = np.asarray(kbars, np.float64).reshape(1, 1, len(kbars), d)
    return oracle.score(q, mk, k, 1, 1, 1, d)


def test_score_spec_examples():
    assert _score1([1, 2], [[3, 4]])["alpha"][0, 0].tolist() == [11.0]
    assert _score1([0, 0], [[3, 4], [-7, 2]])["alpha"][0, 0].tolist() == [0.0, 0.0]
    assert _score1([1, -1], [[1, 1], [2, 0], [0, 3]])["alpha"][0, 0].tolist() == [0.0, 2.0, -3.0]


def test_score_no_sqrt_d_scale_and_linearity():
    rng = np.random.default_rng(1)
    d = 16
    kb = rng.integers(-4, 4, size=(5, d)).astype(np.float64)
    q1 = rng.integers(-4, 4, size=d)
    q2 = rng.integers(-4, 4, size=d)
    a1 = _score1(q1, kb)["alpha"][0, 0]
    a2 = _score1(q2, kb)["alpha"][0, 0]
    a12 = _score1(q1 + q2, kb)["alpha"][0, 0]
    np.testing.assert_array_equal(a1 + a2, a12)  # S:143 linearity (exact on small ints)
    # raw inner product, not divided by sqrt(d): integer inputs give integer alpha
    assert np.all(a1 == np.round(a1)) and np.abs(a1).max() > 4


def test_score_gqa_head_mapping():
    # reading Q6: query head h uses KV head h // G.  kv-head 0 keys favour summary 0,
    # kv-head 1 keys favour summary 1; all-ones queries.
    L, Hq, Hk, d, n = 1, 4, 2, 2, 2
    mk = np.zeros((L, Hk, n, d))
    mk[0, 0, 0] = [5, 5]; mk[0, 0, 1] = [1, 1]
    mk[0, 1, 0] = [1, 1]; mk[0, 1, 1] = [5, 5]
    q = to_bf16_bits(np.ones((L, Hq, d), np.float32))
    r = oracle.score(q, mk, 1, L, Hq, Hk, d)
    assert r["topk"][:, 0].tolist() == [0, 0, 1, 1]


# ----------------------------------------------------------------- O3 -----
def test_topk_spec_examples():
    # S:127 [0.9,0.1,0.5], k=2 -> {1,3} 1-based = {0,2}
    r = _score1([1.0], [[0.9], [0.1], [0.5]], k=2)
    assert sorted(r["topk"][0].tolist()) == [0, 2]
    # S:128 [0.5,0.5,0.1], k=1 -> {1} (smaller index wins the tie)
    r = _score1([1.0], [[0.5], [0.5], [0.1]], k=1)
    assert r["topk"][0].tolist() == [0]
    # S:129 length 2, k=5 -> both
    r = _score1([1.0], [[0.5], [0.7]], k=5)
    assert sorted(r["topk"][0].tolist()) == [0, 1]


def test_topk_zero_query_picks_oldest():
    # q = 0 -> every alpha is 0 -> the first k indices (tie rule)
    r = _score1([0.0, 0.0], [[1, 2], [3, 4], [5, 6], [7, 8]], k=3)
    assert r["topk"][0].tolist() == [0, 1, 2]


def test_topk_matches_sort_then_take_with_duplicates():
    rng = np.random.default_rng(2)
    for trial in range(300):
        n = int(rng.integers(1, 12))
        k = int(rng.integers(1, 6))
        vals = rng.integers(-3, 4, size=n).astype(np.float64)  # many duplicates
        r = _score1([1.0], vals.reshape(n, 1), k=k)
        want = sorted(range(n), key=lambda i: (-vals[i], i))[:k]
        assert r["topk"][0].tolist() == want


# ----------------------------------------------------------------- O4 -----
def test_votes_spec_example():
    # S:184 sets {1,3},{1,2},{3,1},{2,4} (1-based) -> v = {1:3, 2:2, 3:2, 4:1}
    sets = np.array([[1, 3], [1, 2], [3, 1], [2, 4]], np.int32) - 1
    alpha = np.zeros((1, 4, 4))
    v, A = oracle.aggregate(alpha, sets, 1, 4, 1, 1)
    assert v.tolist() == [3, 2, 2, 1]


def test_votes_sum_invariant_and_A():
    rng = np.random.default_rng(3)
    L, Hq, Hk, d, n, k = 2, 4, 2, 8, 7, 3
    mk = rng.integers(-4, 4, size=(L, Hk, n, d)).astype(np.float64)
    q = to_bf16_bits(rng.integers(-3, 3, size=(L, Hq, d)).astype(np.float32))
    r = oracle.score(q, mk, k, L, Hq, Hk, d)
    assert r["votes"].sum() == L * Hq * min(k, n)
    # A_i = sum over voters that chose i of alpha
    A = np.zeros(n)
    for v in range(L * Hq):
        for i in r["topk"][v]:
            A[i] += r["alpha"].reshape(L * Hq, n)[v, i]
    np.testing.assert_array_equal(A, r["A"])


# ----------------------------------------------------------------- O5 -----
def test_consensus_spec_examples():
    v = np.array([0, 3, 2, 2, 1], np.int64)  # index 0 unused (1-based example)
    A = np.zeros(5)
    flags, ag, _ = oracle.select_topc(v, A, 2)
    assert np.nonzero(flags == 2)[0].tolist() == [1, 2]  # S:193 I_c={1,2}
    assert np.nonzero(flags == 1)[0].tolist() == [3, 4]
    assert ag == 5 / 8
    flags, ag, _ = oracle.select_topc(v, A, 0)  # S:194 c = 0
    assert (flags == 2).sum() == 0 and np.nonzero(flags == 1)[0].tolist() == [1, 2, 3, 4]
    v7 = np.zeros(8, np.int64); v7[7] = 4
    flags, ag, _ = oracle.select_topc(v7, np.zeros(8), 3)  # S:195 clamp
    assert np.nonzero(flags == 2)[0].tolist() == [7] and (flags == 1).sum() == 0 and ag == 1.0
    flags, ag, _ = oracle.select_topc(np.array([2, 2], np.int64), np.zeros(2), 1)
    assert ag == 0.5


def test_consensus_tie_breaks_A_then_index():
    v = np.array([2, 2, 2, 5], np.int64)
    A = np.array([1.0, 3.0, 3.0, -9.0])
    flags, _, _ = oracle.select_topc(v, A, 2)
    assert np.nonzero(flags == 2)[0].tolist() == [1, 3]  # 3 by votes, then 1 by A over 0, 2
    A2 = np.array([1.0, 3.0, 3.0 * (1 + 1e-9), -9.0])
    flags, _, near = oracle.select_topc(v, A2, 2)
    assert np.nonzero(flags == 2)[0].tolist() == [2, 3] and near  # kept 2 vs dropped 1: 1e-9 apart
    flags, _, near = oracle.select_topc(v, A2, 3)
    assert not near  # cut between 1 (A=3) and 0 (A=1)
    v2 = np.array([2, 2, 1], np.int64)
    _, _, near = oracle.select_topc(v2, np.array([3.0, 3.0, 0.0]), 1)
    assert not near  # exact ties are never certified (reading Q23)
    _, _, near = oracle.select_topc(v2, np.array([3.0, 3.0 * (1 + 1e-9), 0.0]), 1)
    assert near  # certified near-tie at the cut (reading Q23)


def test_consensus_invariants_random():
    rng = np.random.default_rng(4)
    for _ in range(200):
        n = int(rng.integers(1, 20))
        v = rng.integers(0, 4, size=n).astype(np.int64)
        A = rng.integers(-2, 3, size=n).astype(np.float64)
        c = int(rng.integers(0, 5))
        flags, ag, _ = oracle.select_topc(v, A, c)
        I_all = set(np.nonzero(v > 0)[0].tolist())
        I_c = set(np.nonzero(flags == 2)[0].tolist())
        I_s = set(np.nonzero(flags == 1)[0].tolist())
        assert I_c | I_s == I_all and not (I_c & I_s)
        assert len(I_c) == min(c, len(I_all))
        if I_c and I_s:
            assert min(v[i] for i in I_c) >= max(v[i] for i in I_s)
        if I_all and c >= 1:  # AG in (0, 1]; 1 when |I_all| <= c
            assert 0 < ag <= 1 and (len(I_all) > c or ag == 1.0)


# ----------------------------------------------------------------- O6 -----
def test_index_spec_example():
    # prompt [0,4), R1=[4,10), S1=[10,12), R2=[12,16), S2=[16,18), window {18,19},
    # I_c={2}, I_s={1} -> {0,1,2,3,10,11,12,13,14,15,18,19}
    seg = [[4, 10, 10, 12], [12, 16, 16, 18]]
    idx = oracle.build_index(seg, [1, 2], 20, 4, 2)
    assert idx.tolist() == [0, 1, 2, 3, 10, 11, 12, 13, 14, 15, 18, 19]


def _paper_layout(n_pairs, Np=512, LR=250, LS=20, Nw=512):
    seg, p = [], Np
    for _ in range(n_pairs):
        seg.append([p, p + LR, p + LR, p + LR + LS])
        p += LR + LS
    return seg, p + Nw


def test_index_count_reproduces_paper_memory_examples():
    # N_p=512, N_w=512, c=2, L_R=250, L_S=20, |I_all|=80 -> denominator 3084, 5.48x
    seg, T = _paper_layout(80)
    flags = np.ones(80, np.uint8); flags[:2] = 2
    idx = oracle.build_index(seg, flags, T, 512, 512)
    assert len(idx) == 3084
    assert round((512 + 16384) / len(idx), 2) == 5.48
    # N_g = 32K "approximately 7.11x" (|I_all| = 160 per S:284)
    seg, T = _paper_layout(160)
    flags = np.ones(160, np.uint8); flags[:2] = 2
    idx = oracle.build_index(seg, flags, T, 512, 512)
    assert len(idx) == 4684
    assert round((512 + 32768) / len(idx), 2) == 7.11


def test_index_streaming_and_degenerate_cases():
    # S:342-344 streaming: sink=2, window=3, length 10 -> {0,1,7,8,9}
    assert oracle.build_index(np.zeros((0, 4)), [], 10, 2, 3).tolist() == [0, 1, 7, 8, 9]
    # window >= T -> everything
    assert oracle.build_index([[2, 4, 4, 6]], [0], 8, 1, 100).tolist() == list(range(8))
    # overlapping window and S_2 deduplicated
    seg = [[4, 10, 10, 12], [12, 16, 16, 18]]
    idx = oracle.build_index(seg, [0, 1], 19, 4, 2)
    assert idx.tolist() == [0, 1, 2, 3, 16, 17, 18]


def test_index_count_identity_random():
    # |I_f| = s + w + sum_{I_c}|R_i| + sum_{I_s}|S_i| on disjoint layouts (BJ invariant)
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(0, 10))
        s, w = int(rng.integers(0, 6)), int(rng.integers(1, 6))
        seg, p = [], s
        for _ in range(n):
            lr, ls = int(rng.integers(0, 6)), int(rng.integers(1, 4))
            seg.append([p, p + lr, p + lr, p + lr + ls]); p += lr + ls
        T = p + w + int(rng.integers(0, 4))
        flags = rng.integers(0, 3, size=n).astype(np.uint8)
        idx = oracle.build_index(np.asarray(seg).reshape(-1, 4), flags, T, s, w)
        want = s + w + sum(seg[i][1] - seg[i][0] for i in range(n) if flags[i] == 2) + \
            sum(seg[i][3] - seg[i][2] for i in range(n) if flags[i] == 1)
        assert len(idx) == want
        assert np.all(np.diff(idx) > 0)


# ----------------------------------------------------------------- O7 -----
def test_attention_spec_examples():
    one = to_bf16_bits([[0.5, -2.0]])
    o = oracle.attend_one(to_bf16_bits([1.0, 3.0]), one, to_bf16_bits([[7.0, -1.5]]), [0])
    assert o.tolist() == [7.0, -1.5]  # S:136 single pair -> v exactly
    K = to_bf16_bits([[1.0, 1.0], [1.0, 1.0]])
    V = to_bf16_bits([[2.0, 0.0], [4.0, 8.0]])
    o = oracle.attend_one(to_bf16_bits([0.3, 0.7]), K, V, [0, 1])
    np.testing.assert_allclose(o, [3.0, 4.0], rtol=0, atol=1e-15)  # S:137 equal logits
    o = oracle.attend_one(to_bf16_bits([1.0, 0.0]), to_bf16_bits([[1.0, 0.0], [0.0, 1.0]]),
                          to_bf16_bits([[1.0, 0.0], [0.0, 1.0]]), [0, 1])
    np.testing.assert_allclose(o, [SIGMA_SPEC, 1 - SIGMA_SPEC], rtol=0, atol=1e-15)
    assert abs(SIGMA_SPEC - 0.6698) < 1e-4


def test_attention_matches_torch_sdpa_fp64():
    rng = np.random.default_rng(6)
    for _ in range(20):
        T, d = int(rng.integers(2, 60)), int(rng.choice([4, 16, 64]))
        kb = to_bf16_bits(rng.normal(size=(T, d)) * 2)
        vb = to_bf16_bits(rng.normal(size=(T, d)))
        qb = to_bf16_bits(rng.normal(size=d))
        idx = np.sort(rng.choice(T, size=int(rng.integers(1, T + 1)), replace=False))
        o = oracle.attend_one(qb, kb, vb, idx)
        ref = sdpa_fp64(bf16_bits_to_float(qb), bf16_bits_to_float(kb)[idx],
                        bf16_bits_to_float(vb)[idx])
        np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)


def test_attention_subset_equals_full_and_shift_invariance():
    rng = np.random.default_rng(7)
    T, d = 20, 8
    kb = to_bf16_bits(rng.normal(size=(T, d)))
    vb = to_bf16_bits(rng.normal(size=(T, d)))
    qb = to_bf16_bits(rng.normal(size=d))
    full = oracle.attend_one(qb, kb, vb, np.arange(T))
    # full index set == dense attention (vs torch over all rows)
    ref = sdpa_fp64(bf16_bits_to_float(qb), bf16_bits_to_float(kb), bf16_bits_to_float(vb))
    np.testing.assert_allclose(full, ref, atol=1e-12, rtol=0)
    # S:145 shift invariance: append a constant bias dimension to every key
    k2 = np.concatenate([bf16_bits_to_float(kb), np.full((T, 1), 3.0)], 1)
    q2 = np.concatenate([bf16_bits_to_float(qb), [2.0]])
    v2 = np.concatenate([bf16_bits_to_float(vb), np.zeros((T, 1))], 1)
    o2 = oracle.attend_one(to_bf16_bits(q2), to_bf16_bits(k2), to_bf16_bits(v2), np.arange(T),
                           scale=1 / math.sqrt(d))
    np.testing.assert_allclose(o2[:d], full, atol=1e-12, rtol=0)


def test_attention_gqa_and_layout_addressing():
    rng = np.random.default_rng(8)
    T, L, Hq, Hk, d = 12, 2, 4, 2, 8
    K = to_bf16_bits(rng.normal(size=(T, L, Hk, d)))
    V = to_bf16_bits(rng.normal(size=(T, L, Hk, d)))
    q = to_bf16_bits(rng.normal(size=(L, Hq, d)))
    idx = np.array([0, 3, 4, 9, 11], np.int32)
    out = oracle.sparse_decode_attn(q, K, V, idx, L, Hq, Hk, d)
    Kf, Vf, qf = bf16_bits_to_float(K), bf16_bits_to_float(V), bf16_bits_to_float(q)
    for l in range(L):
        for h in range(Hq):
            ref = sdpa_fp64(qf[l, h], Kf[idx, l, h // 2], Vf[idx, l, h // 2])
            np.testing.assert_allclose(out[l, h], ref, atol=1e-12, rtol=0)


# ------------------------------------------------------------ whole step --
def _random_instance(rng, L, Hq, Hk, d, T, n_pairs, sink):
    seg = random_layout(rng, T, n_pairs, sink)
    K = to_bf16_bits(rng.integers(-3, 4, size=(T, L, Hk, d)) * 0.5)
    V = to_bf16_bits(rng.normal(size=(T, L, Hk, d)))
    q = to_bf16_bits(rng.integers(-3, 4, size=(L, Hq, d)) * 0.25)
    return seg, K, V, q


def test_step_selection_matches_python_brute_force():
    # SPEC acceptance 2 style: L,H in [1,4], d in {2,4,8}, N_t in [0,20], k in [1,4], c in [0,3]
    rng = np.random.default_rng(9)
    for trial in range(150):
        L = int(rng.integers(1, 5)); Hk = int(rng.integers(1, 3)); G = int(rng.integers(1, 3))
        Hq = Hk * G; d = int(rng.choice([2, 4, 8]))
        T = int(rng.integers(8, 90)); sink = int(rng.integers(0, 5)); window = int(rng.integers(1, 12))
        top_k = int(rng.integers(1, 5)); c = int(rng.integers(0, 4))
        seg, K, V, q = _random_instance(rng, L, Hq, Hk, d, T, int(rng.integers(0, 21)), sink)
        r = oracle.step(q, K, V, np.asarray(seg, np.int32).reshape(-1, 4), L, Hq, Hk, d, top_k, c,
                        sink, window)
        sets, votes, I_c, I_s, I_f = brute_selection(
            bf16_bits_to_float(K).tolist(), bf16_bits_to_float(q).tolist(), seg, top_k, c, sink,
            window, T)
        if seg:
            assert [set(x.tolist()) for x in r["topk"]] == sets
            assert {i: int(v) for i, v in enumerate(r["votes"]) if v} == votes
            assert set(np.nonzero(r["flags"] == 2)[0].tolist()) == I_c
            assert set(np.nonzero(r["flags"] == 1)[0].tolist()) == I_s
        assert r["index"].tolist() == I_f


def test_step_dense_equivalence():
    # BJ invariant: k >= N_t and c >= N_t -> I_all = I_c = all, I_s = {} ->
    # I_f = sink u all R_i u window, and the output equals dense attention over exactly that set.
    rng = np.random.default_rng(10)
    L, Hq, Hk, d, T, sink, window = 2, 4, 2, 8, 80, 3, 6
    seg, K, V, q = _random_instance(rng, L, Hq, Hk, d, T, 8, sink)
    n = len(seg)
    r = oracle.step(q, K, V, np.asarray(seg, np.int32), L, Hq, Hk, d, n, n, sink, window)
    assert (r["flags"] == 2).all()
    want = set(range(sink)) | set(range(T - window, T))
    for s in seg:
        want |= set(range(s[0], s[1]))
    assert r["index"].tolist() == sorted(want)
    idx = np.array(sorted(want))
    Kf, Vf, qf = bf16_bits_to_float(K), bf16_bits_to_float(V), bf16_bits_to_float(q)
    for l in range(L):
        for h in range(Hq):
            ref = sdpa_fp64(qf[l, h], Kf[idx, l, h // 2], Vf[idx, l, h // 2])
            np.testing.assert_allclose(r["out"][l, h], ref, atol=1e-12, rtol=0)


def test_step_special_cases_streaming_and_sumr():
    rng = np.random.default_rng(11)
    L, Hq, Hk, d, T, sink, window = 1, 2, 1, 4, 60, 2, 5
    seg, K, V, q = _random_instance(rng, L, Hq, Hk, d, T, 6, sink)
    segs = np.asarray(seg, np.int32).reshape(-1, 4)
    # N_t = 0 -> StreamingLLM
    r = oracle.step(q, K, V, np.zeros((0, 4), np.int32), L, Hq, Hk, d, 2, 2, sink, window)
    assert r["index"].tolist() == sorted(set(range(sink)) | set(range(T - window, T)))
    # c = 0, k >= N_t -> SumR: sink u all S_i u window
    r = oracle.step(q, K, V, segs, L, Hq, Hk, d, len(seg), 0, sink, window)
    want = set(range(sink)) | set(range(T - window, T))
    for s in seg:
        want |= set(range(s[2], s[3]))
    assert r["index"].tolist() == sorted(want)


def test_step_query_scale_invariance():
    # scaling every query by 2^m leaves every set unchanged
    rng = np.random.default_rng(12)
    L, Hq, Hk, d, T, sink, window = 2, 4, 2, 8, 100, 4, 8
    seg, K, V, q = _random_instance(rng, L, Hq, Hk, d, T, 10, sink)
    segs = np.asarray(seg, np.int32)
    r1 = oracle.step(q, K, V, segs, L, Hq, Hk, d, 2, 2, sink, window)
    q8 = to_bf16_bits(bf16_bits_to_float(q) * 8)
    r2 = oracle.step(q8, K, V, segs, L, Hq, Hk, d, 2, 2, sink, window)
    for key in ("topk", "votes", "flags", "index"):
        np.testing.assert_array_equal(r1[key], r2[key])


def test_step_planted_relevance_recall():
    # zero key spread, query planted on one segment -> its R_i is in I_f (recall 1)
    rng = np.random.default_rng(13)
    L, Hq, Hk, d, sink, window = 2, 4, 2, 64, 4, 8
    seg, p = [], sink
    for _ in range(10):
        seg.append([p, p + 12, p + 12, p + 15]); p += 15
    T = p + window
    for target in range(10):
        mu = rng.normal(size=(L, Hk, 10, d))
        K = rng.normal(size=(T, L, Hk, d))
        for i, s in enumerate(seg):
            K[s[0]:s[3]] = mu[:, :, i][None]
        q = np.repeat(mu[:, :, target], Hq // Hk, axis=1)
        r = oracle.step(to_bf16_bits(q), to_bf16_bits(K), to_bf16_bits(K), np.asarray(seg, np.int32),
                        L, Hq, Hk, d, 2, 1, sink, window)
        assert set(range(seg[target][0], seg[target][1])) <= set(r["index"].tolist())


# ----------------------------------------------------------------- O8 -----
# (token-sharded split-K: the softmax normaliser in log form)
def test_log_partition_closed_forms():
    # one row: ln e^z = z = q.k * scale, by hand: (1*2 + 3*(-1)) / sqrt(2)
    q = to_bf16_bits([[[1.0, 3.0]]])
    k = to_bf16_bits([[[[2.0, -1.0]]]])
    lse = oracle.log_partition(q, k, [0], 1, 1, 1, 2)
    assert abs(lse[0, 0] - (-1.0 / math.sqrt(2))) < 1e-15
    # q = 0: every logit is 0, ln(count)
    rng = np.random.default_rng(31)
    K = to_bf16_bits(rng.normal(size=(9, 2, 2, 8)))
    lse = oracle.log_partition(to_bf16_bits(np.zeros((2, 4, 8))), K, [0, 2, 3, 7, 8], 2, 4, 2, 8)
    np.testing.assert_allclose(lse, np.full((2, 4), math.log(5)), rtol=0, atol=1e-15)
    # the same row listed twice: z + ln 2
    qb = to_bf16_bits(rng.normal(size=(2, 4, 8)))
    one = oracle.log_partition(qb, K, [4], 2, 4, 2, 8)
    two = oracle.log_partition(qb, K, [4, 4], 2, 4, 2, 8)
    np.testing.assert_allclose(two, one + math.log(2), rtol=0, atol=1e-13)


def test_log_partition_brute_force_and_gqa():
    rng = np.random.default_rng(32)
    T, L, Hq, Hk, d = 15, 2, 4, 2, 8
    K = to_bf16_bits(rng.normal(size=(T, L, Hk, d)) * 2)
    q = to_bf16_bits(rng.normal(size=(L, Hq, d)))
    idx = np.array([0, 3, 4, 9, 14])
    lse = oracle.log_partition(q, K, idx, L, Hq, Hk, d)
    Kf, qf = bf16_bits_to_float(K).astype(np.float64), bf16_bits_to_float(q).astype(np.float64)
    for l in range(L):
        for h in range(Hq):
            z = [float(np.dot(qf[l, h], Kf[t, l, h // (Hq // Hk)])) / math.sqrt(d) for t in idx]
            assert abs(lse[l, h] - math.log(sum(math.exp(v) for v in z))) < 1e-12


def test_log_partition_combines_attention_over_disjoint_sets():
    # softmax over I1 u I2 = (e^{lse1} o1 + e^{lse2} o2) / (e^{lse1} + e^{lse2}); ties O8 to O7
    rng = np.random.default_rng(33)
    T, d = 30, 16
    kb = to_bf16_bits(rng.normal(size=(T, 1, 1, d)) * 2)
    vb = to_bf16_bits(rng.normal(size=(T, 1, 1, d)))
    qb = to_bf16_bits(rng.normal(size=(1, 1, d)))
    perm = rng.permutation(T)
    I1, I2 = np.sort(perm[:11]), np.sort(perm[11:])
    o1 = oracle.attend_one(qb[0, 0], kb[:, 0, 0], vb[:, 0, 0], I1)
    o2 = oracle.attend_one(qb[0, 0], kb[:, 0, 0], vb[:, 0, 0], I2)
    l1 = oracle.log_partition(qb, kb, I1, 1, 1, 1, d)[0, 0]
    l2 = oracle.log_partition(qb, kb, I2, 1, 1, 1, d)[0, 0]
    full = oracle.attend_one(qb[0, 0], kb[:, 0, 0], vb[:, 0, 0], np.arange(T))
    w1, w2 = math.exp(l1), math.exp(l2)
    np.testing.assert_allclose((w1 * o1 + w2 * o2) / (w1 + w2), full, rtol=0, atol=1e-13)
    lf = oracle.log_partition(qb, kb, np.arange(T), 1, 1, 1, d)[0, 0]
    assert abs(lf - math.log(w1 + w2)) < 1e-13


# ----------------------------------------------------------------- O9 -----
# H2O (rule from SPEC h2o_step S:349-357)
def test_h2o_select_spec_examples():
    # scores {0:0.5, 1:0.1, 2:0.4}, window {3,4}, budget 4 -> evict index 1
    sc = np.array([0.5, 0.1, 0.4, 0.0, 0.0])
    assert oracle.h2o_select([0, 1, 2, 3, 4], sc, 5, 0, 2, 4).tolist() == [0, 2, 3, 4]
    # budget >= length -> nothing evicted
    assert oracle.h2o_select([0, 1, 2, 3, 4], sc, 5, 0, 2, 5).tolist() == [0, 1, 2, 3, 4]
    assert oracle.h2o_select([0, 1, 2, 3, 4], sc, 5, 0, 2, 50).tolist() == [0, 1, 2, 3, 4]
    # equal scores at the eviction boundary -> the smaller index is retained
    sc2 = np.array([0.3, 0.2, 0.2, 0.0, 0.0])
    assert oracle.h2o_select([0, 1, 2, 3, 4], sc2, 5, 0, 2, 4).tolist() == [0, 1, 3, 4]
    # the sink is kept whatever its score; evicted tokens never come back
    sc3 = np.array([0.0, 0.9, 0.1, 0.8, 0.0, 0.0, 0.0])
    assert oracle.h2o_select([0, 2, 3, 5, 6], sc3, 7, 1, 2, 4).tolist() == [0, 3, 5, 6]
    # a token leaving the window becomes a candidate with its accumulated score
    assert oracle.h2o_select([0, 2, 5, 6], np.array([0, 0, 0.1, 0, 0, 0.5, 0, 0]), 8, 1, 2, 4).tolist() == [0, 5, 6, 7]


def test_h2o_select_brute_force():
    rng = np.random.default_rng(41)
    for _ in range(300):
        T = int(rng.integers(1, 60))
        prev = np.sort(rng.choice(T, size=int(rng.integers(0, T + 1)), replace=False))
        sc = rng.integers(0, 6, size=T) / 4.0  # many exact ties
        sink, window, budget = int(rng.integers(0, 6)), int(rng.integers(1, 12)), int(rng.integers(0, 40))
        got = oracle.h2o_select(prev, sc, T, sink, window, budget).tolist()
        sp = min(sink, T)
        w0 = max(sp, T - window)
        fixed = set(range(sp)) | set(range(w0, T))
        cand = [t for t in prev.tolist() if sp <= t < w0]
        K = max(0, budget - len(fixed))
        kept = sorted(cand, key=lambda t: (-sc[t], t))[:K]
        assert got == sorted(fixed | set(kept))


def test_h2o_weights_are_averaged_softmax():
    rng = np.random.default_rng(42)
    T, L, Hq, Hk, d = 25, 2, 4, 2, 8
    K = to_bf16_bits(rng.normal(size=(T, L, Hk, d)) * 2)
    q = to_bf16_bits(rng.normal(size=(L, Hq, d)))
    idx = np.sort(rng.choice(T, size=13, replace=False))
    w = oracle.h2o_weights(q, K, idx, L, Hq, Hk, d)
    assert abs(w.sum() - 1.0) < 1e-12 and np.all(w > 0)  # each (l, h) softmax sums to 1
    import torch
    Kf = torch.from_numpy(bf16_bits_to_float(K).astype(np.float64))
    qf = torch.from_numpy(bf16_bits_to_float(q).astype(np.float64))
    ref = torch.zeros(len(idx), dtype=torch.float64)
    for l in range(L):
        for h in range(Hq):
            z = Kf[idx, l, h // (Hq // Hk)] @ qf[l, h] / math.sqrt(d)
            ref += torch.softmax(z, 0)
    np.testing.assert_allclose(w, (ref / (L * Hq)).numpy(), rtol=0, atol=1e-14)
    # q = 0: uniform weights
    w0 = oracle.h2o_weights(to_bf16_bits(np.zeros((L, Hq, d))), K, idx, L, Hq, Hk, d)
    np.testing.assert_allclose(w0, np.full(len(idx), 1 / len(idx)), rtol=0, atol=1e-15)


def test_h2o_with_full_budget_is_full_attention():
    # H2O with budget = total length equals full attention exactly
    rng = np.random.default_rng(43)
    T, d = 30, 8
    kb = to_bf16_bits(rng.normal(size=(T, 1, 1, d)))
    vb = to_bf16_bits(rng.normal(size=(T, 1, 1, d)))
    qb = to_bf16_bits(rng.normal(size=(1, 1, d)))
    prev = np.arange(T - 1)  # retained before the newest token
    idx = oracle.h2o_select(prev, rng.random(T), T, 2, 4, T)
    assert idx.tolist() == list(range(T))
    o = oracle.sparse_decode_attn(qb, kb, vb, idx, 1, 1, 1, d)
    ref = sdpa_fp64(bf16_bits_to_float(qb[0, 0]), bf16_bits_to_float(kb[:, 0, 0]), bf16_bits_to_float(vb[:, 0, 0]))
    np.testing.assert_allclose(o[0, 0], ref, rtol=0, atol=1e-12)


# ---- SPEC simulate_transfer_schedule, the paper's layer pipeline ----------------
def test_transfer_schedule_spec_examples():
    """in [2,2,2] s, compute [3,3,3] s, write-back free -> pipelined 2 + 3*3 = 11 s vs serial 15 s;
    S:292: a single layer -> pipelined == serial; compute all 0 -> total = sum of transfers."""
    from oracle.transfer import simulate_transfer_schedule as sim
    r = sim([2, 2, 2], [3, 3, 3])
    assert r["total_time"] == 11 and r["serial_time"] == 15
    assert r["peak_resident_layers"] <= 2
    r1 = sim([2.5], [4.0], [1.5])
    assert r1["total_time"] == r1["serial_time"] == 8.0
    r0 = sim([1, 2, 3, 4], [0, 0, 0, 0])
    assert r0["total_time"] == 10


def test_transfer_schedule_invariants():
    """Brute-force checks on random models: the greedy schedule never beats either
    bound (the transfer chain, the compute chain), never exceeds serial, keeps at most
    two slices resident, and respects every dependency of the two-stage pipeline."""
    import random
    from oracle.transfer import simulate_transfer_schedule as sim
    rng = random.Random(7)
    for _ in range(300):
        n = rng.randint(1, 12)
        ti = [rng.uniform(0, 5) for _ in range(n)]
        tc = [rng.uniform(0, 5) for _ in range(n)]
        to = [rng.uniform(0, 2) for _ in range(n)]
        r = sim(ti, tc, to)
        eps = 1e-9
        assert r["total_time"] <= r["serial_time"] + eps
        assert r["total_time"] >= sum(ti) + tc[-1] + to[-1] - eps  # in-chain, then the last compute + write-back
        assert r["total_time"] >= ti[0] + sum(tc) - eps             # first transfer, then the compute chain
        assert r["peak_resident_layers"] <= 2
        ev = r["events"]
        for l, in0, in1, c0, c1, o0, o1 in ev:
            assert c0 >= in1 - eps and o0 >= c1 - eps
            if l:
                assert in0 >= ev[l - 1][2] - eps and c0 >= ev[l - 1][4] - eps and o0 >= ev[l - 1][6] - eps
            if l >= 2:
                assert in0 >= ev[l - 2][6] - eps  # the slot of layer l-2 is free
