"""a3 through the C-ABI on given (v, A): flags and the agreeability AG against the
oracle's O5 (AG = sum_{i in I_c} v_i / sum_{j in I_all} v_j;
SPEC agreeability S:205-213).

Both sides get the same integer votes and the same A: the GPU's fixed-point A
(int64, units of 2^-32, reading Q2') and the oracle's fp64 A = that integer /
2^32, exact.  So flags must be bit-exact (the order (v desc, A desc, i asc) is
total) and AG must equal the oracle's value rounded to fp32 -- the kernel
divides the two integer vote sums in fp64 and rounds once."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    from paper_2604_10898_b200 import _build
    _build.build()


def _gpu_topc(votes_list, A_list, c, ms=None):
    """Run zoomr_select_topc on a batch of (votes, A-fixed-point) rows."""
    from paper_2604_10898_b200 import zoomr as Z
    B = len(votes_list)
    ms = ms or max(1, max(len(v) for v in votes_list))
    partial = torch.zeros(B, 2, ms, dtype=torch.int64)
    nsum = torch.zeros(B, dtype=torch.int32)
    for b, (v, a) in enumerate(zip(votes_list, A_list)):
        n = len(v)
        partial[b, 0, :n] = torch.as_tensor(np.asarray(v, np.int64))
        partial[b, 1, :n] = torch.as_tensor(np.asarray(a, np.int64))
        nsum[b] = n
    partial, nsum = partial.cuda(), nsum.cuda()
    flags = torch.full((B, ms), 9, dtype=torch.uint8, device="cuda")
    ag = torch.full((B,), -1.0, dtype=torch.float32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    Z.select_topc(partial, nsum, c, flags, ag, st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    return flags.cpu().numpy(), ag.cpu().numpy()


def _check(votes_list, A_list, c):
    flags, ag = _gpu_topc(votes_list, A_list, c)
    for b, (v, a) in enumerate(zip(votes_list, A_list)):
        n = len(v)
        f_ref, ag_ref, _ = oracle.select_topc(np.asarray(v, np.int64), np.asarray(a, np.float64) / 2.0 ** 32, c)
        assert np.array_equal(flags[b, :n], f_ref), f"seq {b}: flags"
        assert ag[b] == np.float32(ag_ref), f"seq {b}: AG {ag[b]} vs {ag_ref}"
    return flags, ag


def test_spec_example_s211():
    """SPEC S:211 (P:244's formula): v = {1:3, 2:2, 3:2, 4:1}, I_c = {1, 2} (c = 2,
    the v=2 tie broken by A) -> AG = 5/8; |I_all| = 1 -> 1.0; S:213:
    v = {1:2, 2:2}, c = 1 -> 0.5.  Summary 0 carries no vote here (indices are
    SPEC's 1-based names)."""
    one = 1 << 32
    v = [0, 3, 2, 2, 1]
    a = [0, 3 * one, 5 * one, 4 * one, one]
    flags, ag = _check([v], [a], 2)
    assert flags[0, :5].tolist() == [0, 2, 2, 1, 1]
    assert ag[0] == np.float32(5 / 8)
    _, ag = _check([[0, 0, 4, 0]], [[0, 0, one, 0]], 3)
    assert ag[0] == 1.0
    _, ag = _check([[2, 2]], [[one, one]], 1)  # exact tie in v and A: the older summary wins
    assert ag[0] == 0.5


def test_exact_ties_and_degenerate():
    one = 1 << 32
    # every summary tied in (v, A): I_c = the c oldest, AG = c / n
    n = 37
    flags, ag = _check([[3] * n], [[7 * one] * n], 5)
    assert flags[0, :n].tolist() == [2] * 5 + [1] * (n - 5)
    assert ag[0] == np.float32(5 / n)
    # c = 0: I_c empty, AG = 0; no votes at all: AG = 0, nothing kept
    _, ag = _check([[1, 2, 3]], [[one, one, one]], 0)
    assert ag[0] == 0.0
    flags, ag = _check([[0, 0, 0]], [[0, 0, 0]], 2)
    assert flags[0, :3].tolist() == [0, 0, 0] and ag[0] == 0.0
    # negative A (alpha sums can be negative) ordering
    _check([[4, 4, 4, 1]], [[-5 * one, -one, -3 * one, 9 * one]], 2)


@pytest.mark.parametrize("n", [8, 120, 511, 600, 1631, 4000])
def test_random_cases(n):
    """Random votes with many duplicates and random fixed-point A (ties in v common,
    exact ties in A planted): the <= 512 direct-ranking path and the vote-histogram
    + tie-group path of block_topc."""
    rng = np.random.default_rng(n)
    vl, al, cs = [], [], []
    for _ in range(6):
        v = rng.integers(0, 6, n) * (rng.random(n) < 0.6)
        a = rng.integers(-(1 << 40), 1 << 40, n)
        dup = rng.random(n) < 0.2
        a[dup] = 12345 << 20  # exact A ties inside equal-vote groups
        vl.append(v.tolist())
        al.append(a.tolist())
    for c in (1, 4, 32):
        _check(vl, al, c)
