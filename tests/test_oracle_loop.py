"""Pins of the oracle's Algorithm-1 loop bookkeeping (oracle/loop.py) against
SPEC's worked examples (ingest_token S:36-45, decode_step S:421-427)."""
import numpy as np

import oracle
from oracle.loop import OracleLoop

BEGIN, END, DOT = 1000, 1001, 200


def _loop(n_p, L=1, Hq=2, Hkv=1, d=4, sink=4, window=8):
    rng = np.random.default_rng(0)
    rows = lambda n: [np.asarray(rng.integers(0x3e00, 0x4000, (L, Hkv, d)), np.uint16) for _ in range(n)]
    k, v = rows(n_p), rows(n_p)
    return OracleLoop(L, Hq, Hkv, d, 1, 1, sink, window, BEGIN, END, (DOT,), k, v), rng


def _row(rng, L=1, Hkv=1, d=4):
    return np.asarray(rng.integers(0x3e00, 0x4000, (L, Hkv, d)), np.uint16)


def _q(rng, L=1, Hq=2, d=4):
    return np.asarray(rng.integers(0x3e00, 0x4000, (L, Hq, d)), np.uint16)


def test_delimiters_give_the_spec_example_segments():
    """10 tail tokens [30, 40) before <|begin_of_summary|> at 40 and
    <|end_of_summary|> at 45 -> R_i = [30, 40), S_i = [40, 46)."""
    oracle.build()
    lp, rng = _loop(30)
    for t in range(30, 46):
        tok = BEGIN if t == 40 else END if t == 45 else 7
        r = lp.step(_row(rng), _row(rng), _q(rng), tok)
    assert r["closed"] == 0
    assert r["segs"].tolist() == [[30, 40, 40, 46]]
    assert lp.tail == 46 and lp.open == -1


def test_boundary_with_no_summaries_is_streaming():
    """boundary token with N_t = 0 -> I_f = prompt (sink) u window."""
    oracle.build()
    lp, rng = _loop(20, sink=4, window=8)
    r = lp.step(_row(rng), _row(rng), _q(rng), DOT)
    T = 21
    assert r["update"] and r["index"].tolist() == list(range(4)) + list(range(T - 8, T))


def test_non_boundary_keeps_the_flags():
    """a non-boundary token does not recompute the selection."""
    oracle.build()
    lp, rng = _loop(10)
    for tok in [7] * 4 + [BEGIN, 7, 7, END] + [DOT]:
        r = lp.step(_row(rng), _row(rng), _q(rng), tok)
    assert r["update"] and r["flags"].shape == (1,)
    held = r["flags"].copy()
    for tok in [7, 7, BEGIN, 7, END, 7]:
        r = lp.step(_row(rng), _row(rng), _q(rng), tok)
        assert not r["update"]
        assert np.array_equal(r["flags"][:1], held) and (r["flags"][1:] == 0).all()
