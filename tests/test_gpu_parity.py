"""GPU parity: libzoomr (through the C-ABI) vs the fp64 CPU oracle, element by element.

Marked `gpu`: run on a B200 with the built libzoomr.so.
"""
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


@pytest.mark.parametrize("seed", [1, 11, 12])
def test_tiny_end_to_end(seed):
    inp = S.generate(S.CONFIGS["tiny"], device="cuda", seed=seed)
    st = PY.make_step(inp)
    PY.run_full(inp, st)
    rep = {}
    PY.check_sequence(inp, st, 0, rep)


@pytest.mark.parametrize("query", ["planted", "diffuse"])
def test_tiny_batched_variants(query):
    import dataclasses
    cfg = dataclasses.replace(S.CONFIGS["tiny"], batch=5)
    inp = S.generate(cfg, device="cuda", seed=21, query_mode=query)
    st = PY.make_step(inp)
    PY.run_full(inp, st)
    rep = {}
    for b in range(5):
        PY.check_sequence(inp, st, b, rep)


def test_8b16k_end_to_end():
    inp = S.generate(S.CONFIGS["8b16k"], device="cuda")
    st = PY.make_step(inp, capacity=8192)
    PY.run_full(inp, st)
    rep = {}
    PY.check_sequence(inp, st, 0, rep)
    print(rep)
