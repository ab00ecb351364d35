"""Host logic of bench.py (no GPU): the algorithmic byte count of SURVEY 8(d), the
percentiles, and that both arms describe the workload with the same `config`."""
import argparse
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_algorithmic_bytes_match_survey_formula(bench):
    """a5 = |I_f| L H_kv d 2 2 + q + fp32 out + index; a2 = N_t L H_kv d 4 + q;
    a1 = |S| L H_kv d 2 + L H_kv d 4.  Appendix A: C2 at |I_f| = 2836 is 389 MB per step."""
    import zoomr_synth as S
    cfg = S.CONFIGS["8b16k"]
    by = bench.algorithmic_bytes(cfg, [2836], [120])
    assert by["a5"] == 2836 * 32 * 8 * 128 * 4 + 32 * 32 * 128 * (2 + 4) + 2836 * 4
    assert by["a2"] == 120 * 32 * 8 * 128 * 4 + 32 * 32 * 128 * 2
    assert by["a1"] == 16 * 32 * 8 * 128 * 2 + 32 * 8 * 128 * 4
    assert abs(by["total"] / 1e6 - 389) < 1.5
    # U > 1 steps without a closure: a5 + a4 only
    light = bench.algorithmic_bytes(cfg, [2836], [0], closures=0)
    assert light["a1"] == 0 and light["a2"] == 32 * 32 * 128 * 2


def test_percentiles(bench):
    xs = list(range(1, 101))
    p = bench.pcts(xs)
    assert p["p50"] == pytest.approx(50.5) and p["p10"] == pytest.approx(10.9) and p["p90"] == pytest.approx(90.1)
    assert bench.pct([], 0.5) is None and bench.pct([3.0], 0.9) == 3.0


def test_both_arms_share_the_config(bench):
    import zoomr_synth as S
    args = argparse.Namespace(query="planted", rotate=4)
    cfg = S.CONFIGS["8b16k"]
    ours = bench.workload_config(cfg, args, 1, 1, 120)
    ref = bench.workload_config(cfg, args, 1, 1, 120)
    assert ours == ref and ours["workload"] == "8b16k" and ours["global_batch"] == 1
    assert "inputs larger than L2" in ours["l2"]
    assert bench.workload_config(cfg, args, 4, 1, 120)["parallelism"] == "batch-shard x4"
