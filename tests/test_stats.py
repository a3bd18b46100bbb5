"""Throughput statistics (stats.py) against the reference's own sustained_stats outputs
(tests/golden/stats.npz, made by tests/golden/make_golden.py from deskdl/harness/stats.py:58-79)
and the oracle restatement; these are the numbers bench.py reports under "stats"."""

import os

import numpy as np
import pytest

from oracle import deskdl_port as O
from paper_1810_01993_b200.stats import StepRecord, sustained_stats, weak_scaling_efficiency

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _records(rates):
    return [StepRecord(step=t + 1, rates=tuple(r), wall=1.0 / float(np.mean(r)), loss=0.0)
            for t, r in enumerate(rates)]


def test_sustained_stats_match_reference_golden():
    d = np.load(os.path.join(G, "stats.npz"))
    for i in range(5):
        rates, warm = d[f"s{i}_rates"], int(d[f"s{i}_warmup"])
        st = sustained_stats(_records(rates), per_sample_flops=1.5e12, warmup=warm)
        got = np.array([st.median, st.p16, st.p84, st.world, st.steps, st.flops_per_s, st.global_rate])
        assert np.array_equal(got, d[f"s{i}_result"]), (i, got, d[f"s{i}_result"])
        med, p16, p84 = O.sustained(rates, warmup=warm)
        assert (med, p16, p84) == (st.median, st.p16, st.p84)


def test_sustained_stats_validation_and_scaling():
    with pytest.raises(ValueError):
        sustained_stats([])
    with pytest.raises(ValueError):
        sustained_stats([StepRecord(1, (1.0, 2.0), 1.0, 0.0), StepRecord(2, (1.0,), 1.0, 0.0)])
    with pytest.raises(ValueError):
        StepRecord(1, (), 1.0, 0.0)
    eff = weak_scaling_efficiency({1: 50.0, 2: 49.0, 8: 45.0})
    assert eff == {1: 1.0, 2: 0.98, 8: 0.9}
    with pytest.raises(ValueError):
        weak_scaling_efficiency({2: 1.0})
