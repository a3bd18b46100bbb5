"""Prefetch pipeline (reference data_plane/pipeline.py semantics): W workers ahead of one consumer
through a bounded queue, in-order delivery, failures surfaced, stall log."""

import threading
import time

import numpy as np
import pytest

from paper_1810_01993_b200.pipeline import PipelineError, PrefetchPipeline


def test_in_order_and_bounded():
    made = []
    lock = threading.Lock()

    def make(step):
        time.sleep(0.002 * (step % 3))        # workers finish out of order
        with lock:
            made.append(step)
        return (np.full(4, step, np.float32),)

    p = PrefetchPipeline(make, steps=40, workers=4, capacity=3, pin=False)
    got = [int(x[0][0]) for x in p]
    assert got == list(range(40))
    assert sorted(made) == list(range(40))
    assert p.log.max_in_flight <= 3
    assert len(p.log.items) == 40


def test_worker_failure_surfaces():
    def make(step):
        if step == 5:
            raise RuntimeError("bad tile")
        return (np.zeros(2, np.float32),)

    p = PrefetchPipeline(make, steps=10, workers=2, capacity=2, pin=False)
    with pytest.raises(PipelineError):
        for _ in p:
            pass


def test_stall_fraction_reflects_slow_producer():
    p = PrefetchPipeline(lambda s: (time.sleep(0.01) or np.zeros(1, np.float32),), steps=12, workers=1,
                         capacity=2, pin=False)
    for _ in p:
        pass
    assert 0.5 < p.log.stall_fraction(skip=1) <= 1.0
    assert p.log.to_csv().startswith("index,wait_seconds,timestamp\n")


def test_rejects_bad_config():
    with pytest.raises(ValueError):
        PrefetchPipeline(lambda s: (), steps=1, workers=0)
