"""Input side: a bounded prefetch pipeline of host batches (reference data_plane/pipeline.py:61-118).

Same contract as the reference's `pipeline_run`: W reader workers run ahead of one consumer and
meet it only at a bounded queue of `capacity` items; worker failures surface as PipelineError
after the feed drains; a log records how long the consumer waited for each item (post-warm-up
stall fraction).  Differences that matter on a B200 node:

  * items are delivered in step order (worker w produces steps w, w+W, ...; the consumer takes
    step t when it is ready), so a data-parallel run stays bitwise reproducible;
  * each item is placed in pinned host memory by the worker, so the trainer's `stage()` can
    copy it to the device asynchronously on a copy stream under the running step.

The throughput benchmark does not use it (its scenes are generated on the GPU,
scenes.device_scene_pool); it is the path for CPU-generated or file-backed inputs.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch


class PipelineError(Exception):
    pass


@dataclass
class PipelineLog:
    items: list = field(default_factory=list)   # (step, wait_seconds, dequeue_timestamp)
    workers: int = 0
    capacity: int = 0
    max_in_flight: int = 0

    def stall_fraction(self, skip: int = 0) -> float:
        """Waited time / elapsed time over the items after the first `skip`."""
        tail = self.items[skip:]
        if not tail:
            return 0.0
        waited = sum(w for _, w, _ in tail)
        start = tail[0][2] - tail[0][1]
        elapsed = tail[-1][2] - start
        return waited / elapsed if elapsed > 0 else 0.0

    def to_csv(self) -> str:
        return "index,wait_seconds,timestamp\n" + "".join(
            f"{i},{w:.6f},{ts:.6f}\n" for i, (_, w, ts) in enumerate(self.items))


class PrefetchPipeline:
    """Iterate `make_item(step)` for step in range(steps), W workers ahead, at most `capacity`
    finished-but-unconsumed items (+ W in progress).  Items are tuples of NumPy arrays; with
    pin=True they are returned as pinned CPU torch tensors."""

    def __init__(self, make_item, steps: int, workers: int = 4, capacity: int = 4, pin: bool = True):
        if capacity < 1 or workers < 1 or steps < 0:
            raise ValueError("capacity and workers must be positive")
        self.make_item, self.steps, self.workers, self.capacity, self.pin = make_item, steps, workers, capacity, pin
        self.log = PipelineLog(workers=workers, capacity=capacity)
        self._ready = {}
        self._next = 0          # next step the consumer takes
        self._failure = None
        self._cv = threading.Condition()
        self._threads = [threading.Thread(target=self._work, args=(w,), daemon=True, name=f"reader-{w}")
                         for w in range(workers)]
        for t in self._threads:
            t.start()

    def _convert(self, item):
        if not self.pin:
            return item
        return tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in item)

    def _work(self, w):
        try:
            for step in range(w, self.steps, self.workers):
                with self._cv:   # bounded: do not run more than `capacity` steps ahead
                    self._cv.wait_for(lambda: step - self._next < self.capacity or self._failure is not None)
                    if self._failure is not None:
                        return
                item = self._convert(self.make_item(step))
                with self._cv:
                    self._ready[step] = item
                    self.log.max_in_flight = max(self.log.max_in_flight, len(self._ready))
                    self._cv.notify_all()
        except Exception as exc:  # noqa: BLE001 -- surfaced to the consumer
            with self._cv:
                self._failure = PipelineError(f"reader worker {w} failed: {exc!r}")
                self._cv.notify_all()

    def __iter__(self):
        for step in range(self.steps):
            t0 = time.monotonic()
            with self._cv:
                self._cv.wait_for(lambda: step in self._ready or self._failure is not None)
                if step not in self._ready:
                    raise self._failure
                item = self._ready.pop(step)
                self._next = step + 1
                self._cv.notify_all()
            now = time.monotonic()
            self.log.items.append((step, now - t0, now))
            yield item
        for t in self._threads:
            t.join()
