"""Synchronous data-parallel training step (pkg/src/deskdl/harness/trainer.py:343-421), B200-native.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch for the gradient
exchange.  Per step and rank:
  batch -> forward (fused convs + fused weighted CE) -> backward
  -> bucketed all-reduce(sum) of the flat fp32 gradient buffer, issued per
     bucket while backward is still running (buckets in reverse parameter
     order; each fires when the wgrad of its last parameter is enqueued)
  -> multi-tensor LARC + momentum update with the 1/P mean folded in
  -> repack bf16 operand copies of the weights.
Lag 1 applies the previous step's reduced gradients (trainer.py:378-383,
403-405); the current reduction then overlaps the next step's compute.

The reference's control plane (readiness tree, control_plane.py) only exists to
give every rank the same collective order; here the bucket order is static, so
the order is identical by construction.  NCCL results are bitwise identical on
all ranks, which the step-{1,10,end} weight digests check (trainer.py:263-315).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, nhwc
from .flops import count_graph, train_flops_per_sample
from .loss import ClassWeights, uniform_weights
from .models import NetConfig
from .net import SegmentationNet
from .optimizer import OptimConfig
from .scenes import SceneConfig, generated_batch
from .stats import StepRecord, sustained_stats


class TrainingError(Exception):
    pass


def param_digest(params: dict, order) -> str:
    """SHA-256 over (name, shape, fp32 bytes) in parameter order (trainer.py:263-270)."""
    h = hashlib.sha256()
    for name in order:
        v = np.ascontiguousarray(params[name], dtype=np.float32)
        h.update(name.encode())
        h.update(str(v.shape).encode())
        h.update(v.tobytes())
    return h.hexdigest()


class DataParallelTrainer:
    def __init__(self, net: SegmentationNet, optim: OptimConfig, input_shape, lag: int = 0,
                 class_weights=None, bucket_mb: float = 32.0, group=None, hierarchy=None):
        """hierarchy = (groups, per_group): reduce each bucket in the paper's three stages
        (collectives.py:157-200 hybrid_allreduce): reduce-scatter inside each group of per_group
        consecutive ranks, all-reduce of the shards across groups, all-gather inside the group --
        the 2x4 split-communicator mirror of the reference's hierarchical all-reduce.  None: one
        NCCL all-reduce per bucket (on one NVSwitch node that is the whole of stage 1)."""
        if lag not in (0, 1):
            raise ValueError("lag must be 0 or 1")
        self.net = net
        self.optim = optim
        self.lag = lag
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.eng = net.engine(input_shape)
        eng = self.eng
        cw = uniform_weights(net.cfg.classes) if class_weights is None else class_weights
        eng.set_class_weights(cw)
        self.ntensors = len(net.param_order)
        self.lr_out = torch.zeros(self.ntensors, dtype=torch.float32, device=eng.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=eng.device)
        self.g_other = torch.zeros_like(eng.flat_g) if lag == 1 else None
        self.have_prev = False
        self._make_buckets(bucket_mb)
        # one batched split-K reduction per bucket (a single one on one GPU)
        eng.set_buckets(self.buckets if self.world > 1 else [list(net.param_order)])
        self._works = []
        self.steps_done = 0
        self.hier = None
        if hierarchy is not None and self.world > 1:
            ng, per = hierarchy
            if ng * per != self.world or 64 % per:
                raise ValueError(f"hierarchy {hierarchy} does not tile {self.world} ranks (per_group must divide 64)")
            rank = dist.get_rank()
            local = cross = None
            for gi in range(ng):   # every rank creates every group, in the same order
                grp = dist.new_group([gi * per + j for j in range(per)])
                if rank // per == gi:
                    local = grp
            for j in range(per):
                grp = dist.new_group([gi * per + j for gi in range(ng)])
                if rank % per == j:
                    cross = grp
            self.hier = (local, cross, per, rank % per)
            self.comm_stream = torch.cuda.Stream(device=eng.device)

    def _make_buckets(self, bucket_mb: float):
        """Contiguous parameter ranges of >= bucket_mb, formed from the end of param order
        (the order backward produces gradients); static, hence identical on every rank."""
        eng = self.eng
        limit = int(bucket_mb * 2 ** 20 / 4)
        self.buckets = []
        cur, size = [], 0
        for name in reversed(self.net.param_order):
            cur.append(name)
            size += int(np.prod(eng.slot[name][1]))
            if size >= limit:
                self.buckets.append(cur)
                cur, size = [], 0
        if cur:
            self.buckets.append(cur)
        self.bucket_of = {n: i for i, b in enumerate(self.buckets) for n in b}
        self.bucket_range = []
        for b in self.buckets:
            lo = min(eng.slot[n][0] for n in b)
            hi = max(eng.slot[n][0] + (int(np.prod(eng.slot[n][1])) + 63) // 64 * 64 for n in b)
            self.bucket_range.append((lo, hi))

    # ------------------------------------------------------------------ comm
    def _start_bucket(self, i):
        lo, hi = self.bucket_range[i]
        if getattr(self, "hier", None) is None:
            w = dist.all_reduce(self.eng.flat_g[lo:hi], op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            self._works.append(w)
            return
        # three stages on a communication stream (bucket bounds are 64-float aligned, so the
        # bucket splits evenly into per_group shards; in-place NCCL reduce-scatter / all-gather)
        local, cross, per, me = self.hier
        buf = self.eng.flat_g[lo:hi]
        shard = buf.view(per, -1)[me]
        cs = self.comm_stream
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            dist.reduce_scatter_tensor(shard, buf, op=dist.ReduceOp.SUM, group=local, async_op=True).wait()
            dist.all_reduce(shard, op=dist.ReduceOp.SUM, group=cross, async_op=True).wait()
            w = dist.all_gather_into_tensor(buf, shard, group=local, async_op=True)
        self._works.append(w)

    def _backward_with_overlap(self):
        if self.world == 1:
            self.eng.backward()
            return
        self.eng.backward(on_bucket_ready=self._start_bucket)

    def _wait_comm(self):
        for w in self._works:
            w.wait()
        self._works = []

    # ------------------------------------------------------------------ update
    def _apply(self, g):
        eng = self.eng
        o = self.optim
        # LARC + momentum update; the same pass writes the bf16 weight mirror the convs read
        with _lib.use(eng.half):   # the mirror is written in the engine's 16-bit type
            nhwc.larc_update(eng.flat_w, eng.flat_m, g, eng.offsets, o.lr, o.momentum, o.trust, o.weight_decay,
                             o.eps, 1.0 / (self.world * eng.loss_scale), self.lr_out, self.status, eng.ws,
                             w_bf16=None if eng.fp32 else eng.flat_wbf)
        eng.launches += 3
        eng.repack(mirror=False)

    def capture(self, x: torch.Tensor, labels: torch.Tensor, timed: bool = False, buffers: int = 1):
        """Record one whole training step (every launch, and on N GPUs the bucket all-reduces)
        into a CUDA graph over static input buffers; later `step` calls copy the batch in and
        replay it.  `timed` adds graph event nodes around every conv launch (roofline timing).
        `buffers` = 2 records a second graph over a second input buffer pair, so `stage` can
        copy the next batch from the host while the current step runs (`step_staged`).
        Call after at least one eager step (workspaces sized).

        Lag 1 (trainer.py:378-383): two graphs over the two gradient buffers, replayed
        alternately -- graph k computes into one buffer while it applies the other's (already
        reduced) gradients, so the LARC update never waits on this step's all-reduce; the
        collective is joined at the end of its own graph (a captured graph cannot leave a stream
        forked), which still overlaps it with the update.  With buffers = 2 the input buffer
        alternates with the same period."""
        eng = self.eng
        if self.lag == 1 and not self.have_prev:
            raise RuntimeError("lag-1 capture needs one eager step first (a pending gradient)")
        self.static_xs = [torch.empty_like(x) for _ in range(buffers)]
        self.static_ls = [torch.empty_like(labels) for _ in range(buffers)]
        for sx, sl in zip(self.static_xs, self.static_ls):
            sx.copy_(x)
            sl.copy_(labels)
        self.static_x, self.static_l = self.static_xs[0], self.static_ls[0]
        torch.cuda.synchronize()
        self._wait_comm()
        self.graphs = []
        ngraphs = 2 if self.lag == 1 else buffers
        self._capturing = True
        self._replays = 0
        steps0 = self.steps_done
        for k in range(ngraphs):
            graph = torch.cuda.CUDAGraph()
            launches0 = eng.launches
            t = timed and k == 0
            eng.conv_timing, eng.conv_events, eng.graph_events = t, [], t
            with torch.cuda.graph(graph):
                self._eager_step(self.static_xs[k % buffers], self.static_ls[k % buffers])
            eng.graph_events = False
            if k == 0:
                self.graph_conv_events = eng.conv_events if t else []
                self.graph_launches = eng.launches - launches0
            eng.conv_timing, eng.conv_events = False, []
            self.graphs.append(graph)
        self._capturing = False
        self.steps_done = steps0   # capturing ran no step
        self.graph = self.graphs[0]
        self.copy_stream = torch.cuda.Stream(device=eng.device)
        self._ready = [torch.cuda.Event() for _ in range(buffers)]
        self._consumed = [torch.cuda.Event() for _ in range(buffers)]
        for e in self._consumed:
            e.record()
        self._stage_k, self._staged = 0, []
        torch.cuda.synchronize()

    def step(self, x: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """One training step on device-resident inputs; returns the device loss (no host sync)."""
        g = getattr(self, "graph", None)
        if g is not None:
            k = self._next_graph()
            sx, sl = self.static_xs[k % len(self.static_xs)], self.static_ls[k % len(self.static_ls)]
            if x.data_ptr() != sx.data_ptr():
                sx.copy_(x, non_blocking=True)
            if labels.data_ptr() != sl.data_ptr():
                sl.copy_(labels, non_blocking=True)
            self._replay(k)
            self._consumed[k % len(self._consumed)].record()
            return self.eng.loss
        return self._eager_step(x, labels)

    def _next_graph(self) -> int:
        return self._replays % len(self.graphs) if self.lag == 1 else 0

    def _replay(self, k: int):
        self.graphs[k].replay()
        self._replays += 1
        if self.lag == 1:   # mirror the captured buffer swap: flat_g = the buffer just computed
            self.eng.flat_g, self.g_other = self.g_other, self.eng.flat_g
        self.eng.launches += self.graph_launches
        self.steps_done += 1

    def stage(self, hx: torch.Tensor, hl: torch.Tensor):
        """Asynchronously copy a host batch (pinned) into the next free input buffer on a copy
        stream -- it overlaps the step that is running (needs capture(buffers=2))."""
        k = self._stage_k
        cs = self.copy_stream
        cs.wait_event(self._consumed[k])          # that buffer's previous step has read it
        with torch.cuda.stream(cs):
            self.static_xs[k].copy_(hx, non_blocking=True)
            self.static_ls[k].copy_(hl, non_blocking=True)
            self._ready[k].record()
        self._staged.append(k)
        self._stage_k = (k + 1) % len(self.static_xs)

    def step_staged(self) -> torch.Tensor:
        """Run the training step on the oldest staged batch; returns the device loss."""
        k = self._staged.pop(0)
        torch.cuda.current_stream().wait_event(self._ready[k])
        g = self._next_graph() if self.lag == 1 else k
        if self.lag == 1 and g % len(self.static_xs) != k:
            raise RuntimeError("lag-1 staged replay out of phase with its input buffer")
        self._replay(g)
        self._consumed[k].record()
        return self.eng.loss

    def graph_conv_totals(self, by_pass=False):
        """(ms, FLOPs) of the conv launches of the most recent replay of a timed graph
        (by_pass: {fprop|dgrad|wgrad: (ms, FLOPs)})."""
        from .engine import conv_event_totals
        torch.cuda.synchronize()
        return conv_event_totals(self.graph_conv_events, by_pass)

    def _eager_step(self, x: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        eng = self.eng
        eng.set_batch(x, labels)
        eng.forward()
        if self.lag == 0:
            self._backward_with_overlap()
            self._wait_comm()
            self._apply(eng.flat_g)
        else:
            # the previous step's reduction finishes under this step's compute
            self._backward_with_overlap_lag1()
        self.steps_done += 1
        return eng.loss

    def _backward_with_overlap_lag1(self):
        eng = self.eng
        prev_works = self._works
        self._works = []
        # this step's gradients go to the other buffer; the previous one is applied
        g_prev = eng.flat_g
        eng.flat_g = self.g_other
        self.g_other = g_prev
        self._backward_with_overlap()
        for w in prev_works:
            w.wait()
        if self.have_prev:
            self._apply(g_prev)
        self.have_prev = True
        if getattr(self, "_capturing", False):
            self._wait_comm()   # join this step's collectives inside its own graph

    def finish(self):
        """Lag 1: apply the last step's reduced gradients (trainer.py:403-405)."""
        self._wait_comm()
        if self.lag == 1 and self.have_prev:
            self._apply(self.eng.flat_g)
            self.have_prev = False

    # ------------------------------------------------------------------ run state (resume)
    def export_state(self) -> dict:
        """Weights, momentum, the reduced gradient a lag-1 run has yet to apply, and counters
        (reference-layout NumPy tensors; see checkpoint.save_train_state)."""
        self._wait_comm()
        torch.cuda.synchronize()
        eng = self.eng
        pending = self.lag == 1 and self.have_prev
        # the pending lag-1 gradient is the rank SUM (the 1/P is applied in the update): export
        # the mean so the state is independent of the number of ranks that wrote it
        return {"params": eng.export_params(), "momentum": eng._export(eng.flat_m),
                "lag_grad": ({k: v / np.float32(self.world * eng.loss_scale) for k, v in eng._export(eng.flat_g).items()}
                             if pending else None),
                "steps": self.steps_done, "have_prev": bool(pending), "world": self.world}

    def import_state(self, st: dict):
        eng = self.eng
        self._wait_comm()
        eng.load_params(st["params"])             # also refreshes the bf16 weight mirror
        eng.import_flat(eng.flat_m, st["momentum"])
        if st.get("have_prev"):
            if self.lag != 1:
                raise ValueError("state carries a pending lag-1 gradient but the trainer has lag 0")
            # mean -> this run's rank sum (bitwise when the world sizes match: x / P * P with P a
            # power of two is exact)
            eng.import_flat(eng.flat_g, {k: np.asarray(v, np.float32) * np.float32(self.world * eng.loss_scale)
                                         for k, v in st["lag_grad"].items()})
        self.have_prev = bool(st.get("have_prev")) and self.lag == 1
        self.steps_done = int(st.get("steps", 0))
        self.net._params = eng.export_params()
        torch.cuda.synchronize()

    def release_graph(self):
        """Drop the captured step graph (it references NCCL communicators: release it before the
        process group is destroyed)."""
        if getattr(self, "graph", None) is not None:
            torch.cuda.synchronize()
            for g in self.graphs:
                g.reset()
            self.graph, self.graphs = None, []

    def check_status(self):
        self.check_labels()
        if int(self.status.item()):
            raise FloatingPointError("non-finite norm in LARC")

    def check_labels(self):
        """ValueError if the last step's labels were outside [0, classes) (loss.py:72-74)."""
        if int(self.eng.label_status.item()):
            raise ValueError(f"labels outside [0, {self.eng.plan.classes})")

    def digest(self) -> str:
        return param_digest(self.eng.export_params(), self.net.param_order)

    def hash_sync(self, step: int) -> str:
        d = self.digest()
        if self.world > 1:
            got = [None] * self.world
            dist.all_gather_object(got, d, group=self.group)
            bad = {r: x for r, x in enumerate(got) if x != got[0]}
            if bad:
                raise TrainingError(f"weights diverged at step {step}: " +
                                    "; ".join(f"rank {r}: {x[:12]}" for r, x in sorted(bad.items())))
        return d


@dataclass(frozen=True)
class RunConfig:
    """Training run description (reference harness/config.py:39-157, single-node subset)."""
    lag: int = 0
    steps: int = 10
    local_batch: int = 1
    seed: int = 0
    optim: OptimConfig = field(default_factory=OptimConfig)
    net: object = field(default_factory=NetConfig)
    scene: SceneConfig = field(default_factory=SceneConfig)
    class_weighting: str = "inv_sqrt"
    hash_steps: tuple = ()
    precision: str = "bf16"   # "fp16": IEEE-half storage (libb2dl_f16.so); "fp32": the parity mode (group 3)
    hierarchy: tuple | None = None   # (groups, per_group): three-stage hierarchical all-reduce
    prefetch_workers: int = 0        # > 0: scenes made by a W-worker bounded prefetch pipeline
    prefetch_capacity: int = 4

    def __post_init__(self):
        if self.lag not in (0, 1):
            raise ValueError("lag must be 0 or 1")
        if self.local_batch < 1 or self.steps < 1:
            raise ValueError("local_batch and steps must be positive")
        if self.class_weighting not in ("inv_sqrt", "uniform"):
            raise ValueError("class_weighting must be inv_sqrt or uniform")
        if self.net.channels_in != self.scene.channels:
            raise ValueError("net input channels != scene channels")


@dataclass
class TrainResult:
    records: list
    stats: object
    losses: list
    digests: list
    state: dict


def model_flops_per_sample(net: SegmentationNet, shape) -> float:
    n, c, h, w = shape
    shapes = {k: v.shape for k, v in net._params.items()}
    shapes.update(x=(n, c, h, w), labels=(n, h, w), class_weights=(net.cfg.classes,))
    return train_flops_per_sample(count_graph(net.graph, shapes, batch=n))


def train_run(cfg: RunConfig, net_cls=None) -> TrainResult:
    """This rank's loop of a synchronous data-parallel run (trainer.py:343-476).

    Call from every rank (torchrun); with no process group it is a 1-rank run.
    Returns per-step records with the rank-mean rates (device-timed)."""
    from .net import DeepLabV3Plus, MiniDenseNet
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if net_cls is None:
        net_cls = MiniDenseNet if isinstance(cfg.net, NetConfig) else DeepLabV3Plus
    net = net_cls(cfg.net, seed=cfg.seed, precision=cfg.precision)
    sc = cfg.scene
    shape = (cfg.local_batch, sc.channels, sc.height, sc.width)
    cw = (uniform_weights(cfg.net.classes) if cfg.class_weighting == "uniform"
          else ClassWeights(sc.frequencies).vector())
    tr = DataParallelTrainer(net, cfg.optim, shape, lag=cfg.lag, class_weights=cw, hierarchy=cfg.hierarchy)
    hash_at = {1, 10, cfg.steps} | set(cfg.hash_steps)
    records, losses, digests = [], [], []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    feed = None
    if cfg.prefetch_workers > 0:   # pinned host batches, step order, W workers ahead
        from .pipeline import PrefetchPipeline
        feed = iter(PrefetchPipeline(lambda t: generated_batch(sc, cfg.seed, t, rank, cfg.local_batch), cfg.steps,
                                     workers=cfg.prefetch_workers, capacity=cfg.prefetch_capacity))
    for t in range(cfg.steps):
        if feed is not None:
            hx, hl = next(feed)
            xd = hx.cuda(non_blocking=True)
            ld = hl.cuda(non_blocking=True)
        else:
            x, lab = generated_batch(sc, cfg.seed, t, rank, cfg.local_batch)
            xd = torch.from_numpy(x).cuda(non_blocking=True)
            ld = torch.from_numpy(lab).cuda(non_blocking=True)
        ev0.record()
        loss = tr.step(xd, ld)
        ev1.record()
        ev1.synchronize()
        wall = ev0.elapsed_time(ev1) / 1e3
        lv = float(loss.item())
        if not math.isfinite(lv):
            tr.check_labels()
            raise TrainingError(f"rank {rank}: non-finite loss at step {t + 1}")
        # the LARC status of this step's update (reset by every update): a non-finite norm raises
        # on the step it happens, like optimizer.py:56-57, not at the end of the run
        tr.check_status()
        rate = torch.tensor([cfg.local_batch / wall, lv, wall], dtype=torch.float64)
        if world > 1:
            allr = [torch.zeros_like(rate) for _ in range(world)]
            dist.all_gather_object(allr, rate)
        else:
            allr = [rate]
        rates = tuple(float(r[0]) for r in allr)
        records.append(StepRecord(step=t + 1, rates=rates, wall=max(float(r[2]) for r in allr),
                                  loss=float(np.mean([float(r[1]) for r in allr]))))
        losses.append(records[-1].loss)
        if (t + 1) in hash_at:   # like the reference, before the post-loop lag-1 apply
            digests.append((t + 1, tr.hash_sync(t + 1)))
    tr.finish()
    tr.check_status()
    stats = sustained_stats(records, per_sample_flops=model_flops_per_sample(net, shape))
    return TrainResult(records, stats, losses, digests, net.state_dict() if rank == 0 else {})
