"""Headline benchmark: DeepLabV3+ bf16 training step on 16x1152x768 tiles, batch 2 per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one process per GPU)

Metric (BASELINE.json): train images/s and sustained TF/s at 1152x768x16, whole job.
A step is one full training step (forward, fused weighted CE, backward, bucketed NCCL
all-reduce, LARC + momentum update, weight repack) over the rank's batch of 2 tiles.
`value` is device-timed with CUDA events, inputs resident in HBM, max over ranks;
`e2e` is the same step through the public trainer API with the batch copied from
pinned host memory and every step's loss read back to the host (one step behind, so the
next step is already queued while the host waits).  The working set (~11 GB of
activations and gradients per GPU) is far larger than L2, so no L2 flush is needed.

--impl reference times the reference's CPU step (the oracle/ NumPy restatement of
deskdl's executor + im2col/OpenBLAS kernels + LARC) on a bounded 1x16x288x192
sample of the same workload, reported in full-tile-equivalent images/s.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W, C, LOCAL_BATCH = 1152, 768, 16, 2
METRIC = "DeepLabv3+ train images/s & sustained TF/s, 1152×768×16, at 1/2/4/8 B200"
CPU_SAMPLE = (1, 16, 288, 192)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append([time.time()] + parts[1:])

    def window(self, t0, t1):
        """Restrict to samples taken in [t0, t1] (host wall clock around the timed region);
        falls back to all samples under load when the window holds fewer than 3."""
        sel = [r for r in self.rows if t0 <= r[0] <= t1]
        if len(sel) >= 3:
            self.rows = sel

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist_init(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def _deskdl():
    """The unmodified reference package, installed by `pip install --target baseline/_ref`
    (DESIGN.md §8), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "deskdl")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import deskdl
    return deskdl


def reference_step_times(steps: int, warmup: int):
    """(seconds per step, kind, backend): the reference's own training step -- deskdl's
    executor (ops.run_forward / run_backward, ops.py:44-106) with its stock conv backend
    (kernels.py:19-40, NumPy im2col + OpenBLAS here: the fastest it ships) and its LARC update
    per tensor (optimizer.py:79-83, trainer.py:364-367) -- on the bounded sample, all host
    threads.  Falls back to the oracle port (kind "port") when deskdl is not installed."""
    deskdl = _deskdl()
    if deskdl is None:
        return cpu_step_time(steps, warmup), "port", "oracle/deskdl_port.py"
    os.environ.setdefault("DESKDL_KERNELS", "python")   # im2col+sgemm: ~9x the Cython loops here
    # all host threads for OpenBLAS even under torchrun (which exports OMP_NUM_THREADS=1)
    from threadpoolctl import threadpool_limits
    _limits = threadpool_limits(limits=os.cpu_count())   # noqa: F841  (kept for the run)
    from deskdl.graph import OpGraph
    from deskdl.model import ClassWeights, kernels, ops
    from deskdl.optimizer import LayerParam, OptimConfig, larc_sgd_step
    from paper_1810_01993_b200 import models
    from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng
    graph, params, head, lossn = models.build_deeplab(models.DeepLabConfig(), seed=0, graph_cls=OpGraph)
    order = list(params)
    lps = {k: LayerParam(k, params[k]) for k in order}
    cfg = OptimConfig(lr=0.01, momentum=0.9, trust=0.02)
    n, c, h, w = CPU_SAMPLE
    f, lab = make_scene(SceneConfig(channels=c, height=h, width=w), scene_rng(0, 0, 0))
    cw = ClassWeights((0.982, 0.017, 0.001)).vector()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        values = {k: lps[k].w for k in order}
        values.update(x=f[None], labels=lab[None], class_weights=cw)
        out, tape = ops.run_forward(graph, values, targets=[lossn, head])
        grads = ops.run_backward(graph, tape, lossn, wrt=order)
        for k in order:
            larc_sgd_step(lps[k], grads[k].reshape(lps[k].w.shape), cfg)
        times.append(time.perf_counter() - t0)
    return times[warmup:], "reference", f"deskdl {kernels.BACKEND} backend"


def cpu_step_time(steps: int, warmup: int):
    """Seconds per reference CPU step on the bounded sample (oracle port, all host threads)."""
    from threadpoolctl import threadpool_limits
    _limits = threadpool_limits(limits=os.cpu_count())   # noqa: F841
    from oracle import deskdl_port as O
    from paper_1810_01993_b200 import models
    from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng
    graph, params, head, lossn = models.build_deeplab(models.DeepLabConfig(), seed=0)
    order = list(params)
    moms = {k: np.zeros_like(v) for k, v in params.items()}
    n, c, h, w = CPU_SAMPLE
    f, lab = make_scene(SceneConfig(channels=c, height=h, width=w), scene_rng(0, 0, 0))
    cw = O.class_weights((0.982, 0.017, 0.001))
    opt = dict(lr=0.01, momentum=0.9, trust=0.02)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.train_step(graph, params, order, f[None], lab[None], cw, lossn, head, opt=opt, moms=moms)
        times.append(time.perf_counter() - t0)
    return times[warmup:]


def _sample_desc(kind="reference", backend="deskdl python backend"):
    n, c, h, w = CPU_SAMPLE
    frac = (h * w) / (H * W)
    who = (f"the reference itself (deskdl 0.1.0 from baseline/_ref, {backend}: ops.run_forward/run_backward "
           f"+ per-tensor larc_sgd_step)" if kind == "reference" else
           "oracle/ NumPy port of deskdl's step (im2col + OpenBLAS sgemm, tape VJPs, LARC)")
    return (f"{who} on the same DeepLabV3+ graph at {n}x{c}x{h}x{w} = {frac:.4f} of one {H}x{W} tile; "
            f"EXTRAPOLATED to full tiles: conv FLOPs scale linearly with pixels, so images/s = "
            f"{frac:.4f} / step time (a full-tile deskdl step needs ~40 GB of im2col caches and ~100+ s)"), frac


KERNEL_OF_PASS = {
    "fprop": "conv_fprop_kernel, tcgen05 implicit GEMM (CTA pairs for 256-wide N; the row-window halo "
             "kernel for the stem)",
    "dgrad": "conv_fprop_kernel over dy with tap-flipped master weights (CTA pairs)",
    "wgrad": "conv_wgrad_kernel, tcgen05 implicit GEMM, split-K with deferred fixed-order reduction",
}


def _traffic(dom):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/round2/roofline_traffic.json, written by tools/make_traffic.py), else None."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "round2", "roofline_traffic.json")
    try:
        d = json.load(open(p))
        e = d.get(dom)
        if e:
            return float(e["dram_bytes_per_launch"]), f"{os.path.relpath(p)}: {e['launch']}"
    except (OSError, ValueError, KeyError):
        pass
    return None, None


WORKLOADS = {
    "reference-ops": ("config 2/3: DeepLabV3+ (ResNet-50 OS8, ASPP 12/18/24, full-res decoder) bf16 train step, "
                      "fused weighted CE + LARC", "DeepLabV3+"),
    "bn-bilinear": ("north-star DeepLabV3+ variant (batch norm after every conv, bilinear decoder upsampling) bf16 "
                    "train step, fused weighted CE + LARC", "DeepLabV3+ (BN + bilinear)"),
    "tiramisu": ("config 4: Tiramisu / FC-DenseNet (5 levels, (2,2,2,4,5) dense blocks, growth 32, 5x5) train "
                 "step, fused weighted CE + LARC", "Tiramisu"),
}


def _config(world, variant="reference-ops"):
    wl, model = WORKLOADS[variant]
    return {"workload": wl, "model": model, "variant": variant,
            "global_batch": world * LOCAL_BATCH, "local_batch": LOCAL_BATCH, "tile": [C, H, W],
            "parallelism": f"dp{world}", "l2": "working set ~11 GB/GPU >> 126 MB L2, no flush"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # bounded: each CPU step is ~6-9 s, keep the whole arm within a few minutes
    times, kind, backend = reference_step_times(max(1, min(args.steps, 8)), min(args.warmup, 1))
    desc, frac = _sample_desc(kind, backend)
    ms = 1e3 * float(np.median(times))
    value = frac / (ms / 1e3)
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": len(times), "warmup": min(args.warmup, 1), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (make_scene)",
            "config": dict(_config(world), reference_arm=f"reference CPU step ({kind}: {backend}, all host "
                           "threads) on a bounded sample of the same workload, rank 0 only",
                           sample_batch=CPU_SAMPLE[0], sample_tile=list(CPU_SAMPLE[1:])),
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind, "sample": desc,
                             "extrapolated": True, "step_s": ms / 1e3},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1810_01993_b200.flops import count_graph, exact_train_flops, train_flops_per_sample
    from paper_1810_01993_b200.loss import ClassWeights
    from paper_1810_01993_b200.models import DeepLabConfig
    from paper_1810_01993_b200.net import DeepLabV3Plus
    from paper_1810_01993_b200.optimizer import OptimConfig
    from paper_1810_01993_b200.scenes import SceneConfig, device_scene_pool
    from paper_1810_01993_b200.stats import StepRecord, sustained_stats
    from paper_1810_01993_b200.trainer import DataParallelTrainer

    world, rank, local = _dist_init(args)
    dev = torch.device("cuda", local)
    shape = (LOCAL_BATCH, C, H, W)
    variant = getattr(args, "variant", "reference-ops")
    metric = METRIC
    # config 4 is FP16 (BASELINE.json); the DeepLabV3+ configs are bf16
    precision = args.precision or ("fp16" if variant == "tiramisu" else "bf16")
    if variant == "tiramisu":   # config 4 (the paper's Tiramisu / FC-DenseNet, frozen definition)
        from paper_1810_01993_b200.models import tiramisu_config4
        from paper_1810_01993_b200.net import MiniDenseNet
        net = MiniDenseNet(tiramisu_config4(), seed=0, precision=precision)
        metric = "Tiramisu (FC-DenseNet, config 4) train images/s & sustained TF/s, 1152×768×16"
    else:
        net = DeepLabV3Plus(DeepLabConfig(batchnorm=variant == "bn-bilinear", bilinear=variant == "bn-bilinear"),
                            seed=0, precision=precision)
    scene = SceneConfig(channels=C, height=H, width=W)
    cw = ClassWeights(scene.frequencies).vector()
    hier = tuple(int(v) for v in args.hierarchy.split("x")) if getattr(args, "hierarchy", "") else None
    # lr 0.002: at 0.01 the synthetic run's first steps spike (loss 2 -> 11 at lag 0, -> 158 at lag 1,
    # NaN later); the step's work does not depend on it
    tr = DataParallelTrainer(net, OptimConfig(lr=0.002, momentum=0.9, trust=0.02), shape, class_weights=cw,
                             hierarchy=hier, lag=args.lag, bucket_mb=args.bucket_mb)
    eng = tr.eng
    # synthetic pool, resident in HBM, different tiles per rank
    pool = 4
    fx, fl = device_scene_pool(pool * LOCAL_BATCH, scene, seed=1000 + rank, device=dev)
    batches = [(fx[i * LOCAL_BATCH:(i + 1) * LOCAL_BATCH].contiguous(),
                fl[i * LOCAL_BATCH:(i + 1) * LOCAL_BATCH].contiguous()) for i in range(pool)]

    shapes = {k: v.shape for k, v in net._params.items()}
    shapes.update(x=(LOCAL_BATCH, C, H, W), labels=(LOCAL_BATCH, H, W), class_weights=(3,))
    rep = count_graph(net.graph, shapes, batch=LOCAL_BATCH)
    flops_img = train_flops_per_sample(rep)
    flops_img_exact = exact_train_flops(net.graph, shapes, LOCAL_BATCH)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local).__enter__()   # sampling starts before warm-up (nvidia-smi start-up)
    for i in range(args.warmup):
        tr.step(*batches[i % pool])
    barrier()

    # ---- the step is captured once as a CUDA graph (all launches + NCCL bucket all-reduces);
    # the timed graph carries event nodes around every conv launch for the roofline
    graphed = not args.no_graph
    if graphed:
        tr.capture(*batches[0], timed=True, buffers=2)
        for i in range(2):
            tr.step(*batches[i % pool])
    else:
        eng.conv_timing = True
        eng.conv_events = []
    barrier()

    # ---- timed region: device events around K steps, max over ranks
    launches0 = eng.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one event per step boundary as well: the per-step rates the reference's statistics use
    # (stats.py:58-79 median of per-step rank-mean rates, first step dropped, p16/p84)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    t_lo = time.time()
    e0.record()
    marks[0].record()
    for i in range(args.steps):
        tr.step(*batches[i % pool])
        marks[i + 1].record()
    e1.record()
    barrier()
    t_hi = time.time()
    clk.__exit__(None, None, None)
    clk.window(t_lo, t_hi)
    launches = eng.launches - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if graphed:   # conv launches of the last step of the timed region (events are graph nodes)
        per_pass = {k: (m * args.steps, f * args.steps) for k, (m, f) in tr.graph_conv_totals(by_pass=True).items()}
    else:
        eng.conv_timing = False
        per_pass = eng.conv_kernel_totals(by_pass=True)
    conv_ms = sum(m for m, _ in per_pass.values())
    conv_flops = sum(f for _, f in per_pass.values())
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * LOCAL_BATCH / (ms / 1e3)
    step_ms = torch.tensor([marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)], dtype=torch.float64,
                           device=dev)
    if world > 1:
        allm = [torch.zeros_like(step_ms) for _ in range(world)]
        dist.all_gather(allm, step_ms)
    else:
        allm = [step_ms]
    allm = torch.stack(allm).cpu().numpy()          # [rank][step] ms
    records = [StepRecord(step=i + 1, rates=tuple(LOCAL_BATCH / (allm[:, i] / 1e3)), wall=float(allm[:, i].max()) / 1e3,
                          loss=0.0) for i in range(args.steps)]

    # ---- e2e: public API, host inputs (pinned) copied every step, loss read back every step
    host = [(b[0].cpu().pin_memory(), b[1].cpu().pin_memory()) for b in batches]
    h2d = host[0][0].numel() * 4 + host[0][1].numel()
    dx = tr.static_x if graphed else torch.empty_like(batches[0][0])
    dl = tr.static_l if graphed else torch.empty_like(batches[0][1])
    barrier()
    e_steps = max(2, args.steps)   # the same K steps as the device-timed region
    e0.record()
    if graphed:
        # the next step's host->device copy runs on a copy stream under the current step; every
        # step's loss is copied to pinned host memory behind it and read by the host one step
        # later (while the next step is already queued), so the GPU never idles on the host
        lh = [torch.empty(1, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        lev = [torch.cuda.Event() for _ in range(2)]
        tr.stage(*host[0])
        for i in range(e_steps):
            loss = tr.step_staged()
            lh[i % 2].copy_(loss, non_blocking=True)
            lev[i % 2].record()
            if i + 1 < e_steps:
                tr.stage(*host[(i + 1) % pool])
            if i > 0:
                lev[(i - 1) % 2].synchronize()
                lv = float(lh[(i - 1) % 2][0])
        lev[(e_steps - 1) % 2].synchronize()
        lv = float(lh[(e_steps - 1) % 2][0])
    else:
        for i in range(e_steps):
            hx, hl = host[i % pool]
            dx.copy_(hx, non_blocking=True)
            dl.copy_(hl, non_blocking=True)
            loss = tr.step(dx, dl)
            lv = float(loss.item())
    e1.record()
    barrier()
    e_ms = e0.elapsed_time(e1) / e_steps
    t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e_ms = float(t.item())
    tr.check_status()

    # ---- the conv kernels on their own: in the step, each wgrad shares the GPU with the dgrad it
    # runs beside (and the ASPP branches with each other), so event durations there overlap.  One
    # extra eager step with every launch on one stream times each kernel alone (roofline).
    in_step = per_pass
    eng.serialize(True)
    eng.conv_timing, eng.conv_events, eng.graph_events = True, [], False
    tr._eager_step(*batches[0])
    eng.conv_timing = False
    per_pass = {k: (m * args.steps, f * args.steps) for k, (m, f) in eng.conv_kernel_totals(by_pass=True).items()}
    eng.serialize(False)
    tr.check_status()
    conv_ms = sum(m for m, _ in per_pass.values())
    conv_flops = sum(f for _, f in per_pass.values())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        times, kind, backend = reference_step_times(2, 0)
        desc, frac = _sample_desc(kind, backend)
        cpu = {"value": frac / float(np.median(times)), "unit": "images/s", "cores": os.cpu_count(),
               "kind": kind, "sample": desc, "extrapolated": True, "step_s": float(np.median(times))}

    peak, peak_sust, hbm, src = _peaks()
    achieved_all = conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
    # dominant kernel: the conv pass (fprop | dgrad | wgrad launches) with the most device time
    dom = max(per_pass, key=lambda k: per_pass[k][0]) if per_pass else "fprop"
    dom_ms, dom_fl = per_pass.get(dom, (0.0, 0))
    achieved = dom_fl / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else 0.0
    traffic, traffic_src = _traffic(dom)
    if rank == 0:
        rule_tf = value * flops_img / 1e12
        exec_img = conv_flops / args.steps / LOCAL_BATCH
        exec_tf = value * exec_img / 1e12
        st = sustained_stats(records, per_sample_flops=exec_img)
        line = {
            "metric": metric, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": precision, "data": "synthetic (GPU-generated scenes, resident in HBM)",
            "config": dict(_config(world, variant), lag=args.lag, precision=precision,
                           **({"allreduce": f"hierarchical {args.hierarchy}"} if hier else {})),
            # sustained TF/s = tensor-core FLOPs the step executes x images/s (the convs' MACs; full.c0
            # runs from the low-resolution input, so this is below the reference-rule count)
            "sustained_tflops": exec_tf, "frac_of_peak": exec_tf / peak,
            "executed_conv_flops_per_image": exec_img,
            # the reference's own statistics over the same K device-timed steps (stats.py:58-79):
            # median / p16 / p84 of the per-step rank-mean rate, first step dropped; global = x world
            "stats": {"global_images_per_s_median": st.global_rate, "rank_rate_median": st.median,
                      "rank_rate_p16": st.p16, "rank_rate_p84": st.p84, "steps_used": st.steps,
                      "sustained_tflops_median": st.flops_per_s / 1e12},
            # reference FLOP rule (flops.py:56-112, 3 x forward, full.c0 counted at full resolution)
            "reference_rule": {"flops_per_image": flops_img, "flops_per_image_exact": flops_img_exact,
                               "tflops": rule_tf, "frac_of_peak": rule_tf / peak},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": f"{dom}: {KERNEL_OF_PASS[dom]} (all {dom} launches of one step, each timed "
                                   f"alone with CUDA events on its stream in a serialized step after the "
                                   f"timed region; executed 2*taps*Cin*Cout FLOPs per output pixel / time)",
                         "peak_source": src, "peak_sustained": peak_sust,
                         "per_pass": {k: {"ms_per_step": m / args.steps,
                                          "tflops": (f / (m / 1e3) / 1e12) if m > 0 else 0.0}
                                      for k, (m, f) in sorted(per_pass.items())},
                         "per_pass_in_step": {k: {"ms_per_step": m / args.steps,
                                                  "tflops": (f / (m / 1e3) / 1e12) if m > 0 else 0.0}
                                              for k, (m, f) in sorted(in_step.items())},
                         "all_convs": {"achieved": achieved_all, "frac": achieved_all / peak,
                                       "conv_ms_per_step": conv_ms / args.steps}},
            "e2e": {"value": world * LOCAL_BATCH / (e_ms / 1e3), "unit": "images/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4, "ms_per_step": e_ms},
            "gpu_launches": launches, "cuda_graph": graphed, "clocks": clk.summary(), "cpu_baseline": cpu,
            "last_loss": lv,
        }
        emit(line)
    tr.release_graph()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _json_stdout():
    """Keep fd 1 for the one JSON line: library banners written to stdout (e.g. the NCCL version
    line) are redirected to stderr at the file-descriptor level."""
    global JSON_OUT
    sys.stdout.flush()
    JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


JSON_OUT = sys.stdout


def emit(line):
    print(json.dumps(line), file=JSON_OUT, flush=True)


def main():
    _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--precision", default=None, choices=["bf16", "fp16"],
                    help="16-bit storage / MMA operand type (default: bf16; fp16 for --variant tiramisu, config 4)")
    ap.add_argument("--bucket-mb", type=float, default=32.0, help="gradient all-reduce bucket size (N > 1)")
    ap.add_argument("--lag", type=int, default=0, choices=[0, 1],
                    help="gradient lag (trainer.py:378-383): 1 applies the previous step's reduced gradients")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a captured CUDA graph")
    ap.add_argument("--hierarchy", default="", help="GxL: three-stage hierarchical all-reduce over G groups of L "
                                                     "ranks (the paper's scheme) instead of one flat NCCL all-reduce")
    ap.add_argument("--variant", default="reference-ops", choices=["reference-ops", "bn-bilinear", "tiramisu"],
                    help="model: the frozen reference-op DeepLabV3+ (headline), the north-star DeepLabV3+ with "
                         "batch norm after every conv and bilinear decoder upsampling, or config 4's Tiramisu")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
