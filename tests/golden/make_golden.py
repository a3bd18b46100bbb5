"""Generate golden vectors by running the REFERENCE (deskdl) in the build container.

    python tests/golden/make_golden.py

Imports deskdl from /root/reference (read-only; compiled tree under
pkg/build/lib.*) with the NumPy kernel backend, runs the hot-path functions on
seeded inputs and writes small .npz fixtures next to this file.  The fixtures
pin oracle/ (tests/test_oracle.py) and the GPU path (tests/test_gpu_*.py).
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import glob
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_LIB = sorted(glob.glob("/root/reference/pkg/build/lib.*"))
os.environ["DESKDL_KERNELS"] = "python"
sys.path.insert(0, REF_LIB[0] if REF_LIB else "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from deskdl import flops as rflops  # noqa: E402
from deskdl.graph import OpGraph as RefGraph  # noqa: E402
from deskdl.harness.config import DataConfig, RunConfig  # noqa: E402
from deskdl.harness.trainer import train_run  # noqa: E402
from deskdl.model import ClassWeights, MiniDenseNet, NetConfig as RefNetConfig, SceneConfig  # noqa: E402
from deskdl.model import _kernels_py, make_scene, ops as rops, weighted_ce_loss  # noqa: E402
from deskdl.optimizer import LayerParam, OptimConfig, larc_sgd_step  # noqa: E402

from paper_1810_01993_b200 import models  # noqa: E402  (graph builders only; no GPU)

CONV_CASES = [  # n, cin, h, w, cout, k, dilation
    (1, 3, 7, 6, 4, 3, 1), (2, 5, 9, 7, 4, 3, 2), (1, 8, 6, 6, 5, 1, 1),
    (2, 16, 12, 10, 8, 7, 1), (1, 4, 10, 8, 6, 3, 4), (2, 6, 8, 8, 3, 3, 12),
]


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values()), "bytes raw")


def replica(graph):
    """Copy one of our OpGraphs into a reference OpGraph (same names, kinds, attrs)."""
    g = RefGraph()
    for name, role in graph.inputs.items():
        g.add_input(name, role)
    for nd in graph.nodes:
        from deskdl.graph import OpNode
        g.add_node(OpNode(nd.name, nd.kind, tuple(nd.inputs), dict(nd.attrs)))
    return g


def gen_conv():
    out = {}
    rng = np.random.default_rng(2024)
    for i, (n, cin, h, w, cout, k, d) in enumerate(CONV_CASES):
        for dt in (np.float64, np.float32):
            tag = f"c{i}_{np.dtype(dt).name}"
            x = rng.standard_normal((n, cin, h, w)).astype(dt)
            wt = rng.standard_normal((cout, cin, k, k)).astype(dt)
            dy = rng.standard_normal((n, cout, h, w)).astype(dt)
            y, cache = _kernels_py.conv2d_forward(x, wt, dilation=d)
            out[f"{tag}_x"], out[f"{tag}_w"], out[f"{tag}_dy"] = x, wt, dy
            out[f"{tag}_y"] = y
            out[f"{tag}_dw"] = _kernels_py.conv2d_backward_weights(cache, dy, wt.shape, dilation=d)
            out[f"{tag}_dx"] = _kernels_py.conv2d_backward_input(dy, wt, x.shape, dilation=d)
    out["cases"] = np.array(CONV_CASES, dtype=np.int64)
    save("conv.npz", **out)


def gen_loss():
    out = {}
    rng = np.random.default_rng(7)
    w = ClassWeights((0.982, 0.017, 0.001)).vector()
    out["weights"] = w
    for i, (n, h, wd) in enumerate([(1, 5, 4), (2, 6, 5), (2, 32, 24)]):
        logits = (rng.standard_normal((n, 3, h, wd)) * 3).astype(np.float32)
        labels = rng.integers(0, 3, size=(n, h, wd)).astype(np.uint8)
        loss, dl = weighted_ce_loss(logits, labels, w)
        out[f"l{i}_logits"], out[f"l{i}_labels"] = logits, labels
        out[f"l{i}_loss"] = np.array(loss)
        out[f"l{i}_dlogits"] = dl
        out[f"l{i}_argmax"] = np.argmax(logits, axis=1).astype(np.uint8)
    # ties resolve to the lowest index
    tie = np.zeros((1, 3, 2, 2), np.float32)
    tie[0, 1, 0, 0] = tie[0, 2, 0, 0] = 1.0
    out["tie_logits"], out["tie_argmax"] = tie, np.argmax(tie, axis=1).astype(np.uint8)
    save("loss.npz", **out)


def gen_larc():
    out = {}
    rng = np.random.default_rng(99)
    cfgs = [OptimConfig(), OptimConfig(lr=0.05, momentum=0.9, trust=0.02, weight_decay=1e-4),
            OptimConfig(lr=0.7, momentum=0.0, trust=0.5)]
    for ci, cfg in enumerate(cfgs):
        for li in range(6):
            n = int(rng.integers(1, 300))
            w = (rng.standard_normal(n) * rng.uniform(0.01, 3)).astype(np.float32)
            g = (rng.standard_normal(n) * rng.uniform(0.001, 10)).astype(np.float32)
            if li == 4:
                w[:] = 0
            if li == 5:
                g[:] = 0
            m = (rng.standard_normal(n) * 0.1).astype(np.float32)
            p = LayerParam("w", w.copy())
            p.m = m.copy()
            lrs = [larc_sgd_step(p, g, cfg) for _ in range(3)]
            tag = f"o{ci}_{li}"
            out[f"{tag}_w0"], out[f"{tag}_g"], out[f"{tag}_m0"] = w, g, m
            out[f"{tag}_w3"], out[f"{tag}_m3"] = p.w.copy(), p.m.copy()
            out[f"{tag}_lr"] = np.array(lrs)
            out[f"{tag}_cfg"] = np.array([cfg.lr, cfg.momentum, cfg.trust, cfg.weight_decay, cfg.eps])
    save("larc.npz", **out)


def gen_scenes():
    out = {}
    for i, (c, h, w) in enumerate([(16, 32, 24), (8, 64, 48)]):
        kw = dict(channels=c, height=h, width=w)
        if c < 16:
            kw.update(streak_channels=(0, 1), blob_channels=(2, 3))
        cfg = SceneConfig(**kw)
        for t, j in [(0, 0), (3, 1)]:
            sc = make_scene(cfg, np.random.default_rng((0, 0, t, j)), name="g")
            out[f"s{i}_{t}_{j}_field"], out[f"s{i}_{t}_{j}_labels"] = sc.field, sc.labels
            out[f"s{i}_{t}_{j}_counts"] = sc.class_counts(3)
        out[f"s{i}_shape"] = np.array([c, h, w])
    save("scenes.npz", **out)


def _run_ref_graph(graph, params, order, x, labels, cw, loss_name, logits_name):
    g = replica(graph)
    vals = dict(params)
    vals.update(x=x, labels=labels, class_weights=cw)
    out, tape = rops.run_forward(g, vals, targets=[loss_name, logits_name])
    grads = rops.run_backward(g, tape, loss_name, wrt=order)
    return float(out[loss_name][0]), out[logits_name], grads


def gen_models():
    cw = ClassWeights((0.982, 0.017, 0.001)).vector()
    # (1) the reference's own network: init bytes + one forward/backward
    out = {}
    rcfg = RefNetConfig(channels_in=8, growth=16, block_layers=2, levels=2)
    ref = MiniDenseNet(rcfg, seed=3)
    sc_cfg = SceneConfig(channels=8, height=32, width=24, streak_channels=(0, 1), blob_channels=(2, 3))
    xs, ls = [], []
    for j in range(2):
        s = make_scene(sc_cfg, np.random.default_rng((3, 0, 0, j)), name="m")
        xs.append(s.field)
        ls.append(s.labels)
    x, lab = np.stack(xs), np.stack(ls)
    loss, logits, tape = ref.forward_loss(x, lab, cw)
    grads = ref.backward(tape)
    out.update(x=x, labels=lab, loss=np.array(loss), logits=logits,
               order=np.array(ref.param_order))
    for k in ref.param_order:
        out[f"p:{k}"] = ref.params[k]
        out[f"g:{k}"] = grads[k]
    save("minidensenet.npz", **out)

    # (2) our DeepLabV3+ topology (small widths), executed by the reference's executor
    out = {}
    cfg = models.deeplab_small()
    graph, params, head, lossn = models.build_deeplab(cfg, seed=5)
    order = list(params)
    sc_cfg = SceneConfig(channels=16, height=32, width=32)
    xs, ls = [], []
    for j in range(2):
        s = make_scene(sc_cfg, np.random.default_rng((5, 0, 0, j)), name="d")
        xs.append(s.field)
        ls.append(s.labels)
    x, lab = np.stack(xs), np.stack(ls)
    loss, logits, grads = _run_ref_graph(graph, params, order, x, lab, cw, lossn, head)
    out.update(x=x, labels=lab, loss=np.array(loss), logits=logits, order=np.array(order))
    for k in order:
        out[f"p:{k}"] = params[k]
        out[f"g:{k}"] = grads[k]
    save("deeplab_small.npz", **out)


def gen_flops():
    out = {}
    g = RefGraph()
    g.add_input("x")
    g.add_input("w", role="param")
    g.conv2d("x", "w", "c", kh=3, kw=3, cin=48, cout=32)
    out["worked"] = np.array(rflops.count_graph(g, {"x": (2, 48, 1152, 768), "w": (32, 48, 3, 3)}, 2).total)
    for tag, cfg in [("deeplab", models.DeepLabConfig()), ("deeplab_small", models.deeplab_small())]:
        graph, params, _, _ = models.build_deeplab(cfg, seed=0)
        for h, w in [(1152, 768), (288, 192)]:
            shapes = {k: v.shape for k, v in params.items()}
            shapes.update(x=(2, 16, h, w), labels=(2, h, w), class_weights=(3,))
            rep = rflops.count_graph(replica(graph), shapes, batch=2)
            out[f"{tag}_{h}x{w}_fwd"] = np.array(rep.total)
            out[f"{tag}_{h}x{w}_train_per_sample"] = np.array(rflops.train_flops_per_sample(rep))
    save("flops.npz", **out)


def gen_trainer():
    """Reference trainer: 1 rank x batch 2 vs 2 ranks x batch 1, lag 0 and 1."""
    from deskdl.core import RankTopology
    out = {}
    scene = SceneConfig(channels=8, height=16, width=16, streak_channels=(0, 1), blob_channels=(2, 3))
    net = RefNetConfig(channels_in=8, growth=16, block_layers=1, levels=1)
    for lag in (0, 1):
        for world, lb in ((1, 2), (2, 1)):
            cfg = RunConfig(topology=RankTopology(1, world, 1), lag=lag, steps=3, local_batch=lb,
                            seed=4, optim=OptimConfig(lr=0.1), net=net,
                            data=DataConfig(scene=scene))
            res = train_run(cfg)
            tag = f"lag{lag}_w{world}"
            out[f"{tag}_losses"] = np.array([r.loss for r in res.records])
            for k, v in res.state.items():
                out[f"{tag}_state:{k}"] = v
    save("trainer.npz", **out)


def gen_checkpoint():
    """A CKP1 file written by the reference's own save_checkpoint (model/checkpoint.py:18-28)."""
    from deskdl.model.checkpoint import save_checkpoint
    rng = np.random.default_rng(11)
    params = {"conv.w": rng.normal(size=(4, 3, 3, 3)).astype(np.float32),
              "conv.b": rng.normal(size=(4,)).astype(np.float32),
              "scalar": np.array(2.5, dtype=np.float32),
              "µ-unicode/name": rng.normal(size=(2, 5)).astype(np.float32)}
    save_checkpoint(os.path.join(HERE, "ckp1_reference.bin"), params)
    save("ckp1_reference_arrays.npz", **{f"a{i}": v for i, v in enumerate(params.values())},
         names=np.array(list(params.keys())))


def gen_stats():
    """The reference's throughput statistics (harness/stats.py:58-79, scaling.py:44-69) on seeded
    per-step per-rank rate series."""
    from deskdl.harness.stats import StepRecord, sustained_stats
    out = {}
    rng = np.random.default_rng(5)
    for i, (steps, world, warm) in enumerate([(20, 1, 1), (9, 4, 1), (1, 2, 1), (6, 8, 2), (2, 3, 1)]):
        rates = rng.uniform(1.0, 3.0, size=(steps, world))
        recs = [StepRecord(step=t + 1, rates=tuple(rates[t]), wall=1.0 / rates[t].mean(), loss=0.0)
                for t in range(steps)]
        st = sustained_stats(recs, per_sample_flops=1.5e12, warmup=warm)
        out[f"s{i}_rates"] = rates
        out[f"s{i}_warmup"] = np.array(warm)
        out[f"s{i}_result"] = np.array([st.median, st.p16, st.p84, st.world, st.steps, st.flops_per_s,
                                        st.global_rate])
    save("stats.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:   # e.g. `make_golden.py gen_checkpoint`: regenerate selected fixtures
        for fn in sys.argv[1:]:
            globals()[fn]()
        sys.exit(0)
    gen_checkpoint()
    gen_conv()
    gen_loss()
    gen_larc()
    gen_scenes()
    gen_models()
    gen_flops()
    gen_trainer()
    gen_stats()
