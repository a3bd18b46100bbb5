"""fp32 parity mode (b2dl.h group 3): the same engine program with fp32 buffers and fp32 FMA
kernels must meet the north star's fp32 bar -- loss, logits and every per-layer gradient within
1e-3 relative (max|a-b| / max|b|, pkg/tests/test_kernels.py:17-19) of the reference on identical
inputs and seeds; argmax masks and label histograms exact."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FP32_TOL = 1e-3


def load(name):
    return np.load(os.path.join(G, name))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _check(net, x, labels, cw, loss_ref, logits_ref, grads_ref):
    loss, logits, tape = net.forward_loss(x, labels, cw)
    assert abs(loss - loss_ref) < FP32_TOL * abs(loss_ref)
    lg = logits.cpu().numpy()
    assert rel(lg, logits_ref) < FP32_TOL
    assert np.array_equal(tape.engine.predictions().cpu().numpy(), np.argmax(lg, axis=1))
    counts = tape.engine.counts.cpu().numpy().reshape(x.shape[0], 3)
    for i in range(x.shape[0]):
        assert np.array_equal(counts[i], np.bincount(np.asarray(labels[i]).reshape(-1), minlength=3))
    grads = net.backward(tape)
    errs = {k: rel(grads[k], grads_ref[k]) for k in net.param_order}
    bad = {k: e for k, e in errs.items() if e > FP32_TOL}
    assert not bad, bad


def test_fp32_minidensenet_matches_reference_golden():
    from paper_1810_01993_b200.loss import ClassWeights
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.net import MiniDenseNet
    d = load("minidensenet.npz")
    net = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=2, levels=2), seed=3, precision="fp32")
    cw = ClassWeights((0.982, 0.017, 0.001)).vector()
    _check(net, d["x"], d["labels"], cw, float(d["loss"]), d["logits"],
           {k: d[f"g:{k}"] for k in net.param_order})


def test_fp32_deeplab_small_matches_reference_golden():
    from paper_1810_01993_b200.loss import ClassWeights
    from paper_1810_01993_b200.models import deeplab_small
    from paper_1810_01993_b200.net import DeepLabV3Plus
    d = load("deeplab_small.npz")
    net = DeepLabV3Plus(deeplab_small(), seed=5, precision="fp32")
    cw = ClassWeights((0.982, 0.017, 0.001)).vector()
    _check(net, d["x"], d["labels"], cw, float(d["loss"]), d["logits"],
           {k: d[f"g:{k}"] for k in net.param_order})


def test_fp32_deeplab_full_config1_matches_oracle():
    """Config 1 exactly: full DeepLabV3+, fp32, batch 1, 16x288x192.

    At this size a handful of pre-activations sit within fp32 round-off of zero, so *any* two fp32
    implementations (the reference's own fp32 step included) disagree on a few relu decisions, and
    a single flipped pixel moves the max-abs gradient metric of the layers behind it by ~1e-3
    (tests/diagnostics/fp32_flips.py: 1-2 flips per affected tensor, the same count as the reference's own
    fp32 step against float64).  The oracle is therefore run in float64 with the GPU's relu
    decisions imposed (relu_masks) -- the flips are counted and bounded separately -- and every
    gradient must then agree to 1e-3."""
    from oracle import deskdl_port as O
    from paper_1810_01993_b200.models import DeepLabConfig
    from paper_1810_01993_b200.net import DeepLabV3Plus
    from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng
    net = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp32")
    f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
    x, labels = f[None], lab[None]
    cw = O.class_weights((0.982, 0.017, 0.001))
    loss, logits, tape = net.forward_loss(x, labels, cw)
    eng = tape.engine
    masks, flips, total = {}, 0, 0
    p64 = {k: v.astype(np.float64) for k, v in net.params.items()}
    _, free = O.run_forward(net.graph, dict(p64, x=x.astype(np.float64), labels=labels,
                                              class_weights=cw.astype(np.float64)))
    for nd in net.graph.nodes:
        if nd.kind == "relu":
            m = eng.v(nd.name).tensor().float().cpu().numpy().transpose(0, 3, 1, 2) > 0
            masks[nd.name] = m
            flips += int((m != (free.values[nd.name] > 0)).sum())
            total += m.size
    assert flips <= 1e-5 * total, (flips, total)      # a few isolated near-zero decisions
    loss_ref, logits_ref, grads_ref, _ = O.train_step(net.graph, p64, net.param_order, x.astype(np.float64),
                                                     labels, cw.astype(np.float64), net.loss_name,
                                                     net.logits_name, relu_masks=masks)
    _check(net, x, labels, cw, loss_ref, logits_ref, grads_ref)


@pytest.mark.parametrize("lag", [0, 1])
def test_fp32_trainer_matches_reference_trainer(lag):
    """3 reference-trainer steps (1 rank, batch 2, lr 0.1, LARC): losses and final weights at 1e-3."""
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.optimizer import OptimConfig
    from paper_1810_01993_b200.scenes import SceneConfig
    from paper_1810_01993_b200.trainer import RunConfig, train_run
    d = load("trainer.npz")
    sc = SceneConfig(channels=8, height=16, width=16, streak_channels=(0, 1), blob_channels=(2, 3))
    cfg = RunConfig(lag=lag, steps=3, local_batch=2, seed=4, optim=OptimConfig(lr=0.1),
                    net=NetConfig(channels_in=8, growth=16, block_layers=1, levels=1), scene=sc, precision="fp32")
    res = train_run(cfg)
    tag = f"lag{lag}_w1"
    assert np.allclose(res.losses, d[tag + "_losses"], rtol=FP32_TOL)
    for k, v in res.state.items():
        ref = d[f"{tag}_state:{k}"]
        assert rel(v, ref) < FP32_TOL, k


def test_fp32_tiramisu_config4_topology_matches_oracle():
    """Config 4's Tiramisu topology (5x5, growth 32, (2,2,2,4,5)) on a 2 x 16 x 64 x 48 tile, fp32
    mode vs the oracle at the north-star 1e-3."""
    from oracle import deskdl_port as O
    from paper_1810_01993_b200.models import tiramisu_config4
    from paper_1810_01993_b200.net import MiniDenseNet
    from paper_1810_01993_b200.scenes import SceneConfig, generated_batch
    net = MiniDenseNet(tiramisu_config4(), seed=0, precision="fp32")
    x, labels = generated_batch(SceneConfig(height=64, width=48), seed=1, step=0, rank=0, local_batch=2)
    cw = O.class_weights((0.982, 0.017, 0.001))
    loss_ref, logits_ref, grads_ref, _ = O.train_step(net.graph, net.params, net.param_order, x, labels, cw,
                                                     net.loss_name, net.logits_name)
    _check(net, x, labels, cw, loss_ref, logits_ref, grads_ref)
