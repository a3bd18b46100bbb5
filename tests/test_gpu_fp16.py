"""IEEE fp16 storage (config 4's FP16): the same kernels built with fp16 as the
16-bit type (libb2dl_f16.so: kind::f16 MMAs on f16 operands, fp32 accumulation) and a static loss
scale for the per-pixel gradients.  Against the oracle restatement of the reference's fp32 step,
with the bf16 tests' rule: every gradient within max(2e-2, 4 x the error of an ideal fp16-storage
emulation of the same graph)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _check(net, x, labels, cw):
    from oracle import deskdl_port as O
    from oracle import bf16_emulation as E
    loss_ref, logits_ref, grads_ref, _ = O.train_step(net.graph, net.params, net.param_order, x, labels, cw,
                                                     net.loss_name, net.logits_name)
    loss, logits, tape = net.forward_loss(x, labels, cw)
    eng = tape.engine
    assert eng.half == "fp16" and eng.act[next(iter(eng.act))].dtype == torch.float16
    E.set_half(torch.float16, eng.loss_scale)
    try:
        _, emu = E.emulated_grads(net.graph, net.params, x, labels, cw, net.loss_name)
    finally:
        E.set_half(torch.bfloat16, 1.0)
    assert abs(loss - loss_ref) < 1e-2 * abs(loss_ref)
    lg = logits.cpu().numpy()
    assert rel(lg, logits_ref) < 1e-2
    assert np.array_equal(eng.predictions().cpu().numpy(), np.argmax(lg, axis=1))
    grads = net.backward(tape)
    bad = {}
    errs = []
    for k in net.param_order:
        e, ee = rel(grads[k], grads_ref[k]), rel(emu[k], grads_ref[k])
        errs.append(e)
        if e > max(2e-2, 4 * ee):
            bad[k] = (e, ee)
    assert not bad, bad
    return float(np.median(errs))


def test_fp16_tiramisu_config4_topology_matches_oracle():
    from oracle import deskdl_port as O
    from paper_1810_01993_b200.models import tiramisu_config4
    from paper_1810_01993_b200.net import MiniDenseNet
    from paper_1810_01993_b200.scenes import SceneConfig, generated_batch
    net = MiniDenseNet(tiramisu_config4(), seed=0, precision="fp16")
    x, labels = generated_batch(SceneConfig(height=64, width=48), seed=1, step=0, rank=0, local_batch=2)
    med = _check(net, x, labels, O.class_weights((0.982, 0.017, 0.001)))
    assert med < 1e-2


def test_fp16_deeplab_config1_matches_oracle():
    """Config 1's DeepLabV3+ in fp16 storage; fp16 keeps 3 more mantissa bits than bf16, so its
    median gradient error is well below the bf16 run's (~1.4e-2)."""
    from oracle import deskdl_port as O
    from paper_1810_01993_b200.models import DeepLabConfig
    from paper_1810_01993_b200.net import DeepLabV3Plus
    from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng
    net = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp16")
    f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
    med = _check(net, f[None], lab[None], O.class_weights((0.982, 0.017, 0.001)))
    assert med < 1e-2


def test_fp16_conv_kernel_vs_fp64():
    from paper_1810_01993_b200 import _lib, nhwc
    import torch.nn.functional as F
    torch.manual_seed(3)
    n, h, w, c, k = 2, 32, 48, 128, 3
    x = torch.randn(n, h, w, c, device="cuda").half()
    wm = (torch.randn(k * k, c, 256, device="cuda") / (k * k * c) ** 0.5).half()
    y = torch.empty(n, h, w, 256, dtype=torch.float16, device="cuda")
    with _lib.use("fp16"):
        nhwc.conv_fprop(nhwc.View(x), None, 256, k, k, 2, nhwc.View(y), w_master=wm, w_mode=1)
    ref = F.conv2d(x.permute(0, 3, 1, 2).double(), wm.double().view(k, k, c, 256).permute(3, 2, 0, 1),
                   padding=2, dilation=2)
    e = float((y.permute(0, 3, 1, 2).double() - ref).abs().max() / ref.abs().max())
    assert e < 2e-3, e   # fp16 output rounding (bf16 would be ~8e-3)
