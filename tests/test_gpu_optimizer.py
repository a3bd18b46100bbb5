"""Known-answer tests of the reference optimizer (pkg/tests/test_optimizer.py), restated against
the device implementation (multi-tensor LARC kernel behind paper_1810_01993_b200.optimizer)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _w(p):
    return p.w.cpu().numpy()


def test_larc_hand_example():
    from paper_1810_01993_b200.optimizer import OptimConfig, larc_effective_lr
    # |w| = 2, |g| = 1, trust 0.02 -> 0.04
    lr = larc_effective_lr(np.array([2.0, 0.0], np.float32), np.array([0.0, 1.0], np.float32),
                           OptimConfig(lr=1.0, trust=0.02))
    assert abs(lr - 0.04) < 1e-7


def test_larc_clips_and_falls_back_to_global_rate():
    from paper_1810_01993_b200.optimizer import OptimConfig, larc_effective_lr
    assert larc_effective_lr(np.ones(4, np.float32), np.zeros(4, np.float32), OptimConfig(lr=0.5)) == 0.5
    # the device returns the rate as the float32 it applies (w -= f32(lr_eff) * m)
    assert larc_effective_lr(np.zeros(3, np.float32), np.ones(3, np.float32), OptimConfig(lr=0.3)) == \
        float(np.float32(0.3))
    with pytest.raises(FloatingPointError):
        larc_effective_lr(np.array([np.inf], np.float32), np.ones(1, np.float32), OptimConfig())


def test_sgd_plain_and_zero_gradient():
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, sgd_step
    p = LayerParam("w", np.array([1.0, 2.0], np.float32))
    sgd_step(p, np.array([0.5, -0.5], np.float32), 0.1, OptimConfig(lr=1.0, momentum=0.0))
    assert np.allclose(_w(p), [0.95, 2.05])
    q = LayerParam("w", np.array([3.0], np.float32))
    sgd_step(q, np.zeros(1, np.float32), 0.1, OptimConfig())
    assert _w(q)[0] == 3.0
    with pytest.raises(ValueError):
        sgd_step(q, np.zeros(4, np.float32), 0.1, OptimConfig())


def test_momentum_two_step_closed_form():
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, sgd_step
    g = np.array([1.0], np.float32)
    p = LayerParam("w", np.array([10.0], np.float32))
    cfg = OptimConfig(lr=1.0, momentum=0.9)
    sgd_step(p, g, 0.1, cfg)
    w1 = 10.0 - 0.1
    assert abs(_w(p)[0] - w1) < 1e-6
    sgd_step(p, g, 0.1, cfg)
    assert abs(_w(p)[0] - (w1 - 0.1 * 1.9)) < 1e-6


def test_weight_decay_folds_into_momentum():
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, sgd_step
    p = LayerParam("w", np.array([2.0], np.float32))
    sgd_step(p, np.zeros(1, np.float32), 0.5, OptimConfig(lr=1.0, momentum=0.0, weight_decay=0.1))
    assert abs(_w(p)[0] - 1.9) < 1e-6


def test_lag1_buffers_then_applies_previous_gradient():
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, lagged_apply, larc_sgd_step
    p = LayerParam("w", np.array([1.0], np.float32))
    cfg = OptimConfig(lr=10.0, trust=1000.0, momentum=0.0, lag=1)
    assert not lagged_apply(p, np.array([0.25], np.float32), cfg)
    assert _w(p)[0] == 1.0
    assert lagged_apply(p, np.array([0.125], np.float32), cfg)
    q = LayerParam("w", np.array([1.0], np.float32))
    larc_sgd_step(q, np.array([0.25], np.float32), OptimConfig(lr=10.0, trust=1000.0, momentum=0.0))
    assert _w(p)[0] == _w(q)[0]


def test_lag_shift_equivalence_bitwise():
    """Weight-independent gradient stream: the lag-1 trajectory is the lag-0 one delayed a step."""
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, lagged_apply
    rng = np.random.default_rng(17)
    stream = [rng.normal(size=6).astype(np.float32) for _ in range(40)]
    base = rng.normal(size=6).astype(np.float32)
    p0, p1 = LayerParam("w", base), LayerParam("w", base)
    c0 = OptimConfig(lr=0.05, momentum=0.9, trust=0.02, lag=0)
    c1 = OptimConfig(lr=0.05, momentum=0.9, trust=0.02, lag=1)
    h0, h1 = [], []
    for g in stream:
        lagged_apply(p0, g, c0)
        h0.append(_w(p0).tobytes())
        lagged_apply(p1, g, c1)
        h1.append(_w(p1).tobytes())
    assert h1[0] == base.tobytes()
    for t in range(1, len(stream)):
        assert h1[t] == h0[t - 1], t


def test_update_magnitude_bound():
    """|dw| <= min(lr, trust |w| / |g|) |m| on sampled layers (no decay)."""
    from paper_1810_01993_b200.optimizer import LayerParam, OptimConfig, larc_sgd_step
    rng = np.random.default_rng(99)
    cfg = OptimConfig(lr=0.7, momentum=0.9, trust=0.02)
    for _ in range(200):
        n = int(rng.integers(1, 40))
        w = (rng.normal(size=n) * rng.uniform(0.01, 10)).astype(np.float32)
        g = (rng.normal(size=n) * rng.uniform(0.001, 100)).astype(np.float32)
        p = LayerParam("w", w)
        lr = larc_sgd_step(p, g, cfg)
        bound = min(0.7, 0.02 * np.linalg.norm(w) / np.linalg.norm(g))
        assert lr <= bound * (1 + 1e-5)
        assert np.linalg.norm(_w(p) - w) <= lr * np.linalg.norm(g) * (1 + 1e-4) + 1e-12


def test_zero_head_gives_ln3_and_class_equal_logits():
    """Reference test_model.py:178-184 / 260-270 on the GPU path: a zeroed head makes every logit 0
    (uniform softmax -> loss ln 3 for any class weights); zero input + zero biases -> class-equal."""
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.net import MiniDenseNet
    net = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=1, levels=1), seed=2)
    st = net.state_dict()
    st["head.w"][:] = 0
    net.load_state(st)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(2, 8, 16, 16)).astype(np.float32)
    lab = rng.integers(0, 3, size=(2, 16, 16)).astype(np.uint8)
    loss, logits, _ = net.forward_loss(x, lab, np.array([1.0, 7.5, 31.6], np.float32))
    assert abs(loss - np.log(3.0)) < 1e-6
    assert float(torch.abs(logits).max()) == 0.0
    net2 = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=1, levels=1), seed=2)
    lg = net2.forward(np.zeros((1, 8, 16, 16), np.float32)).cpu().numpy()
    assert np.allclose(lg, lg[:, :1], atol=0)
