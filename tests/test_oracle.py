"""Pin the CPU oracle (oracle/) and the host-side model definitions against
golden vectors produced by the reference itself (tests/golden/make_golden.py).
CPU only."""

import os

import numpy as np
import pytest

from oracle import deskdl_port as O
from paper_1810_01993_b200 import flops, models, scenes
from paper_1810_01993_b200.graph import OpGraph, ShapeError, infer_shapes

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def rel(a, b):
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


def test_conv_matches_reference_golden():
    d = load("conv.npz")
    for i, (n, cin, h, w, cout, k, dil) in enumerate(d["cases"]):
        for dt, tol in (("float64", 1e-12), ("float32", 1e-5)):
            t = f"c{i}_{dt}"
            y, cols = O.conv2d_forward(d[t + "_x"], d[t + "_w"], dilation=int(dil))
            assert rel(y, d[t + "_y"]) < tol
            assert rel(O.conv2d_backward_weights(cols, d[t + "_dy"], d[t + "_w"].shape), d[t + "_dw"]) < tol
            assert rel(O.conv2d_backward_input(d[t + "_dy"], d[t + "_w"], d[t + "_x"].shape, dilation=int(dil)),
                       d[t + "_dx"]) < tol


def test_conv_loops_match_golden():
    d = load("conv.npz")
    for i, (*_, dil) in enumerate(d["cases"]):
        t = f"c{i}_float64"
        assert rel(O.conv2d_loops(d[t + "_x"], d[t + "_w"], int(dil)), d[t + "_y"]) < 1e-12


def test_conv_validation():
    x = np.zeros((1, 2, 4, 4), np.float32)
    with pytest.raises(NotImplementedError):
        O.conv2d_forward(x, np.zeros((2, 2, 3, 3), np.float32), stride=2)
    with pytest.raises(ValueError):
        O.conv2d_forward(x, np.zeros((2, 3, 3, 3), np.float32))


def test_weighted_ce_matches_golden():
    d = load("loss.npz")
    for i in range(3):
        loss, dl = O.weighted_ce_loss(d[f"l{i}_logits"], d[f"l{i}_labels"], d["weights"])
        assert abs(loss - float(d[f"l{i}_loss"])) <= 1e-6 * abs(float(d[f"l{i}_loss"]))
        assert rel(dl, d[f"l{i}_dlogits"]) < 1e-6
        assert np.array_equal(np.argmax(d[f"l{i}_logits"], axis=1).astype(np.uint8), d[f"l{i}_argmax"])
    assert np.array_equal(d["tie_argmax"], np.array([[[1, 0], [0, 0]]], np.uint8))


def test_uniform_logits_give_ln3():
    lab = np.random.default_rng(4).integers(0, 3, size=(2, 5, 5))
    loss, _ = O.weighted_ce_loss(np.zeros((2, 3, 5, 5)), lab, O.class_weights((0.982, 0.017, 0.001), np.float64))
    assert abs(loss - np.log(3)) < 1e-12


def test_larc_bitwise_matches_golden():
    d = load("larc.npz")
    for ci in range(3):
        for li in range(6):
            t = f"o{ci}_{li}"
            lr, mom, trust, wd, eps = d[t + "_cfg"]
            w, m = d[t + "_w0"].copy(), d[t + "_m0"].copy()
            lrs = [O.larc_sgd_step(w, m, d[t + "_g"], lr=lr, momentum=mom, trust=trust, weight_decay=wd, eps=eps)
                   for _ in range(3)]
            assert np.allclose(lrs, d[t + "_lr"], rtol=0, atol=0)
            assert w.tobytes() == d[t + "_w3"].tobytes()
            assert m.tobytes() == d[t + "_m3"].tobytes()


def test_larc_hand_example():
    assert abs(O.larc_effective_lr(np.array([2.0, 0.0]), np.array([0.0, 1.0])) - 0.04) < 1e-12
    with pytest.raises(FloatingPointError):
        O.larc_effective_lr(np.array([np.inf]), np.ones(1))


def test_scenes_bitwise_match_reference():
    d = load("scenes.npz")
    for i in range(2):
        c, h, w = (int(v) for v in d[f"s{i}_shape"])
        kw = dict(channels=c, height=h, width=w)
        if c < 16:
            kw.update(streak_channels=(0, 1), blob_channels=(2, 3))
        cfg = scenes.SceneConfig(**kw)
        for t, j in [(0, 0), (3, 1)]:
            f, lab = scenes.make_scene(cfg, scenes.scene_rng(0, t, j))
            assert f.tobytes() == d[f"s{i}_{t}_{j}_field"].tobytes()
            assert lab.tobytes() == d[f"s{i}_{t}_{j}_labels"].tobytes()
            assert np.array_equal(scenes.class_counts(lab), d[f"s{i}_{t}_{j}_counts"])


def _oracle_step(graph, params, order, d, head, lossn):
    cw = O.class_weights((0.982, 0.017, 0.001))
    return O.train_step(graph, {k: v.copy() for k, v in params.items()}, order, d["x"], d["labels"], cw,
                        lossn, head)


def test_minidensenet_init_and_grads_match_reference():
    d = load("minidensenet.npz")
    graph, params, head, lossn = models.build_minidensenet(
        models.NetConfig(channels_in=8, growth=16, block_layers=2, levels=2), seed=3)
    order = list(params)
    assert order == list(d["order"])
    for k in order:
        assert params[k].tobytes() == d[f"p:{k}"].tobytes(), k
    loss, logits, grads, _ = _oracle_step(graph, params, order, d, head, lossn)
    assert abs(loss - float(d["loss"])) < 1e-5 * abs(float(d["loss"]))
    assert rel(logits, d["logits"]) < 1e-5
    for k in order:
        assert rel(grads[k], d[f"g:{k}"]) < 1e-4, k


def test_deeplab_small_oracle_matches_reference_executor():
    d = load("deeplab_small.npz")
    graph, params, head, lossn = models.build_deeplab(models.deeplab_small(), seed=5)
    order = list(params)
    assert order == list(d["order"])
    for k in order:
        assert params[k].tobytes() == d[f"p:{k}"].tobytes(), k
    loss, logits, grads, _ = _oracle_step(graph, params, order, d, head, lossn)
    assert abs(loss - float(d["loss"])) < 1e-5 * abs(float(d["loss"]))
    for k in order:
        assert rel(grads[k], d[f"g:{k}"]) < 1e-4, k


def test_flops_match_reference():
    d = load("flops.npz")
    g = OpGraph()
    g.add_input("x")
    g.add_input("w", role="param")
    g.conv2d("x", "w", "c", kh=3, kw=3, cin=48, cout=32)
    assert flops.count_graph(g, {"x": (2, 48, 1152, 768), "w": (32, 48, 3, 3)}, 2).total == int(d["worked"])
    assert int(d["worked"]) == 48_922_361_856
    for tag, cfg in [("deeplab", models.DeepLabConfig()), ("deeplab_small", models.deeplab_small())]:
        graph, params, _, _ = models.build_deeplab(cfg, seed=0)
        for h, w in [(1152, 768), (288, 192)]:
            shapes = {k: v.shape for k, v in params.items()}
            shapes.update(x=(2, 16, h, w), labels=(2, h, w), class_weights=(3,))
            rep = flops.count_graph(graph, shapes, batch=2)
            assert rep.total == int(d[f"{tag}_{h}x{w}_fwd"])
            assert flops.train_flops_per_sample(rep) == float(d[f"{tag}_{h}x{w}_train_per_sample"])
            assert O.graph_flops(graph, infer_shapes(graph, shapes)) == rep.total


def test_shape_errors():
    g = OpGraph()
    g.add_input("x")
    g.avgpool("x", "p", window=2)
    with pytest.raises(ShapeError):
        infer_shapes(g, {"x": (1, 2, 5, 4)})
    with pytest.raises(ValueError):
        g.add_input("x")


def _oracle_train(net_cfg, scene_cfg, world, lb, lag, steps, seed, lr):
    """Data-parallel step semantics (trainer.py:343-405) on the oracle: per-rank
    grads of each rank's slice, mean over ranks (collectives.py:196-197), LARC."""
    graph, params, head, lossn = models.build_minidensenet(net_cfg, seed=seed)
    order = list(params)
    moms = {k: np.zeros_like(v) for k, v in params.items()}
    cw = O.class_weights((0.982, 0.017, 0.001))
    losses, pending = [], None
    for t in range(steps):
        rank_grads, rank_loss = [], []
        for r in range(world):
            x, lab = scenes.generated_batch(scene_cfg, seed, t, r, lb)
            loss, _, grads, _ = O.train_step(graph, params, order, x, lab, cw, lossn, head)
            rank_grads.append(grads)
            rank_loss.append(loss)
        mean = {k: (np.sum([g[k] for g in rank_grads], axis=0, dtype=np.float32)
                    * np.float32(1.0 / world)).astype(np.float32) for k in order}
        losses.append(float(np.mean(rank_loss)))
        if lag == 0:
            apply = mean
        else:
            apply, pending = pending, mean
        if apply is not None:
            for k in order:
                O.larc_sgd_step(params[k], moms[k], apply[k], lr=lr)
    if lag == 1:
        for k in order:
            O.larc_sgd_step(params[k], moms[k], pending[k], lr=lr)
    return losses, params


@pytest.mark.parametrize("lag", [0, 1])
@pytest.mark.parametrize("world,lb", [(1, 2), (2, 1)])
def test_oracle_dp_trainer_matches_reference_trainer(lag, world, lb):
    d = load("trainer.npz")
    scene_cfg = scenes.SceneConfig(channels=8, height=16, width=16, streak_channels=(0, 1), blob_channels=(2, 3))
    net = models.NetConfig(channels_in=8, growth=16, block_layers=1, levels=1)
    losses, params = _oracle_train(net, scene_cfg, world, lb, lag, 3, 4, 0.1)
    tag = f"lag{lag}_w{world}"
    assert np.allclose(losses, d[tag + "_losses"], rtol=1e-5, atol=0)
    for k, v in params.items():
        assert rel(v, d[f"{tag}_state:{k}"]) < 1e-4, k


# ---- north-star extensions (no reference implementation): pinned by finite differences
def _fd_check(fn, args, gout, analytic, idx_arg, h=1e-6, n=12, seed=0):
    rng = np.random.default_rng(seed)
    a = args[idx_arg]
    flat = a.reshape(-1)
    for i in rng.choice(flat.size, size=min(n, flat.size), replace=False):
        old = flat[i]
        flat[i] = old + h
        fp = float((fn(*args) * gout).sum())
        flat[i] = old - h
        fm = float((fn(*args) * gout).sum())
        flat[i] = old
        num = (fp - fm) / (2 * h)
        assert abs(num - analytic.reshape(-1)[i]) <= 1e-6 * max(1.0, abs(num)), (idx_arg, i, num)


def test_batchnorm_oracle_vjp_matches_finite_differences():
    from oracle import deskdl_port as O
    rng = np.random.default_rng(1)
    x = rng.normal(size=(2, 3, 4, 5)) * 2 + 1
    gamma, beta = rng.normal(size=3), rng.normal(size=3)
    g = rng.normal(size=x.shape)
    y, cache = O.batchnorm_forward(x, gamma, beta, 1e-5)
    assert np.allclose(y.mean(axis=(0, 2, 3)), beta) and np.allclose(y.std(axis=(0, 2, 3)), np.abs(gamma), rtol=1e-4)
    gx, gg, gb = O.batchnorm_backward(g, cache, gamma)
    f = lambda x_, ga, be: O.batchnorm_forward(x_, ga, be, 1e-5)[0]  # noqa: E731
    _fd_check(f, [x, gamma, beta], g, gx, 0)
    _fd_check(f, [x, gamma, beta], g, gg, 1, n=3)
    _fd_check(f, [x, gamma, beta], g, gb, 2, n=3)


@pytest.mark.parametrize("f", [2, 4])
def test_bilinear_oracle_matches_torch_and_finite_differences(f):
    import torch
    from oracle import deskdl_port as O
    rng = np.random.default_rng(2)
    x = rng.normal(size=(2, 3, 5, 7))
    y = O.bilinear_upsample(x, f)
    ref = torch.nn.functional.interpolate(torch.from_numpy(x), scale_factor=f, mode="bilinear", align_corners=False)
    assert np.allclose(y, ref.numpy(), atol=1e-12)
    g = rng.normal(size=y.shape)
    gx = O.bilinear_upsample_backward(g, f, x.shape)
    _fd_check(lambda x_: O.bilinear_upsample(x_, f), [x], g, gx, 0)
