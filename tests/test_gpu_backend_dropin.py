"""B1 drop-in, end to end: the reference package itself (`deskdl`, installed unmodified into
baseline/_ref by `pip install --target baseline/_ref`) running on the GPU backend.

* The cases of the reference's own kernel tests (pkg/tests/test_kernels.py:28-110) at the
  reference's tolerances, with `paper_1810_01993_b200.backend` in the role of a backend:
  float64 forward vs the direct-loop oracle < 1e-12 (:28-38), float32 agreement with deskdl's
  python and cython backends < 1e-5 (:41-58), dW and dx vs central differences < 1e-7
  (:61-82), dilation changes the result (:85-92), stride / channel validation (:95-110).
* `backend.install()` rebinds deskdl's kernel selector (kernels.py:19-40, what a
  DESKDL_KERNELS=b200 branch would do) and deskdl's OWN executor (ops.run_forward /
  run_backward, ops.py:44-106) and model (MiniDenseNet.forward_loss / backward, net.py:132-157)
  run through it, against the same calls on deskdl's stock backend.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def deskdl():
    if not os.path.isdir(os.path.join(REF, "deskdl")):
        pytest.skip("baseline/_ref has no deskdl install (pip install --target baseline/_ref)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import deskdl  # noqa: F401
    from deskdl.model import kernels
    return kernels


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


def _fd(fn, x, eps=1e-6):
    """Central differences in float64 (restates pkg/tests/reference.py:97-111)."""
    x = np.array(x, dtype=np.float64)
    g = np.zeros_like(x)
    flat, gf = x.reshape(-1), g.reshape(-1)
    for i in range(flat.size):
        keep = flat[i]
        flat[i] = keep + eps
        up = fn(x)
        flat[i] = keep - eps
        dn = fn(x)
        flat[i] = keep
        gf[i] = (up - dn) / (2 * eps)
    return g


def test_forward_matches_loop_oracle_float64(deskdl):
    from oracle.deskdl_port import conv2d_loops
    from paper_1810_01993_b200 import backend
    rng = np.random.default_rng(7)
    for n, cin, h, w, cout, k, dil in [(1, 2, 5, 4, 3, 3, 1), (2, 3, 7, 6, 2, 3, 2), (1, 4, 6, 6, 5, 1, 1),
                                       (2, 16, 12, 10, 8, 7, 1), (1, 5, 9, 11, 4, 3, 4)]:
        x = rng.standard_normal((n, cin, h, w))
        wgt = rng.standard_normal((cout, cin, k, k))
        got, _ = backend.conv2d_forward(x, wgt, dilation=dil)
        want = conv2d_loops(x, wgt, dilation=dil)
        assert got.dtype == np.float64 and got.shape == want.shape
        assert _rel(got, want) < 1e-12, (n, cin, h, w, cout, k, dil, _rel(got, want))


def test_backends_agree_forward_backward_float32(deskdl):
    from paper_1810_01993_b200 import backend
    rng = np.random.default_rng(8)
    x = rng.standard_normal((2, 5, 9, 7)).astype(np.float32)
    wgt = rng.standard_normal((4, 5, 3, 3)).astype(np.float32)
    dy = rng.standard_normal((2, 4, 9, 7)).astype(np.float32)
    outs = {}
    impls = dict(deskdl.available_backends())
    impls["b200"] = backend
    for name, impl in impls.items():
        y, cache = impl.conv2d_forward(x, wgt)
        dw = impl.conv2d_backward_weights(cache, dy, wgt.shape)
        dx = impl.conv2d_backward_input(dy, wgt, x.shape)
        outs[name] = (y, dw, dx)
    for name in impls:
        if name == "b200":
            continue
        for ta, tb in zip(outs["b200"], outs[name]):
            assert ta.dtype == tb.dtype == np.float32
            assert _rel(ta.astype(np.float64), tb.astype(np.float64)) < 1e-5, name


def test_backward_weights_matches_fd(deskdl):
    from paper_1810_01993_b200 import backend
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1, 2, 5, 4))
    wgt = rng.standard_normal((3, 2, 3, 3))
    y, cache = backend.conv2d_forward(x, wgt)
    dw = backend.conv2d_backward_weights(cache, np.ones_like(y), wgt.shape)
    fd = _fd(lambda v: float(backend.conv2d_forward(x, v)[0].sum()), wgt)
    assert _rel(dw, fd) < 1e-7


def test_backward_input_matches_fd(deskdl):
    from paper_1810_01993_b200 import backend
    rng = np.random.default_rng(10)
    x = rng.standard_normal((1, 3, 4, 5))
    wgt = rng.standard_normal((2, 3, 3, 3))
    y, _ = backend.conv2d_forward(x, wgt, dilation=2)
    dx = backend.conv2d_backward_input(np.ones_like(y), wgt, x.shape, dilation=2)
    fd = _fd(lambda v: float(backend.conv2d_forward(v, wgt, dilation=2)[0].sum()), x)
    assert _rel(dx, fd) < 1e-7


def test_dilation_changes_result_and_validation(deskdl):
    from paper_1810_01993_b200 import backend
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 2, 8, 8))
    wgt = rng.standard_normal((2, 2, 3, 3))
    y1, _ = backend.conv2d_forward(x, wgt, dilation=1)
    y2, _ = backend.conv2d_forward(x, wgt, dilation=2)
    assert _rel(y1, y2) > 1e-3
    xf = x.astype(np.float32)
    with pytest.raises(NotImplementedError):
        backend.conv2d_forward(xf, wgt.astype(np.float32), stride=2)
    with pytest.raises(NotImplementedError):
        backend.conv2d_backward_input(xf, wgt.astype(np.float32), xf.shape, stride=2)
    with pytest.raises(ValueError):
        backend.conv2d_forward(xf, rng.standard_normal((2, 3, 3, 3)).astype(np.float32))


def _deskdl_step(dtype):
    """deskdl's own MiniDenseNet step (forward_loss + backward, net.py:132-157) on its own
    executor, whatever backend kernels.py currently binds."""
    from deskdl.model import MiniDenseNet, NetConfig, SceneConfig, make_scene
    net = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=2, levels=2), seed=5)
    sc = SceneConfig(channels=8, height=32, width=24, streak_channels=(0, 1), blob_channels=(2, 3))
    scenes = [make_scene(sc, np.random.default_rng((5, 0, 0, j)), f"s{j}") for j in range(2)]
    x = np.stack([s.field for s in scenes]).astype(dtype)
    lab = np.stack([s.labels for s in scenes])
    params = {k: v.astype(dtype) for k, v in net.params.items()}
    cw = np.array([1.0, 7.7, 31.6], dtype=dtype)
    loss, logits, tape = net.forward_loss(x, lab, cw, params=params)
    grads = net.backward(tape)
    return loss, logits, grads


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 1e-4)])
def test_deskdl_own_model_step_runs_on_b200_backend(deskdl, dtype, tol):
    from paper_1810_01993_b200 import backend
    import deskdl.model.ops as ops
    calls = {"n": 0}
    stock_fwd = deskdl.conv2d_forward
    loss0, logits0, grads0 = _deskdl_step(dtype)
    handle = backend.install(deskdl)
    try:
        assert deskdl.BACKEND == "b200" and ops.kernels is deskdl
        orig = deskdl.conv2d_forward

        def counted(*a, **k):
            calls["n"] += 1
            return orig(*a, **k)
        deskdl.conv2d_forward = counted
        loss1, logits1, grads1 = _deskdl_step(dtype)
    finally:
        backend.uninstall(handle)
    assert deskdl.conv2d_forward is stock_fwd
    assert calls["n"] > 0                      # the executor really called the GPU backend
    assert abs(loss1 - loss0) <= tol * abs(loss0)
    assert logits1.dtype == logits0.dtype == dtype
    assert _rel(logits1, logits0) < tol
    for k, g in grads0.items():
        assert grads1[k].dtype == g.dtype
        assert _rel(grads1[k], g) < max(tol, 1e-9 if dtype == np.float64 else 1e-4), k
