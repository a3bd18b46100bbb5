"""Graphs using the op kinds outside conv-bias-relu chains -- standalone bias_add / relu,
elementwise mul / scale, width-axis matmul, a bias-less conv (ops.py:115-148, VJPs :152-203) --
through the engine vs the oracle restatement of the reference's executor: fp32 mode at the
north-star 1e-3, bf16 mode at 2e-2 (max|a-b| / max|b| per tensor, test_kernels.py:17-19)."""

import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("which", ["build", "build_wide"])
@pytest.mark.parametrize("precision,tol", [("fp32", 1e-3), ("bf16", 2e-2)])
def test_generic_graph_matches_oracle(which, precision, tol):
    import generic_graph
    from oracle import deskdl_port as O
    from paper_1810_01993_b200.engine import Engine
    g, p, logits, loss = getattr(generic_graph, which)(seed=3)
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 8, 16, 16)).astype(np.float32)
    lab = rng.integers(0, 3, size=(2, 16, 16)).astype(np.uint8)
    cw = np.array([1.0, 7.7, 31.6], np.float32)
    order = list(p)
    ref_loss, ref_logits, ref_grads, _ = O.train_step(g, {k: v.copy() for k, v in p.items()}, order, x, lab, cw,
                                                       loss, logits)
    eng = Engine(g, p, order, x.shape, loss, logits, precision=precision)
    eng.set_batch(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda())
    eng.set_class_weights(cw)
    eng.forward()
    eng.backward()
    torch.cuda.synchronize()
    got_loss = float(eng.loss.item())
    assert abs(got_loss - ref_loss) <= tol * abs(ref_loss), (got_loss, ref_loss)
    assert rel(eng.logits_nchw().cpu().numpy(), ref_logits) < tol
    grads = eng.export_grads()
    errs = {k: rel(grads[k], ref_grads[k]) for k in order}
    bound = {k: tol for k in order}
    if precision == "bf16":
        # as tests/test_gpu_model.py: where an ideal bf16-storage implementation (bf16 rounding at
        # exactly the engine's stored tensors, oracle/bf16_emulation.py) is itself worse than the
        # bar -- cancellation in a gradient summed over many terms of both signs -- the GPU may be
        # at most 4x that emulation's error
        from oracle.bf16_emulation import emulated_grads
        stored = {o.out for o in eng.plan.ops}
        _, emu = emulated_grads(g, p, x, lab, cw, loss, stored=stored)
        bound = {k: max(tol, 4.0 * rel(emu[k], ref_grads[k])) for k in order}
    bad = {k: (e, bound[k]) for k, e in errs.items() if e > bound[k]}
    assert not bad, (bad, errs)
