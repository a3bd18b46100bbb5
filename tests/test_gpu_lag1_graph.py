"""Lag 1 (trainer.py:378-383,403-405: apply the previous step's reduced gradients) captured as two
alternating CUDA graphs gives bitwise the same trajectory as the eager lag-1 loop, staged or not."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(captured: bool, staged: bool = False, steps: int = 6):
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.net import MiniDenseNet
    from paper_1810_01993_b200.optimizer import OptimConfig
    from paper_1810_01993_b200.scenes import SceneConfig, generated_batch
    from paper_1810_01993_b200.trainer import DataParallelTrainer
    sc = SceneConfig(channels=8, height=32, width=32, streak_channels=(0, 1), blob_channels=(2, 3))
    net = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=2, levels=2), seed=2)
    batches = [generated_batch(sc, 2, t, 0, 2) for t in range(steps)]
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()) for x, lab in batches]
    tr = DataParallelTrainer(net, OptimConfig(lr=0.05), dev[0][0].shape, lag=1)
    losses = [float(tr.step(*dev[0]).item())]
    if captured:
        tr.capture(*dev[0], buffers=2 if staged else 1)
    for t in range(1, steps):
        if staged:
            host = [(b[0].cpu().pin_memory(), b[1].cpu().pin_memory()) for b in dev]
            tr.stage(*host[t])
            loss = tr.step_staged()
        else:
            loss = tr.step(*dev[t])
        losses.append(float(loss.item()))
    tr.finish()
    tr.check_status()
    torch.cuda.synchronize()
    state = tr.eng.export_params()
    tr.release_graph()
    return losses, state, tr.steps_done


@pytest.mark.parametrize("staged", [False, True])
def test_lag1_graph_matches_eager(staged):
    l0, s0, n0 = _run(False)
    l1, s1, n1 = _run(True, staged)
    assert n0 == n1 == 6
    assert l0 == l1, (l0, l1)
    for k in s0:
        assert np.array_equal(s0[k], s1[k]), k
