"""Resume from a training-state checkpoint: N steps straight == K steps, save,
fresh trainer, load, N-K steps -- bitwise, for lag 0 and lag 1 (the pending reduced gradient of
a lag-1 run travels in the file)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _trainer(lag):
    from paper_1810_01993_b200.loss import ClassWeights
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.net import MiniDenseNet
    from paper_1810_01993_b200.optimizer import OptimConfig
    from paper_1810_01993_b200.trainer import DataParallelTrainer
    net = MiniDenseNet(NetConfig(channels_in=8, growth=16, block_layers=1, levels=1), seed=4)
    return DataParallelTrainer(net, OptimConfig(lr=0.1), (2, 8, 16, 16), lag=lag,
                               class_weights=ClassWeights((0.982, 0.017, 0.001)).vector())


def _batch(t):
    from paper_1810_01993_b200.scenes import SceneConfig, generated_batch
    sc = SceneConfig(channels=8, height=16, width=16, streak_channels=(0, 1), blob_channels=(2, 3))
    x, lab = generated_batch(sc, 4, t, 0, 2)
    return torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()


@pytest.mark.parametrize("lag", [0, 1])
def test_resume_is_bitwise(lag, tmp_path):
    from paper_1810_01993_b200.checkpoint import load_train_state, save_train_state
    a = _trainer(lag)
    for t in range(4):
        a.step(*_batch(t))
    a.finish()
    straight = a.eng.export_params()

    b = _trainer(lag)
    for t in range(2):
        b.step(*_batch(t))
    p = str(tmp_path / "state.ckpt")
    save_train_state(p, b)
    c = _trainer(lag)
    load_train_state(p, c)
    assert c.steps_done == 2
    for t in range(2, 4):
        c.step(*_batch(t))
    c.finish()
    resumed = c.eng.export_params()
    for k in straight:
        assert np.array_equal(straight[k], resumed[k]), k


def test_prefetch_pipeline_run_is_identical():
    """train_run fed by the W-worker prefetch pipeline (pinned host batches, step order) follows
    exactly the trajectory of the synchronous feed."""
    from paper_1810_01993_b200.models import NetConfig
    from paper_1810_01993_b200.optimizer import OptimConfig
    from paper_1810_01993_b200.scenes import SceneConfig
    from paper_1810_01993_b200.trainer import RunConfig, train_run
    sc = SceneConfig(channels=8, height=16, width=16, streak_channels=(0, 1), blob_channels=(2, 3))
    base = dict(lag=0, steps=4, local_batch=2, seed=4, optim=OptimConfig(lr=0.1),
                net=NetConfig(channels_in=8, growth=16, block_layers=1, levels=1), scene=sc)
    a = train_run(RunConfig(**base))
    b = train_run(RunConfig(**base, prefetch_workers=3, prefetch_capacity=2))
    assert a.losses == b.losses
    for k in a.state:
        assert np.array_equal(a.state[k], b.state[k]), k
