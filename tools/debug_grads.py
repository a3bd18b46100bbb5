"""Per-tensor gradient error of the GPU path vs the golden reference (development aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1810_01993_b200.loss import ClassWeights  # noqa: E402
from paper_1810_01993_b200.models import NetConfig, deeplab_small  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus, MiniDenseNet  # noqa: E402

G = "tests/golden"


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


for fname, net in [("minidensenet.npz", MiniDenseNet(NetConfig(channels_in=8), seed=3)),
                   ("deeplab_small.npz", DeepLabV3Plus(deeplab_small(), seed=5))]:
    d = np.load(os.path.join(G, fname))
    loss, logits, tape = net.forward_loss(d["x"], d["labels"], ClassWeights((0.982, 0.017, 0.001)).vector())
    grads = net.backward(tape)
    print(fname, "loss", loss, float(d["loss"]))
    for k in net.param_order:
        e = rel(grads[k], d[f"g:{k}"])
        flag = " <<<" if e > 2e-2 else ""
        print(f"  {k:28s} {str(d[f'g:{k}'].shape):20s} {e:.2e}{flag}")
