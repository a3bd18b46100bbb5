"""fp32 parity diagnostic (config 1): GPU fp32 and the reference-arithmetic fp32 oracle, each
against the same oracle in float64 (development aid; run from the repo root on a GPU box)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import deskdl_port as O  # noqa: E402
from paper_1810_01993_b200.models import DeepLabConfig  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus  # noqa: E402
from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


net = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp32")
f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
x, labels = f[None], lab[None]
cw = O.class_weights((0.982, 0.017, 0.001))
l32, lg32, g32, _ = O.train_step(net.graph, net.params, net.param_order, x, labels, cw, net.loss_name, net.logits_name)
p64 = {k: v.astype(np.float64) for k, v in net.params.items()}
l64, lg64, g64, _ = O.train_step(net.graph, p64, net.param_order, x.astype(np.float64), labels,
                                 cw.astype(np.float64), net.loss_name, net.logits_name)
loss, logits, tape = net.forward_loss(x, labels, cw)
gg = net.backward(tape)
print("loss  ref32 %.3e  gpu32 %.3e" % (abs(l32 - l64) / abs(l64), abs(loss - l64) / abs(l64)))
print("logits ref32 %.3e  gpu32 %.3e" % (rel(lg32, lg64), rel(logits.cpu().numpy(), lg64)))
rows = []
for k in net.param_order:
    rows.append((rel(gg[k], g64[k]), rel(g32[k], g64[k]), rel(gg[k], g32[k]), k))
rows.sort(reverse=True)
print("tensor  gpu32-vs-f64  ref32-vs-f64  gpu32-vs-ref32")
for r in rows[:15]:
    print("%-22s %.3e %.3e %.3e" % (r[3], r[0], r[1], r[2]))
a = np.array([r[0] for r in rows])
b = np.array([r[1] for r in rows])
print("median gpu32 %.3e ref32 %.3e ; max gpu32 %.3e ref32 %.3e" % (np.median(a), np.median(b), a.max(), b.max()))
