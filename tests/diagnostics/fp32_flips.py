"""Count relu sign flips between the GPU fp32 forward, the fp32 oracle and the float64 oracle
on config 1 (development aid)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import deskdl_port as O  # noqa: E402
from paper_1810_01993_b200.models import DeepLabConfig  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus  # noqa: E402
from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng  # noqa: E402

net = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp32")
f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
x, labels = f[None], lab[None]
cw = O.class_weights((0.982, 0.017, 0.001))
vals = dict(net.params)
vals.update(x=x, labels=labels, class_weights=cw)
_, t32 = O.run_forward(net.graph, vals)
v64 = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v) for k, v in vals.items()}
_, t64 = O.run_forward(net.graph, v64)
loss, logits, tape = net.forward_loss(x, labels, cw)
eng = tape.engine
for nd in net.graph.nodes:
    if nd.kind != "relu" or not nd.name.startswith(("s2.b4", "s3")):
        continue
    try:
        g = eng.v(nd.name).tensor().float().cpu().numpy().transpose(0, 3, 1, 2)
    except KeyError:
        continue
    a32, a64 = t32.values[nd.name], t64.values[nd.name]
    fg = int(((g > 0) != (a64 > 0)).sum())
    fr = int(((a32 > 0) != (a64 > 0)).sum())
    print(f"{nd.name:20s} gpu-flips {fg:4d}  ref32-flips {fr:4d}  max|pre|~{np.abs(a64).max():.3g}")
