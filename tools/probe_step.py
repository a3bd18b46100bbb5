"""Quick device-timed probe of the full DeepLabV3+ training step (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200.models import DeepLabConfig  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus  # noqa: E402
from paper_1810_01993_b200.optimizer import OptimConfig  # noqa: E402
from paper_1810_01993_b200.scenes import SceneConfig, device_scene_pool  # noqa: E402
from paper_1810_01993_b200.trainer import DataParallelTrainer  # noqa: E402

h, w = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1152, 768)
steps = 5
net = DeepLabV3Plus(DeepLabConfig(), seed=0)
t0 = time.time()
tr = DataParallelTrainer(net, OptimConfig(lr=0.01), (2, 16, h, w))
print("engine build s", time.time() - t0, flush=True)
x, lab = device_scene_pool(2, SceneConfig(channels=16, height=h, width=w), seed=1)
for i in range(2):
    loss = tr.step(x, lab)
torch.cuda.synchronize()
print("warm loss", float(loss), "launches/step", tr.eng.launches // 3, flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
e0.record()
for i in range(steps):
    loss = tr.step(x, lab)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"step {ms:.2f} ms  host {1e3 * (time.time() - t0) / steps:.2f} ms  img/s {2e3 / ms:.2f}  "
      f"TF/s {2 * 13.3408e12 / (ms / 1e3) / 1e12:.1f} loss {float(loss):.4f}", flush=True)
# per-phase breakdown
eng = tr.eng
for name, fn in [("fwd", eng.forward), ("bwd", eng.backward)]:
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, f"{e0.elapsed_time(e1):.2f} ms", flush=True)
