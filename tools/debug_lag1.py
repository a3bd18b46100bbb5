import os, sys, torch
sys.path.insert(0, ".")
import torch.distributed as dist
world = int(os.environ.get("WORLD_SIZE", "1")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
from paper_1810_01993_b200.loss import ClassWeights
from paper_1810_01993_b200.models import DeepLabConfig
from paper_1810_01993_b200.net import DeepLabV3Plus
from paper_1810_01993_b200.optimizer import OptimConfig
from paper_1810_01993_b200.scenes import SceneConfig, device_scene_pool
from paper_1810_01993_b200.trainer import DataParallelTrainer
H, W = int(os.environ.get("H", "1152")), int(os.environ.get("W", "768"))
net = DeepLabV3Plus(DeepLabConfig(), seed=0)
sc = SceneConfig(channels=16, height=H, width=W)
tr = DataParallelTrainer(net, OptimConfig(lr=0.01, momentum=0.9, trust=0.02), (2, 16, H, W),
                         class_weights=ClassWeights(sc.frequencies).vector(), lag=1)
fx, fl = device_scene_pool(8, sc, seed=1000)
b = [(fx[2*i:2*i+2].contiguous(), fl[2*i:2*i+2].contiguous()) for i in range(4)]
def st(tag):
    torch.cuda.synchronize()
    print(tag, int(tr.status.item()), float(tr.eng.loss.item()), flush=True)
for i in range(3):
    tr.step(*b[i % 4]); st(f"eager{i}")
tr.capture(*b[0], timed=True, buffers=2)
for i in range(4):
    tr.step(*b[i % 4]); st(f"replay{i}")
host = [(x.cpu().pin_memory(), l.cpu().pin_memory()) for x, l in b]
tr.stage(*host[0])
for i in range(3):
    tr.step_staged(); st(f"staged{i}")
    if i < 2:
        tr.stage(*host[(i + 1) % 4])
tr.eng.serialize(True)
tr._eager_step(*b[0]); st("serial")
