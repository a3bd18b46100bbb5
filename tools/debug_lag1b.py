import os, sys, torch
sys.path.insert(0, ".")
from paper_1810_01993_b200.loss import ClassWeights
from paper_1810_01993_b200.models import DeepLabConfig
from paper_1810_01993_b200.net import DeepLabV3Plus
from paper_1810_01993_b200.optimizer import OptimConfig
from paper_1810_01993_b200.scenes import SceneConfig, device_scene_pool
from paper_1810_01993_b200.trainer import DataParallelTrainer
H, W = 1152, 768
sc = SceneConfig(channels=16, height=H, width=W)
fx, fl = device_scene_pool(8, sc, seed=1000)
b = [(fx[2*i:2*i+2].contiguous(), fl[2*i:2*i+2].contiguous()) for i in range(4)]
for lag in (0, 1):
    net = DeepLabV3Plus(DeepLabConfig(), seed=0)
    tr = DataParallelTrainer(net, OptimConfig(lr=0.01, momentum=0.9, trust=0.02), (2, 16, H, W),
                             class_weights=ClassWeights(sc.frequencies).vector(), lag=lag)
    ls = []
    for i in range(6):
        ls.append(round(float(tr.step(*b[i % 4]).item()), 4))
    print("lag", lag, ls, "lr", tr.lr_out[:6].tolist(), flush=True)
