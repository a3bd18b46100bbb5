"""Config 4 probe: time one Tiramisu train step at a given size (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200.loss import ClassWeights  # noqa: E402
from paper_1810_01993_b200.models import tiramisu_config4  # noqa: E402
from paper_1810_01993_b200.net import MiniDenseNet  # noqa: E402

h, w, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
if len(sys.argv) > 4:   # trace every conv launch (debug)
    from paper_1810_01993_b200 import nhwc
    _orig = nhwc.conv_fprop

    def traced(x, w_packed, cout, kh, kw, dilation, y, **kw_):
        print(f"conv x{x.shape} cs{x.buf.shape[3]} -> y{y.shape} cs{y.buf.shape[3]} k{kh} d{dilation} "
              f"mode{kw_.get('w_mode', 0)} res{kw_.get('residual') is not None} mask{kw_.get('mask') is not None} "
              f"acc{kw_.get('accumulate')} f32{kw_.get('y_f32')}", file=sys.stderr, flush=True)
        _orig(x, w_packed, cout, kh, kw, dilation, y, **kw_)
        torch.cuda.synchronize()
    nhwc.conv_fprop = traced
net = MiniDenseNet(tiramisu_config4(), seed=0)
x = np.random.default_rng(0).normal(size=(n, 16, h, w)).astype(np.float32)
lab = np.random.default_rng(1).integers(0, 3, size=(n, h, w)).astype(np.uint8)
cw = ClassWeights((0.982, 0.017, 0.001)).vector()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    loss, logits, tape = net.forward_loss(x, lab, cw)
    g = net.backward(tape)
    torch.cuda.synchronize()
    print(f"step {it}: loss {loss:.4f}  {time.time() - t0:.3f} s", flush=True)
eng = tape.engine
eng.conv_timing = True
eng.forward()
eng.backward()
ms, fl = eng.conv_kernel_totals()
print(f"conv kernels {ms:.2f} ms  {fl / ms / 1e9:.1f} TF/s", flush=True)
