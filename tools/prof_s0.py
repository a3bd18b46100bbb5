"""DeepLab stage-0 3x3 64->64 convs at 2 x 288 x 192 (generic vs row-tap kernels; development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
N, H, W, C = 2, 288, 192, 64
x = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
dy = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
w = torch.randn(9, C, C, device="cuda") * 0.05
wm = w.to(torch.bfloat16).contiguous()
wp = torch.empty(C, 9, 64, dtype=torch.bfloat16, device="cuda")
wd = torch.empty(C, 9, 64, dtype=torch.bfloat16, device="cuda")
nhwc.pack_weights(w, 3, 3, C, C, fprop=wp, dgrad=wd)
y = torch.empty_like(x)
dw = torch.empty(9 * C * C, device="cuda")
ws = nhwc.Workspace()
ops = {
    "fprop_master": lambda: nhwc.conv_fprop(nhwc.View(x), None, C, 3, 3, 1, nhwc.View(y), w_master=wm, w_mode=1),
    "fprop_packed": lambda: nhwc.conv_fprop(nhwc.View(x), wp, C, 3, 3, 1, nhwc.View(y)),
    "dgrad_master": lambda: nhwc.conv_dgrad(nhwc.View(dy), None, C, 3, 3, 1, nhwc.View(y), w_master=wm),
    "dgrad_packed": lambda: nhwc.conv_dgrad(nhwc.View(dy), wd, C, 3, 3, 1, nhwc.View(y)),
    "wgrad": lambda: nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), 3, 3, 1, dw, ws),
}
fl = 2 * 9 * C * C * N * H * W
for k, f in ops.items():
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k, f in ops.items():
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{k:14s} {ms * 1e3:7.1f} us  {fl / ms / 1e9:7.1f} TF/s", flush=True)
