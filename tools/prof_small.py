"""Time the memory-bound kernels of the step at full size (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

N, H, W = 2, 1152, 768
x = torch.randn(N, H, W, 256, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
dyb = torch.randn(N, H, W, 8, device="cuda").to(torch.bfloat16)
wt = torch.randn(256, 3, device="cuda")
parts = nhwc.head_backward_parts()
dwp = torch.empty(parts * 256 * 3, device="cuda")
dbp = torch.empty(parts * 3, device="cuda")
lo = torch.randn(N, H // 4, W // 4, 256, device="cuda").to(torch.bfloat16)
ops = {
    "head_backward": lambda: nhwc.head_backward(nhwc.View(dyb, 0, 3), wt, nhwc.View(x), nhwc.View(dx), dwp, dbp,
                                                mask_dx=True),
    "dgrad_small": lambda: nhwc.dgrad_1x1_small(nhwc.View(dyb, 0, 3), wt, nhwc.View(dx), mask=nhwc.View(x)),
    "upsample4_fwd": lambda: nhwc.upsample_fwd(nhwc.View(lo), nhwc.View(dx), 4),
    "upsample4_bwd": lambda: nhwc.upsample_bwd(nhwc.View(x), nhwc.View(lo), 4),
    "relu_mask": lambda: nhwc.relu_mask(nhwc.View(dx), nhwc.View(x)),
}
byts = {"head_backward": 2 * x.numel() * 2, "dgrad_small": 2 * x.numel() * 2, "upsample4_fwd": x.numel() * 2,
        "upsample4_bwd": x.numel() * 2, "relu_mask": 3 * x.numel() * 2}
sel = sys.argv[1:] or list(ops)
for k in sel:
    ops[k]()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in sel:
    e0.record()
    for _ in range(5):
        ops[k]()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{k:14s} {ms:.3f} ms  {byts[k] / ms / 1e6:.0f} GB/s", flush=True)
