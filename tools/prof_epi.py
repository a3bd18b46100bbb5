"""Epilogue-operand sweep on the 1/8-resolution 1x1 dgrad shape (2x144x96, 512 -> 2048 channels):
the same launch with 0, 1 and 2 TMA epilogue operands, CUDA-event timed (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
d8 = torch.randn(2, 144, 96, 512, device="cuda").to(torch.bfloat16)
r8 = torch.randn(2, 144, 96, 2048, device="cuda").to(torch.bfloat16)
m8 = torch.randn(2, 144, 96, 2048, device="cuda").to(torch.bfloat16)
y8 = torch.empty_like(r8)
w8bf = (torch.randn(1, 512, 2048, device="cuda") * 0.02).to(torch.bfloat16)
x8 = torch.randn(2, 144, 96, 2048, device="cuda").to(torch.bfloat16)
yq = torch.empty(2, 144, 96, 512, dtype=torch.bfloat16, device="cuda")
w8f = (torch.randn(1, 2048, 512, device="cuda") * 0.02).to(torch.bfloat16)
b512 = torch.zeros(512, device="cuda")
V = nhwc.View
ops = {
    "dgrad_0op": lambda: nhwc.conv_dgrad(V(d8), None, 2048, 1, 1, 1, V(y8), w_master=w8bf),
    "dgrad_mask": lambda: nhwc.conv_dgrad(V(d8), None, 2048, 1, 1, 1, V(y8), mask=V(m8), w_master=w8bf),
    "dgrad_mask_res": lambda: nhwc.conv_dgrad(V(d8), None, 2048, 1, 1, 1, V(y8), mask=V(m8), residual=V(r8),
                                              w_master=w8bf),
    "fprop_2048_512": lambda: nhwc.conv_fprop(V(x8), None, 512, 1, 1, 1, V(yq), bias=b512, relu=True,
                                              w_master=w8f, w_mode=1),
}
sel = sys.argv[1:] or list(ops)
for k in sel:
    ops[k]()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in sel:
    for _ in range(2):
        ops[k]()
    e0.record()
    for _ in range(10):
        ops[k]()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{k:16s} {ms * 1e3:7.1f} us", flush=True)
