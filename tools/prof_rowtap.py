"""Narrow-output (growth-32, 5x5) conv launches at the Tiramisu's full resolution, for ncu captures
and CUDA-event timing (development aid): rowtap fprop, rowtap wgrad, and the dgrad over dy."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
N, H, W = 2, 1152, 768
sel = sys.argv[1:] or ["fprop32", "wgrad32", "wgrad64", "wgrad96", "dgrad32"]
ws = nhwc.Workspace()
ops = {}
for cin in (32, 64, 96):
    x = torch.randn(N, H, W, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(N, H, W, 32, device="cuda").to(torch.bfloat16)
    w = torch.randn(25, cin, 32, device="cuda") * 0.02
    wp = torch.empty(32, 25, nhwc.cin_pad(cin), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w, 5, 5, cin, 32, fprop=wp)
    y = torch.empty(N, H, W, 32, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(25 * cin * 32, device="cuda")
    db = torch.empty(32, device="cuda")
    wm = w.to(torch.bfloat16).contiguous()
    wdp = torch.empty(cin, 25, nhwc.cin_pad(32), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w, 5, 5, cin, 32, dgrad=wdp)
    dx = torch.empty(N, H, W, cin, dtype=torch.bfloat16, device="cuda")
    ops[f"fprop{cin}"] = (lambda x=x, wp=wp, y=y: nhwc.conv_fprop(nhwc.View(x), wp, 32, 5, 5, 1, nhwc.View(y),
                                                                   relu=True), 2 * 25 * cin * 32 * N * H * W)
    ops[f"wgrad{cin}"] = (lambda x=x, dy=dy, dw=dw, db=db: nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), 5, 5, 1, dw,
                                                                           ws, bias_grad=db),
                          2 * 25 * cin * 32 * N * H * W)
    ops[f"dgrad{cin}"] = (lambda dy=dy, wdp=wdp, dx=dx, cin=cin: nhwc.conv_dgrad(nhwc.View(dy), wdp, cin, 5, 5, 1,
                                                                                  nhwc.View(dx)),
                          2 * 25 * cin * 32 * N * H * W)
for k in sel:
    ops[k][0]()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in sel:
    e0.record()
    for _ in range(3):
        ops[k][0]()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{k:10s} {ms:.3f} ms  {ops[k][1] / ms / 1e9:.1f} TF/s", flush=True)
