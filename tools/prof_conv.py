"""One launch each of the full-resolution conv kernels (fprop, dgrad, wgrad) and the stem
wgrad, for `ncu --set full` captures (development aid).  Timed with CUDA events too."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
N, H, W, C = 2, 1152, 768, 256
x = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
dy = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
w = torch.randn(9, C, C, device="cuda") * 0.02
wf = torch.empty(C, 9, C, dtype=torch.bfloat16, device="cuda")
wd = torch.empty(C, 9, C, dtype=torch.bfloat16, device="cuda")
nhwc.pack_weights(w, 3, 3, C, C, fprop=wf, dgrad=wd)
b = torch.zeros(C, device="cuda")
dw = torch.empty(9 * C * C, device="cuda")
ws = nhwc.Workspace()
xs = torch.randn(N, H, W, 16, device="cuda").to(torch.bfloat16)
ys = torch.randn(N, H, W, 64, device="cuda").to(torch.bfloat16)
dws = torch.empty(49 * 16 * 64, device="cuda")
x8 = torch.randn(2, 144, 96, 512, device="cuda").to(torch.bfloat16)
r8 = torch.randn(2, 144, 96, 2048, device="cuda").to(torch.bfloat16)
y8 = torch.empty_like(r8)
w8 = torch.randn(1, 512, 2048, device="cuda") * 0.02
wf8 = torch.empty(2048, 1, 512, dtype=torch.bfloat16, device="cuda")
nhwc.pack_weights(w8, 1, 1, 512, 2048, fprop=wf8)
b8 = torch.zeros(2048, device="cuda")
wbf = w.to(torch.bfloat16).contiguous()   # master HWIO bf16
w8bf = w8.to(torch.bfloat16).contiguous()
d8 = torch.randn(2, 144, 96, 512, device="cuda").to(torch.bfloat16)
xwin = torch.zeros(N, H, W + 6, 16, dtype=torch.bfloat16, device="cuda")
xwin[:, :, 3:3 + W] = xs
ws7 = torch.randn(49, 16, 64, device="cuda") * 0.05
wp7 = torch.empty(64, 7, 128, dtype=torch.bfloat16, device="cuda")
nhwc.pack_weights(ws7, 7, 1, 112, 64, fprop=wp7)
b64 = torch.zeros(64, device="cuda")
xa = torch.randn(2, 144, 96, 2048, device="cuda").to(torch.bfloat16)
ya = torch.empty(2, 144, 96, 256, dtype=torch.bfloat16, device="cuda")
wa = (torch.randn(9, 2048, 256, device="cuda") * 0.01).to(torch.bfloat16)
xb = torch.randn(2, 144, 96, 256, device="cuda").to(torch.bfloat16)
wb = (torch.randn(9, 256, 256, device="cuda") * 0.02).to(torch.bfloat16)
xq = torch.randn(2, 288, 192, 256, device="cuda").to(torch.bfloat16)
yq = torch.empty_like(xq)
wm = torch.empty(C, 36, C, dtype=torch.bfloat16, device="cuda")
nhwc.pack_upsampled_dgrad(w, 3, C, C, 4, wm)
wpf = torch.empty(nhwc.upsampled_fprop_taps(3, 4) * C * C, dtype=torch.bfloat16, device="cuda")
nhwc.pack_upsampled_fprop(w, 3, C, C, 4, wpf)
ops = {
    "q_fprop": lambda: nhwc.conv_fprop(nhwc.View(xq), None, 256, 3, 3, 1, nhwc.View(yq), bias=b, relu=True,
                                       w_master=wbf, w_mode=1),
    "aspp_fprop": lambda: nhwc.conv_fprop(nhwc.View(xa), None, 256, 3, 3, 12, nhwc.View(ya), bias=b, relu=True,
                                          w_master=wa, w_mode=1),
    "s2b_fprop": lambda: nhwc.conv_fprop(nhwc.View(xb), None, 256, 3, 3, 2, nhwc.View(ya), bias=b, relu=True,
                                         w_master=wb, w_mode=1),
    "s2b_dgrad": lambda: nhwc.conv_dgrad(nhwc.View(ya), None, 256, 3, 3, 2, nhwc.View(xb), mask=nhwc.View(xb),
                                         w_master=wb),
    "stem_fprop_win": lambda: nhwc.conv_fprop(nhwc.View(xwin), wp7, 64, 7, 1, 1, nhwc.View(ys), bias=b64, relu=True,
                                              window=7),
    "stem_wgrad_win": lambda: nhwc.conv_wgrad(nhwc.View(xwin), nhwc.View(ys), 7, 1, 1, dws, ws, window=7),
    "fprop_mn": lambda: nhwc.conv_fprop(nhwc.View(x), None, C, 3, 3, 1, nhwc.View(y), bias=b, relu=True,
                                        w_master=wbf, w_mode=1),
    "dgrad_m": lambda: nhwc.conv_dgrad(nhwc.View(dy), None, C, 3, 3, 1, nhwc.View(y), mask=nhwc.View(x),
                                       w_master=wbf),
    "fprop": lambda: nhwc.conv_fprop(nhwc.View(x), wf, C, 3, 3, 1, nhwc.View(y), bias=b, relu=True),
    "dgrad": lambda: nhwc.conv_dgrad(nhwc.View(dy), wd, C, 3, 3, 1, nhwc.View(y), mask=nhwc.View(x)),
    "wgrad": lambda: nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), 3, 3, 1, dw, ws),
    "c1x1_fprop": lambda: nhwc.conv_fprop(nhwc.View(x8), wf8, 2048, 1, 1, 1, nhwc.View(y8), bias=b8,
                                          residual=nhwc.View(r8), relu=True),
    "c1x1_dgrad": lambda: nhwc.conv_dgrad(nhwc.View(d8), None, 2048, 1, 1, 1, nhwc.View(y8), mask=nhwc.View(r8),
                                          residual=nhwc.View(r8), w_master=w8bf),
    "up_dgrad": lambda: nhwc.upsampled_dgrad(nhwc.View(dy), wm, C, 3, 4, nhwc.View(yq), mask=nhwc.View(xq)),
    "up_fprop": lambda: nhwc.upsampled_fprop(nhwc.View(xq), wpf, C, C, 3, 4, nhwc.View(y), bias=b, relu=True),
    "stem_wgrad": lambda: nhwc.conv_wgrad(nhwc.View(xs), nhwc.View(ys), 7, 7, 1, dws, ws),
}
sel = sys.argv[1:] or list(ops)
for k in sel:
    ops[k]()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in sel:
    e0.record()
    for _ in range(3):
        ops[k]()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    fl = {"q_fprop": 2 * 9 * 256 * 256 * 2 * 288 * 192, "aspp_fprop": 2 * 9 * 2048 * 256 * 2 * 144 * 96, "s2b_fprop": 2 * 9 * 256 * 256 * 2 * 144 * 96,
          "s2b_dgrad": 2 * 9 * 256 * 256 * 2 * 144 * 96, "stem_wgrad": 2 * 49 * 16 * 64 * N * H * W, "stem_wgrad_win": 2 * 49 * 16 * 64 * N * H * W,
          "stem_fprop_win": 2 * 49 * 16 * 64 * N * H * W, "c1x1_fprop": 2 * 512 * 2048 * 2 * 144 * 96,
                                                  "c1x1_dgrad": 2 * 512 * 2048 * 2 * 144 * 96,
          "up_dgrad": 2 * 36 * C * C * 2 * 288 * 192, "up_fprop": 2 * 36 * C * C * 2 * 288 * 192}.get(
        k, 2 * 9 * C * C * N * H * W)
    print(f"{k:10s} {ms:.3f} ms  {fl / ms / 1e9:.1f} TF/s", flush=True)
