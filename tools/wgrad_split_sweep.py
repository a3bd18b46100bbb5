import sys, torch
sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc
for (n, h, w, ci, co, k, d) in [(2, 288, 192, 64, 64, 3, 1), (2, 288, 192, 304, 256, 3, 1), (2, 144, 96, 512, 512, 3, 4)]:
    x = torch.randn(n, h, w, ci, device="cuda").to(torch.bfloat16)
    dy = torch.randn(n, h, w, co, device="cuda").to(torch.bfloat16)
    dw = torch.empty(k * k * ci * co, device="cuda")
    ws = nhwc.Workspace()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fl = 2 * k * k * ci * co * n * h * w
    for s in (0, 4, 8, 16, 32, 48, 74, 148, 296):
        nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), k, k, d, dw, ws, splits=s)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), k, k, d, dw, ws, splits=s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{ci}->{co} h{h} splits {s:4d}: {ms*1e3:7.1f} us  {fl/ms/1e9:7.1f} TF/s", flush=True)
