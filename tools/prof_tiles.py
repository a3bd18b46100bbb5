"""N-tile width sweep of the generic fprop (block_n 256 / 128 / 64) on representative shapes, CUDA-event
timed, to re-calibrate fprop_choose's relative tile speeds (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
V = nhwc.View
shapes = {  # name: (n, h, w, cin, cout, k, dil)
    "3x3_256_h288": (2, 288, 192, 256, 256, 3, 1),
    "3x3_512_h144": (2, 144, 96, 512, 512, 3, 4),
    "1x1_512to2048_h144": (2, 144, 96, 512, 2048, 1, 1),
    "1x1_2048to512_h144": (2, 144, 96, 2048, 512, 1, 1),
    "3x3_128_h144": (2, 144, 96, 128, 128, 3, 1),
    "1x1_96to320_h1152": (2, 1152, 768, 96, 320, 1, 1),
    "3x3_304to256_h288": (2, 288, 192, 304, 256, 3, 1),
}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, (n, h, w, cin, cout, k, d) in shapes.items():
    cp = (cin + 7) // 8 * 8
    x = torch.randn(n, h, w, cp, device="cuda").to(torch.bfloat16)
    y = torch.empty(n, h, w, (cout + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    wm = (torch.randn(k * k, cin, cout, device="cuda") * 0.02).to(torch.bfloat16)
    b = torch.zeros(cout, device="cuda")
    fl = 2 * k * k * cin * cout * n * h * w
    row = []
    for bn in (0, 256, 128, 64):
        f = lambda: nhwc.conv_fprop(V(x, 0, cin), None, cout, k, k, d, V(y, 0, cout), bias=b, relu=True,
                                    w_master=wm, w_mode=1, block_n=bn)
        f()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        row.append(f"bn{bn or 'auto'} {ms * 1e3:7.1f}us {fl / ms / 1e9:6.0f}TF/s")
    print(f"{name:22s} " + " | ".join(row), flush=True)
