"""Batch-norm apply / VJP / statistics streams at the BN variant's shapes, CUDA-event timed with
achieved HBM bandwidth (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

torch.manual_seed(0)
V = nhwc.View
ws = nhwc.Workspace()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(f, n=5):
    f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (n, h, w, c) in [(2, 1152, 768, 256), (2, 288, 192, 256), (2, 144, 96, 2048), (2, 1152, 768, 64)]:
    x = torch.randn(n, h, w, c, device="cuda").to(torch.bfloat16)
    g = torch.randn(n, h, w, c, device="cuda").to(torch.bfloat16)
    r = torch.randn(n, h, w, c, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    gamma = torch.ones(c, device="cuda")
    beta = torch.zeros(c, device="cuda")
    stats = torch.empty(4 * c, device="cuda")
    dg = torch.empty(c, device="cuda")
    db = torch.empty(c, device="cuda")
    nb = n * h * w * c * 2
    ms = timeit(lambda: nhwc.bn_forward(V(x), gamma, beta, 1e-5, V(y), stats, ws, relu=True))
    print(f"{n}x{h}x{w}x{c} bn_forward(stats+apply) {ms * 1e3:7.1f} us  {3 * nb / ms / 1e6:6.0f} GB/s (3 passes)")
    ms = timeit(lambda: nhwc.bn_forward(V(x), gamma, beta, 1e-5, V(y), stats, ws, residual=V(r), relu=True))
    print(f"{n}x{h}x{w}x{c} bn_forward+res          {ms * 1e3:7.1f} us  {4 * nb / ms / 1e6:6.0f} GB/s (4 passes)")
    ms = timeit(lambda: nhwc.bn_backward(V(x), V(g), gamma, stats, dg, db, V(dx), ws))
    print(f"{n}x{h}x{w}x{c} bn_backward             {ms * 1e3:7.1f} us  {5 * nb / ms / 1e6:6.0f} GB/s (5 passes)")

# bilinear x4 (decoder -> full resolution, 256 channels) and x2 (ASPP -> decoder)
for (n, h, w, c, f) in [(2, 288, 192, 256, 4), (2, 144, 96, 256, 2)]:
    x = torch.randn(n, h, w, c, device="cuda").to(torch.bfloat16)
    y = torch.empty(n, h * f, w * f, c, dtype=torch.bfloat16, device="cuda")
    m = torch.randn(n, h, w, c, device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(x)
    ms = timeit(lambda: nhwc.bilinear_fwd(V(x), V(y), f))
    nb = (x.numel() + y.numel()) * 2
    print(f"bilinear_fwd x{f} {n}x{h}x{w}x{c}  {ms * 1e3:7.1f} us  {nb / ms / 1e6:6.0f} GB/s")
    ms = timeit(lambda: nhwc.bilinear_bwd(V(y), V(dx), f, mask=V(m), ws=ws))
    print(f"bilinear_bwd x{f} {n}x{h}x{w}x{c}  {ms * 1e3:7.1f} us  {(nb + m.numel() * 2) / ms / 1e6:6.0f} GB/s (dy+dx+mask)")
