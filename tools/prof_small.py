"""Achieved HBM bandwidth of the memory-bound kernels of the step, at the step's own shapes
(2 x 1152 x 768 full resolution, 256 channels; the 41.5 M-parameter LARC update), timed with
CUDA events over back-to-back launches.  Bytes are algorithmic (each tensor read / written once).
Usage: python tools/prof_small.py [kernel ...] [--out file]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_01993_b200 import nhwc  # noqa: E402

N, H, W = 2, 1152, 768
PEAK = 6535.1
x = torch.randn(N, H, W, 256, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
g2 = torch.randn_like(x)
dyb = torch.randn(N, H, W, 8, device="cuda").to(torch.bfloat16)
wt = torch.randn(256, 3, device="cuda")
parts = nhwc.head_backward_parts()
dwp = torch.empty(parts * 256 * 3, device="cuda")
dbp = torch.empty(parts * 3, device="cuda")
lo = torch.randn(N, H // 4, W // 4, 256, device="cuda").to(torch.bfloat16)
lo2 = torch.empty_like(lo)
stem = torch.randn(N, H, W, 64, device="cuda").to(torch.bfloat16)
stem_p = torch.empty(N, H // 4, W // 4, 64, dtype=torch.bfloat16, device="cuda")
logits = torch.randn(N, H, W, 3, device="cuda")
labels = torch.randint(0, 3, (N * H * W,), dtype=torch.uint8, device="cuda")
cw = torch.tensor([1.0, 7.7, 31.6], device="cuda")
loss = torch.zeros(1, device="cuda")
counts = torch.zeros(N * 3, dtype=torch.int32, device="cuda")
dlog = torch.empty(N, H, W, 8, dtype=torch.bfloat16, device="cuda")
pred = torch.empty(N * H * W, dtype=torch.uint8, device="cuda")
P = 41_539_827
pw = torch.randn(P, device="cuda") * 0.01
pm = torch.zeros(P, device="cuda")
pg = torch.randn(P, device="cuda") * 1e-3
pwb = torch.empty(P, dtype=torch.bfloat16, device="cuda")
offs = torch.tensor(np.linspace(0, P, 131).astype(np.int64) // 64 * 64, device="cuda")
offs[-1] = P
lr_out = torch.zeros(130, device="cuda")
status = torch.zeros(1, dtype=torch.int32, device="cuda")
xin = torch.randn(N, 16, H, W, device="cuda")
xwin = torch.zeros(N, H, W + 6, 16, dtype=torch.bfloat16, device="cuda")
stats = torch.empty(4 * 256, device="cuda")
gam = torch.ones(256, device="cuda")
bet = torch.zeros(256, device="cuda")
dg = torch.empty(256, device="cuda")
db = torch.empty(256, device="cuda")
ws = nhwc.Workspace()
gsum = torch.empty(N * (H // 4) * (W // 4) * 9 * 256, dtype=torch.bfloat16, device="cuda")
E = x.numel() * 2   # bytes of one full-resolution 256-channel bf16 tensor
ops = {
    "head_backward": (lambda: nhwc.head_backward(nhwc.View(dyb, 0, 3), wt, nhwc.View(x), nhwc.View(dx), dwp, dbp,
                                                 mask_dx=True), 2 * E),
    "upsample4_fwd": (lambda: nhwc.upsample_fwd(nhwc.View(lo), nhwc.View(dx), 4), E + E // 16),
    "upsample4_bwd": (lambda: nhwc.upsample_bwd(nhwc.View(x), nhwc.View(lo2), 4, mask=nhwc.View(lo)), E + E // 8),
    "avgpool4_fwd": (lambda: nhwc.avgpool_fwd(nhwc.View(stem), nhwc.View(stem_p), 4), stem.numel() * 2 * 17 // 16),
    "avgpool4_bwd": (lambda: nhwc.avgpool_bwd(nhwc.View(stem_p), nhwc.View(stem), 4, mask=nhwc.View(stem)),
                     stem.numel() * 2 * 2 + stem_p.numel() * 2),
    "relu_mask": (lambda: nhwc.relu_mask(nhwc.View(g2), nhwc.View(x)), 3 * E),
    "wce": (lambda: nhwc.wce(nhwc.View(logits), labels, cw, loss, counts, nhwc.View(dlog, 0, 3), pred, ws),
            N * H * W * (12 + 1 + 16 + 1)),
    "larc_update": (lambda: nhwc.larc_update(pw, pm, pg, offs, 0.01, 0.9, 0.02, 0.0, 1e-8, 1.0, lr_out, status, ws,
                                             w_bf16=pwb), P * (8 + 12 + 8 + 2)),
    "nchw_to_nhwc_halo": (lambda: nhwc.nchw_to_nhwc_halo(xin, xwin, 3), xin.numel() * 4 + xwin.numel() * 2),
    "bn_forward": (lambda: nhwc.bn_forward(nhwc.View(x), gam, bet, 1e-5, nhwc.View(dx), stats, ws, relu=True), 3 * E),
    "bn_backward": (lambda: nhwc.bn_backward(nhwc.View(x), nhwc.View(g2), gam, stats, dg, db, nhwc.View(dx), ws),
                    5 * E),
    "bilinear4_fwd": (lambda: nhwc.bilinear_fwd(nhwc.View(lo), nhwc.View(dx), 4), E + E // 16),
    "upsampled_wgrad_sums": (lambda: nhwc.upsampled_wgrad_sums(nhwc.View(x), 3, 4, gsum), E + E * 9 // 16),
    "bilinear4_bwd": (lambda: nhwc.bilinear_bwd(nhwc.View(x), nhwc.View(lo2), 4), E + E // 16),
}
args = [a for a in sys.argv[1:] if not a.startswith("--")]
out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
if out in args:
    args.remove(out)
sel = args or list(ops)
for k in sel:
    ops[k][0]()
torch.cuda.synchronize()
lines = [f"{'kernel':20s} {'ms':>8s} {'GB/s':>8s} {'% of ' + str(PEAK):>12s}   algorithmic bytes"]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in sel:
    fn, byts = ops[k]
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gbs = byts / ms / 1e6
    lines.append(f"{k:20s} {ms:8.3f} {gbs:8.0f} {100 * gbs / PEAK:11.1f}%   {byts / 1e6:.0f} MB")
print("\n".join(lines), flush=True)
if out:
    open(out, "w").write("\n".join(lines) + "\n")
