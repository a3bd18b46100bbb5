"""Config 5: atrous conv microbenchmark sweep.

3x3, stride 1, "same"; dilation in {1, 2, 4, 12, 18, 24} x (Cin, Cout) in {(256, 256) at the
full-resolution and /4 maps, (512, 512), (1024, 256), (2048, 256) at the /8 map}; N = 2; inputs
U(-1, 1) from a fixed seed.  fprop, dgrad and wgrad are timed separately with CUDA events (after
warm-up, median of repeats), each 2*9*Cin*Cout*N*H*W FLOPs, against the measured bf16 peak.
Numerical parity of the same kernels on these shapes against the reference's conv arithmetic is
tests/test_gpu_conv.py::test_atrous_sweep_shapes_vs_oracle (cropped maps).

Usage: python tools/atrous_sweep.py [--out profiles/round1/atrous_sweep.json] [--reps 10]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01993_b200 import nhwc  # noqa: E402

DILATIONS = (1, 2, 4, 12, 18, 24)
SHAPES = [(256, 256, 1152, 768), (256, 256, 288, 192), (512, 512, 144, 96), (1024, 256, 144, 96),
          (2048, 256, 144, 96)]


def peak():
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
        for k in ("bf16_tflops", "bf16_dense_tflops", "bf16"):
            if k in d:
                return float(d[k])
    except (OSError, ValueError):
        pass
    return 1684.4


def time_op(fn, reps):
    """Median over 3 groups of `reps` back-to-back launches (per-launch ms)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    pk = peak()
    g = torch.Generator(device="cuda").manual_seed(5)
    ws = nhwc.Workspace()
    rows = []
    for cin, cout, h, w in SHAPES:
        n = 2
        x = (torch.rand(n, h, w, cin, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        dy = (torch.rand(n, h, w, cout, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        wm = ((torch.rand(9, cin, cout, device="cuda", generator=g) * 2 - 1) / (9 * cin) ** 0.5).to(torch.bfloat16)
        bias = torch.zeros(cout, device="cuda")
        y = torch.empty(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
        dx = torch.empty(n, h, w, cin, dtype=torch.bfloat16, device="cuda")
        dw = torch.empty(9 * cin * cout, device="cuda")
        fl = 2 * 9 * cin * cout * n * h * w
        for d in DILATIONS:
            ops = {
                "fprop": lambda: nhwc.conv_fprop(nhwc.View(x), None, cout, 3, 3, d, nhwc.View(y), bias=bias,
                                                 relu=True, w_master=wm, w_mode=1),
                "dgrad": lambda: nhwc.conv_dgrad(nhwc.View(dy), None, cin, 3, 3, d, nhwc.View(dx), w_master=wm),
                "wgrad": lambda: nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), 3, 3, d, dw, ws),
            }
            for pas, fn in ops.items():
                ms = time_op(fn, args.reps)
                tf = fl / (ms * 1e-3) / 1e12
                r = {"pass": pas, "cin": cin, "cout": cout, "dilation": d, "n": n, "h": h, "w": w, "ms": round(ms, 4),
                     "tflops": round(tf, 1), "frac_of_peak": round(tf / pk, 3), "peak_tflops": pk}
                rows.append(r)
                print(f"{pas:5s} {cin:4d}->{cout:4d} d{d:2d} {h:4d}x{w:<4d} {ms:8.3f} ms {tf:7.1f} TF/s "
                      f"{100 * tf / pk:5.1f}% of {pk:.0f}", flush=True)
        del x, dy, y, dx, dw
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
