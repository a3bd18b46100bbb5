"""Torch-tensor front end of the NHWC fast path (device memory via torch, compute via libb2dl).

torch is plumbing here: it allocates device buffers and supplies the current
CUDA stream.  Every arithmetic operation below is a launch of a kernel in
libb2dl.so through its C ABI (include/b2dl.h).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from ._lib import LIB, NULL_ACT, Act, ConvArgs, LarcArgs, Segment, WgradArgs, check


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class View:
    """Channel slice [c_off, c_off + c) of an NHWC buffer `buf` [N, H, W, C_total]."""
    buf: torch.Tensor
    c_off: int = 0
    c: int = -1

    def __post_init__(self):
        if self.buf.dim() != 4:
            raise ValueError("NHWC buffer must be 4-D")
        if self.c < 0:
            self.c = self.buf.shape[3] - self.c_off
        if self.c_off + self.c > self.buf.shape[3]:
            raise ValueError("view exceeds buffer channels")

    @property
    def shape(self):
        n, h, w, _ = self.buf.shape
        return (n, h, w, self.c)

    def act(self) -> Act:
        n, h, w, cs = self.buf.shape
        ptr = self.buf.data_ptr() + self.c_off * self.buf.element_size()
        return Act(ptr, n, h, w, self.c, cs)

    def tensor(self) -> torch.Tensor:
        return self.buf[..., self.c_off:self.c_off + self.c]


def _act(v):
    return NULL_ACT if v is None else v.act()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def cin_pad(cin: int) -> int:
    return LIB.b2dl_cin_pad(cin)


def same_pads(k: int, d: int):
    """TF 'same' split (_kernels_py.py:18-21): before = total // 2."""
    total = (k - 1) * d
    return total // 2, total - total // 2


def conv_fprop(x: View, w_packed: torch.Tensor | None, cout: int, kh: int, kw: int, dilation: int,
               y: View, bias=None, residual: View | None = None, relu=False, accumulate=False,
               mask: View | None = None, y_f32=False, pads=None, block_n=0, w_master=None, w_mode=0, window=0,
               in_stride=0, out_stride=0, out_phase=(0, 0), bn_partial=None, bn_rows_only=False,
               bnb_stats=None, bnb_partial=None):
    """w_mode 0: w_packed bf16 [cout][taps][cin_pad]; 1: w_master bf16 HWIO of this conv;
    2: w_master bf16 HWIO of the forward conv whose input gradient this is (see b2dl.h).
    window > 0: row-window mode over a haloed x (pass kw=1; see b2dl_conv_args.window).
    bn_partial: fp32 [rows][2][cout] batch-norm statistics of the output (epilogue-computed).
    bn_rows_only: return the number of bn_partial rows the launch writes instead of launching."""
    pt, pl = pads if pads is not None else (same_pads(kh, dilation)[0], same_pads(kw, dilation)[0])
    a = ConvArgs(x.act(), _ptr(w_packed), cout, kh, kw, dilation, pt, pl,
                 y.act(), int(y_f32), _ptr(bias), _act(residual), int(relu), int(accumulate),
                 _act(mask), block_n, _ptr(w_master), w_mode, window, in_stride, out_stride, *out_phase,
                 _ptr(bn_partial), _ptr(bnb_stats), _ptr(bnb_partial))
    if bn_rows_only:
        n = LIB.b2dl_conv_fprop_bn_rows(ctypes.byref(a))
        if n < 0:
            check(-n, "conv_fprop_bn_rows")
        return n
    check(LIB.b2dl_conv_fprop(ctypes.byref(a), _stream()), "conv_fprop")


def conv_dgrad(dy: View, w_dgrad: torch.Tensor | None, cin: int, kh: int, kw: int, dilation: int,
               dx: View, accumulate=False, mask: View | None = None, dx_f32=False, w_master=None,
               residual: View | None = None, block_n=0, bnb_stats=None, bnb_partial=None, bn_rows_only=False):
    """Input gradient as a forward conv over dy with tap-flipped weights and 'after' pads;
    weights from the dgrad-packed copy, or straight from the forward conv's bf16 HWIO master.
    bnb_stats / bnb_partial: dx is d loss / d y of a batch norm's output; mask = the BN input
    (see b2dl_conv_args.bnb_partial)."""
    pads = (same_pads(kh, dilation)[1], same_pads(kw, dilation)[1])
    return conv_fprop(dy, w_dgrad, cin, kh, kw, dilation, dx, accumulate=accumulate, mask=mask, residual=residual,
                      y_f32=dx_f32, pads=pads, block_n=block_n, w_master=w_master,
                      w_mode=2 if w_master is not None else 0, bnb_stats=bnb_stats, bnb_partial=bnb_partial,
                      bn_rows_only=bn_rows_only)


class Workspace:
    """Grow-only device scratch buffer shared by the launches of one stream."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.device)
        return self.buf


def conv_wgrad(x: View, dy: View, kh: int, kw: int, dilation: int, dw: torch.Tensor,
               ws: Workspace, bias_grad=None, accumulate=False, splits=0, window=0):
    """dw fp32 HWIO [kh*kw][cin][cout] (+)= x^T dy per tap; bias_grad[cout] (+)= sum dy."""
    pt, pl = same_pads(kh, dilation)[0], same_pads(kw, dilation)[0]
    a = WgradArgs(x.act(), dy.act(), kh, kw, dilation, pt, pl, ctypes.c_void_p(dw.data_ptr()),
                  _ptr(bias_grad), int(accumulate), None, 0, splits, 0, window)
    need = LIB.b2dl_wgrad_workspace_size(ctypes.byref(a))
    buf = ws.get(need)
    a.workspace = ctypes.c_void_p(buf.data_ptr())
    a.workspace_bytes = buf.numel()
    check(LIB.b2dl_conv_wgrad(ctypes.byref(a), _stream()), "conv_wgrad")


def _wgrad_args(x: View, dy: View, kh: int, kw: int, dilation: int, defer: bool, window=0):
    pt, pl = same_pads(kh, dilation)[0], same_pads(kw, dilation)[0]
    return WgradArgs(x.act(), dy.act(), kh, kw, dilation, pt, pl, None, None, 0, None, 0, 0, int(defer), window)


def wgrad_partials(x: View, dy: View, kh: int, kw: int, dilation: int, window=0):
    """(workspace bytes, weight parts, bias parts, bias byte offset) of a deferred wgrad."""
    a = _wgrad_args(x, dy, kh, kw, dilation, True, window)
    a.bias_grad = ctypes.c_void_p(1)  # bias partials requested (layout query only)
    nbytes = LIB.b2dl_wgrad_workspace_size(ctypes.byref(a))
    wp, bp, bo = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    check(LIB.b2dl_wgrad_partials(ctypes.byref(a), ctypes.byref(wp), ctypes.byref(bp), ctypes.byref(bo)),
          "wgrad_partials")
    return nbytes, wp.value, bp.value, bo.value


def conv_wgrad_deferred(x: View, dy: View, kh: int, kw: int, dilation: int, partials: torch.Tensor, window=0):
    """wgrad + bias column sums left as split-K partials in `partials` (see wgrad_partials)."""
    a = _wgrad_args(x, dy, kh, kw, dilation, True, window)
    a.dw = ctypes.c_void_p(partials.data_ptr())        # unused in deferred mode, must be non-null
    a.bias_grad = ctypes.c_void_p(partials.data_ptr())
    a.workspace = ctypes.c_void_p(partials.data_ptr())
    a.workspace_bytes = partials.numel()
    check(LIB.b2dl_conv_wgrad(ctypes.byref(a), _stream()), "conv_wgrad")


def segment_table(segs, device) -> torch.Tensor:
    """Pack (src_ptr, dst_off, n, parts, accumulate) records into a device array."""
    arr = (Segment * len(segs))(*[Segment(src, off, n, parts, acc) for src, off, n, parts, acc in segs])
    host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    return host.to(device)


def reduce_segments(table: torch.Tensor, nseg: int, max_n: int, dst_base: torch.Tensor):
    check(LIB.b2dl_reduce_segments(ctypes.c_void_p(table.data_ptr()), nseg, max_n,
                                   ctypes.c_void_p(dst_base.data_ptr()), _stream()), "reduce_segments")


def pack_weights(w_hwio: torch.Tensor, kh: int, kw: int, cin: int, cout: int, fprop=None, dgrad=None):
    check(LIB.b2dl_pack_weights(ctypes.c_void_p(w_hwio.data_ptr()), kh, kw, cin, cout,
                                _ptr(fprop), _ptr(dgrad), _stream()), "pack_weights")


def nchw_to_nhwc(x: torch.Tensor, y: View, dst_f32=False):
    check(LIB.b2dl_nchw_to_nhwc(ctypes.c_void_p(x.data_ptr()), y.act(), int(dst_f32), _stream()),
          "nchw_to_nhwc")


def head_backward_parts() -> int:
    return LIB.b2dl_head_backward_parts()


def head_backward(dy: View, w_hwio: torch.Tensor, x: View, dx: View | None, dw_partials: torch.Tensor,
                  db_partials: torch.Tensor, accumulate=False, mask_dx=False):
    """Few-output-channel 1x1 conv backward in one pass: dW / db block partials (+ optional dx)."""
    check(LIB.b2dl_head_backward(dy.act(), ctypes.c_void_p(w_hwio.data_ptr()), x.act(), _act(dx), int(accumulate),
                                 int(mask_dx), ctypes.c_void_p(dw_partials.data_ptr()),
                                 ctypes.c_void_p(db_partials.data_ptr()), _stream()), "head_backward")


def pack_upsampled_dgrad(w_hwio: torch.Tensor, k: int, cin: int, cout: int, f: int, out: torch.Tensor):
    """Merged weights of the (dgrad + nearest-upsample VJP) of a k x k conv over an x f upsampling."""
    check(LIB.b2dl_pack_upsampled_dgrad(ctypes.c_void_p(w_hwio.data_ptr()), k, cin, cout, f,
                                        ctypes.c_void_p(out.data_ptr()), _stream()), "pack_upsampled_dgrad")


def upsampled_dgrad(dy: View, w_merged: torch.Tensor, cin: int, k: int, f: int, dx: View, accumulate=False,
                    mask: View | None = None):
    """dx (low resolution) (+)= block-summed input gradient of a k x k 'same' conv whose input was a
    nearest x f upsampling of dx's tensor: one (k+f-1)^2-tap conv over dy with input stride f."""
    kk, pad = k + f - 1, k - 1 - (k - 1) // 2
    conv_fprop(dy, w_merged, cin, kk, kk, 1, dx, accumulate=accumulate, mask=mask, pads=(pad, pad), in_stride=f)


def upsampled_fprop_phases(k: int, f: int):
    """Per output phase (a, b) of a 'same' k x k conv over a nearest x f upsampling:
    (a, b, ka, kb, pad_top, pad_left, first tap) -- the layout b2dl_pack_upsampled_fprop writes."""
    P = (k - 1) // 2
    rng = [((a - P) // f, (a + k - 1 - P) // f) for a in range(f)]
    S = sum(hi - lo + 1 for lo, hi in rng)
    out, rows = [], 0
    for a, (la, ha) in enumerate(rng):
        ka, cols = ha - la + 1, 0
        for b, (lb, hb) in enumerate(rng):
            kb = hb - lb + 1
            out.append((a, b, ka, kb, -la, -lb, rows * S + ka * cols))
            cols += kb
        rows += ka
    return out


def pack_upsampled_fprop(w_hwio: torch.Tensor, k: int, cin: int, cout: int, f: int, out: torch.Tensor):
    """Merged phase weights (bf16 HWIO blocks, upsampled_fprop_phases order) of a k x k conv over
    a nearest x f upsampling; out holds b2dl_upsampled_fprop_taps(k, f) * cin * cout values."""
    check(LIB.b2dl_pack_upsampled_fprop(ctypes.c_void_p(w_hwio.data_ptr()), k, cin, cout, f,
                                        ctypes.c_void_p(out.data_ptr()), _stream()), "pack_upsampled_fprop")


def upsampled_fprop_taps(k: int, f: int) -> int:
    return LIB.b2dl_upsampled_fprop_taps(k, f)


def upsampled_fprop(x: View, w_phases: torch.Tensor, cin: int, cout: int, k: int, f: int, y: View, bias=None,
                    relu=False):
    """y (full resolution) = conv_k(nearest_up_f(x)) + bias (relu), from the low-resolution x: one
    launch per output phase, each a <= ceil-sized conv over x with merged weights writing a
    stride-f phase view of y (no upsampled tensor; ~(1 + (k-1)/f)^2 / k^2 of the MACs)."""
    per = cin * cout
    for a, b, ka, kb, pt, pl, t0 in upsampled_fprop_phases(k, f):
        conv_fprop(x, None, cout, ka, kb, 1, y, bias=bias, relu=relu, pads=(pt, pl),
                   w_master=w_phases[t0 * per:(t0 + ka * kb) * per], w_mode=1, out_stride=f, out_phase=(a, b))


def upsampled_wgrad_sums(dy: View, k: int, f: int, g: torch.Tensor):
    """g [n][h/f][w/f][k*k][c] bf16 = shifted f x f block sums of dy (see b2dl_upsampled_wgrad_sums)."""
    check(LIB.b2dl_upsampled_wgrad_sums(dy.act(), k, f, ctypes.c_void_p(g.data_ptr()), _stream()),
          "upsampled_wgrad_sums")


def upsampled_wgrad_layout(x: View, cout: int, k: int):
    """Partial-buffer layout (bytes, weight parts, bias parts, bias offset) of the 1x1 wgrad
    x_low^T g of a k x k conv over a nearest upsampling."""
    n, h, w, _ = x.shape
    g = View(torch.empty((n, h, w, k * k * cout), dtype=torch.bfloat16, device="meta"))
    return wgrad_partials(x, g, 1, 1, 1)


def upsampled_wgrad(x: View, dy: View, k: int, f: int, g: torch.Tensor, partials: torch.Tensor, layout,
                    dw: torch.Tensor, db: torch.Tensor | None):
    """dw HWIO [k*k][cin][cout] (fp32) and db[cout] of a k x k 'same' conv whose input was the nearest
    x f upsampling of x: block sums of dy, one 1x1 wgrad at the low resolution, a permuting reduce."""
    upsampled_wgrad_sums(dy, k, f, g)
    n, h, w, cin = x.shape
    cout = dy.c
    conv_wgrad_deferred(x, View(g.view(n, h, w, k * k * cout)), 1, 1, 1, partials)
    _, wp, bp, bo = layout
    check(LIB.b2dl_upsampled_wgrad_reduce(ctypes.c_void_p(partials.data_ptr()), wp, bp, bo, cin, k, cout,
                                          ctypes.c_void_p(dw.data_ptr()), _ptr(db), _stream()),
          "upsampled_wgrad_reduce")


def nchw_to_nhwc_halo(x: torch.Tensor, y: torch.Tensor, left: int):
    """x fp32 [n][c][h][w] -> y bf16 [n][h][wp][c], column xx at left + xx, zero halo columns."""
    n, c, h, w = x.shape
    check(LIB.b2dl_nchw_to_nhwc_halo(ctypes.c_void_p(x.data_ptr()), n, c, h, w, ctypes.c_void_p(y.data_ptr()),
                                     y.shape[2], left, _stream()), "nchw_to_nhwc_halo")


def nhwc_to_nchw(x: View, y: torch.Tensor, src_f32=False):
    check(LIB.b2dl_nhwc_to_nchw(x.act(), int(src_f32), ctypes.c_void_p(y.data_ptr()), _stream()),
          "nhwc_to_nchw")


def avgpool_fwd(x: View, y: View, k: int):
    check(LIB.b2dl_avgpool_fwd(x.act(), y.act(), k, _stream()), "avgpool_fwd")


def avgpool_bwd(dy: View, dx: View, k: int, accumulate=False, mask: View | None = None):
    check(LIB.b2dl_avgpool_bwd(dy.act(), dx.act(), k, int(accumulate), _act(mask), _stream()),
          "avgpool_bwd")


def upsample_fwd(x: View, y: View, f: int):
    check(LIB.b2dl_upsample_fwd(x.act(), y.act(), f, _stream()), "upsample_fwd")


def upsample_bwd(dy: View, dx: View, f: int, accumulate=False, mask: View | None = None):
    check(LIB.b2dl_upsample_bwd(dy.act(), dx.act(), f, int(accumulate), _act(mask), _stream()),
          "upsample_bwd")


def add(x: View, y: View, accumulate=True, mask: View | None = None):
    check(LIB.b2dl_add(x.act(), y.act(), int(accumulate), _act(mask), _stream()), "add")


def ewise(x0: View, y: View, x1: View | None = None, mask: View | None = None, bias=None, alpha=1.0,
          relu=False, accumulate=False, f32=False):
    """y (+)= mask? * relu?(alpha * x0 * x1? + bias?) (b2dl_ewise): mul / scale / bias_add / relu and VJPs."""
    check(LIB.b2dl_ewise(x0.act(), _act(x1), _act(mask), y.act(), _ptr(bias), float(alpha), int(relu),
                         int(accumulate), int(f32), _stream()), "ewise")


def matmul_w(x: View, b: torch.Tensor, y: View, trans=False, mask: View | None = None, accumulate=False,
             f32=False):
    """Y = X @ B over the width axis (b2dl_matmul_w); trans: dX = dY @ B^T."""
    ldb = x.shape[2] if trans else y.shape[2]
    check(LIB.b2dl_matmul_w(x.act(), ctypes.c_void_p(b.data_ptr()), ldb, int(trans), y.act(), _act(mask),
                            int(accumulate), int(f32), _stream()), "matmul_w")


def matmul_w_grad(x: View, g: View, gb: torch.Tensor, accumulate=False, f32=False):
    check(LIB.b2dl_matmul_w_grad(x.act(), g.act(), ctypes.c_void_p(gb.data_ptr()), int(accumulate), int(f32),
                                 _stream()), "matmul_w_grad")


def channel_sum(g: View, out: torch.Tensor, accumulate=False, f32=False):
    """out[c] (+)= sum over pixels of g (b2dl_channel_sum; bf16 or fp32 storage)."""
    check(LIB.b2dl_channel_sum(g.act(), ctypes.c_void_p(out.data_ptr()), int(accumulate), int(f32), _stream()),
          "channel_sum")


def dgrad_1x1_small(dy: View, w_hwio: torch.Tensor, dx: View, accumulate=False, mask: View | None = None):
    """Input gradient of a 1x1 conv with <= 16 output channels on CUDA cores (channel expansion)."""
    check(LIB.b2dl_dgrad_1x1_small(dy.act(), ctypes.c_void_p(w_hwio.data_ptr()), dx.act(), int(accumulate),
                                   _act(mask), _stream()), "dgrad_1x1_small")


def relu_mask(g: View, act: View):
    check(LIB.b2dl_relu_mask(g.act(), act.act(), _stream()), "relu_mask")


def bias_grad(g: View, out: torch.Tensor, ws: Workspace, accumulate=False):
    a = g.act()
    need = LIB.b2dl_bias_grad_workspace_size(a)
    buf = ws.get(need)
    check(LIB.b2dl_bias_grad(a, ctypes.c_void_p(out.data_ptr()), int(accumulate),
                             ctypes.c_void_p(buf.data_ptr()), buf.numel(), _stream()), "bias_grad")


def wce(logits: View, labels: torch.Tensor, class_weights: torch.Tensor, loss_out: torch.Tensor,
        counts: torch.Tensor, dlogits: View, pred: torch.Tensor | None, ws: Workspace, dlogits_f32=False,
        status: torch.Tensor | None = None, dlogits_scale: float = 1.0):
    n, h, w, c = logits.shape
    need = LIB.b2dl_wce_workspace_size(n, h, w, c)
    buf = ws.get(need)
    check(LIB.b2dl_wce(logits.act(), ctypes.c_void_p(labels.data_ptr()),
                       ctypes.c_void_p(class_weights.data_ptr()), c,
                       ctypes.c_void_p(loss_out.data_ptr()), ctypes.c_void_p(counts.data_ptr()),
                       dlogits.act(), int(dlogits_f32), float(dlogits_scale), _ptr(pred), _ptr(status),
                       ctypes.c_void_p(buf.data_ptr()),
                       buf.numel(), _stream()), "wce")


def larc_update(w: torch.Tensor, m: torch.Tensor, g: torch.Tensor, offsets: torch.Tensor,
                lr: float, momentum: float, trust: float, weight_decay: float, eps: float,
                grad_scale: float, lr_out: torch.Tensor, status: torch.Tensor, ws: Workspace, mode=0,
                w_bf16: torch.Tensor | None = None):
    nt = offsets.numel() - 1
    need = LIB.b2dl_larc_workspace_size(w.numel(), nt)
    buf = ws.get(need)
    a = LarcArgs(w.data_ptr(), m.data_ptr(), g.data_ptr(), offsets.data_ptr(), nt, lr, momentum,
                 trust, weight_decay, eps, grad_scale, lr_out.data_ptr(), status.data_ptr(),
                 buf.data_ptr(), buf.numel(), mode, None if w_bf16 is None else w_bf16.data_ptr())
    check(LIB.b2dl_larc_update(ctypes.byref(a), _stream()), "larc_update")


# ---------------------------------------------------------------- fp32 parity mode (b2dl.h group 3)
def f32_conv(x: View, w_hwio: torch.Tensor, cout: int, kh: int, kw: int, dilation: int, y: View, bias=None,
             residual: View | None = None, relu=False, accumulate=False, mask: View | None = None, pads=None,
             w_mode=1):
    """fp32 NHWC conv (w_mode 1) or input gradient (w_mode 2, w_hwio = the forward conv's HWIO)."""
    pt, pl = pads if pads is not None else (same_pads(kh, dilation)[0], same_pads(kw, dilation)[0])
    a = ConvArgs(x.act(), None, cout, kh, kw, dilation, pt, pl, y.act(), 1, _ptr(bias), _act(residual),
                 int(relu), int(accumulate), _act(mask), 0, ctypes.c_void_p(w_hwio.data_ptr()), w_mode, 0)
    check(LIB.b2dl_f32_conv_fprop(ctypes.byref(a), _stream()), "f32_conv")


def f32_conv_dgrad(dy: View, w_hwio: torch.Tensor, cin: int, kh: int, kw: int, dilation: int, dx: View,
                   accumulate=False, mask: View | None = None, residual: View | None = None):
    pads = (same_pads(kh, dilation)[1], same_pads(kw, dilation)[1])
    f32_conv(dy, w_hwio, cin, kh, kw, dilation, dx, residual=residual, accumulate=accumulate, mask=mask, pads=pads,
             w_mode=2)


def f32_conv_wgrad(x: View, dy: View, kh: int, kw: int, dilation: int, dw: torch.Tensor, ws: Workspace,
                   bias_grad=None, accumulate=False):
    pt, pl = same_pads(kh, dilation)[0], same_pads(kw, dilation)[0]
    a = WgradArgs(x.act(), dy.act(), kh, kw, dilation, pt, pl, ctypes.c_void_p(dw.data_ptr()), _ptr(bias_grad),
                  int(accumulate), None, 0, 0, 0, 0)
    buf = ws.get(LIB.b2dl_f32_wgrad_workspace_size(ctypes.byref(a)))
    a.workspace = ctypes.c_void_p(buf.data_ptr())
    a.workspace_bytes = buf.numel()
    check(LIB.b2dl_f32_conv_wgrad(ctypes.byref(a), _stream()), "f32_conv_wgrad")


def f32_avgpool_fwd(x: View, y: View, k: int):
    check(LIB.b2dl_f32_avgpool_fwd(x.act(), y.act(), k, _stream()), "f32_avgpool_fwd")


def f32_avgpool_bwd(dy: View, dx: View, k: int, accumulate=False, mask: View | None = None):
    check(LIB.b2dl_f32_avgpool_bwd(dy.act(), dx.act(), k, int(accumulate), _act(mask), _stream()), "f32_avgpool_bwd")


def f32_upsample_fwd(x: View, y: View, f: int):
    check(LIB.b2dl_f32_upsample_fwd(x.act(), y.act(), f, _stream()), "f32_upsample_fwd")


def f32_upsample_bwd(dy: View, dx: View, f: int, accumulate=False, mask: View | None = None):
    check(LIB.b2dl_f32_upsample_bwd(dy.act(), dx.act(), f, int(accumulate), _act(mask), _stream()),
          "f32_upsample_bwd")


def f32_add(x: View, y: View, accumulate=False, mask: View | None = None):
    check(LIB.b2dl_f32_add(x.act(), y.act(), int(accumulate), _act(mask), _stream()), "f32_add")


def f32_relu_mask(g: View, act: View):
    f32_add(g, g, accumulate=False, mask=act)


# ---------------------------------------------------------------- batch norm + bilinear
def _is_f32(v: View) -> int:
    return int(v.buf.dtype == torch.float32)


def bn_forward(x: View, gamma: torch.Tensor, beta: torch.Tensor, eps: float, y: View, stats: torch.Tensor,
               ws: Workspace, residual: View | None = None, relu=False):
    """Training-mode batch norm (+ residual, relu); stats [4][C] <- mean, rstd, scale, shift."""
    buf = ws.get(LIB.b2dl_bn_workspace_size(x.c))
    check(LIB.b2dl_bn_forward(x.act(), _ptr(gamma), _ptr(beta), float(eps), _act(residual), int(relu), y.act(),
                              _ptr(stats), ctypes.c_void_p(buf.data_ptr()), buf.numel(), _is_f32(x), _stream()),
          "bn_forward")


def bn_forward_partials(partials: torch.Tensor, tiles: int, x: View, gamma: torch.Tensor, beta: torch.Tensor,
                        eps: float, y: View, stats: torch.Tensor, ws: Workspace, residual: View | None = None,
                        relu=False):
    """bn_forward with the statistics from the producing conv's epilogue partials."""
    buf = ws.get(LIB.b2dl_bn_workspace_size(x.c))
    check(LIB.b2dl_bn_forward_partials(_ptr(partials), int(tiles), x.act(), _ptr(gamma), _ptr(beta), float(eps),
                                       _act(residual), int(relu), y.act(), _ptr(stats),
                                       ctypes.c_void_p(buf.data_ptr()), buf.numel(), _is_f32(x), _stream()),
          "bn_forward_partials")


def bn_backward_partials(partials: torch.Tensor, rows: int, x: View, gy: View, gamma: torch.Tensor,
                         stats: torch.Tensor, dgamma, dbeta, dx: View | None, ws: Workspace, accumulate=False,
                         param_accumulate=False):
    """bn_backward with (sum gy, sum gy*xhat) rows from the consumer dgrad's epilogue."""
    buf = ws.get(LIB.b2dl_bn_workspace_size(x.c))
    check(LIB.b2dl_bn_backward_partials(_ptr(partials), int(rows), x.act(), gy.act(), _ptr(gamma), _ptr(stats),
                                        _ptr(dgamma), _ptr(dbeta), int(param_accumulate), _act(dx), int(accumulate),
                                        ctypes.c_void_p(buf.data_ptr()), buf.numel(), _is_f32(x), _stream()),
          "bn_backward_partials")


def bn_backward(x: View, gy: View, gamma: torch.Tensor, stats: torch.Tensor, dgamma, dbeta, dx: View | None,
                ws: Workspace, accumulate=False, param_accumulate=False):
    buf = ws.get(LIB.b2dl_bn_workspace_size(x.c))
    check(LIB.b2dl_bn_backward(x.act(), gy.act(), _ptr(gamma), _ptr(stats), _ptr(dgamma), _ptr(dbeta),
                               int(param_accumulate), _act(dx), int(accumulate), ctypes.c_void_p(buf.data_ptr()),
                               buf.numel(), _is_f32(x), _stream()), "bn_backward")


def bilinear_fwd(x: View, y: View, f: int):
    check(LIB.b2dl_bilinear_fwd(x.act(), y.act(), f, _is_f32(x), _stream()), "bilinear_fwd")


def bilinear_bwd(dy: View, dx: View, f: int, accumulate=False, mask: View | None = None,
                 ws: Workspace | None = None):
    global _BL_WS
    if ws is None:
        if _BL_WS is None:
            _BL_WS = Workspace(dy.buf.device)
        ws = _BL_WS
    buf = ws.get(LIB.b2dl_bilinear_workspace_size(dy.act(), f))
    check(LIB.b2dl_bilinear_bwd(dy.act(), dx.act(), f, int(accumulate), _act(mask), _is_f32(dy),
                                ctypes.c_void_p(buf.data_ptr()), buf.numel(), _stream()), "bilinear_bwd")


_BL_WS = None
