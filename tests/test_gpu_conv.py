"""tcgen05 implicit-GEMM convolution vs an fp64 reference on bf16-rounded operands.

The kernels compute bf16 x bf16 -> fp32; rounding the operands to bf16 first
leaves only accumulation-order and output-rounding error, so the tolerance is
tight (2e-3 relative, max-abs over max-abs as in the reference's tests,
pkg/tests/test_kernels.py:17-19).
"""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

CASES = [
    # n, cin, h, w, cout, k, dilation
    (1, 64, 16, 32, 64, 3, 1),
    (2, 128, 24, 48, 256, 3, 2),
    (2, 64, 18, 12, 64, 3, 12),
    (2, 256, 16, 16, 512, 1, 1),
    (1, 16, 32, 32, 64, 7, 1),
    (1, 304, 16, 16, 256, 3, 1),
    (2, 256, 16, 16, 3, 1, 1),
    (1, 64, 8, 8, 48, 1, 1),
    (1, 256, 36, 24, 256, 3, 4),
    (2, 128, 9, 13, 128, 3, 1),
]


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


def _bf(t):
    return t.to(torch.bfloat16).to(torch.float64)


def _ref_conv(x, w, d):
    k = w.shape[2]
    p = (k - 1) * d // 2
    return F.conv2d(x, w, padding=p, dilation=d)


@pytest.mark.parametrize("case", CASES)
def test_conv2d_forward_nchw(case):
    from paper_1810_01993_b200.backend_bf16 import conv2d_forward_device
    n, cin, h, w, cout, k, d = case
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, cin, h, w, device="cuda", generator=g)
    wt = torch.randn(cout, cin, k, k, device="cuda", generator=g) / (cin * k * k) ** 0.5
    y = conv2d_forward_device(x, wt, dilation=d)
    ref = _ref_conv(_bf(x), _bf(wt), d)
    assert y.shape == ref.shape
    assert _rel(y, ref) < 2e-3, case


@pytest.mark.parametrize("case", CASES)
def test_conv2d_backward_input_nchw(case):
    from paper_1810_01993_b200.backend_bf16 import conv2d_backward_input_device
    n, cin, h, w, cout, k, d = case
    g = torch.Generator(device="cuda").manual_seed(2)
    dy = torch.randn(n, cout, h, w, device="cuda", generator=g)
    wt = torch.randn(cout, cin, k, k, device="cuda", generator=g)
    dx = conv2d_backward_input_device(dy, wt, (n, cin, h, w), dilation=d)
    xr = torch.zeros(n, cin, h, w, dtype=torch.float64, device="cuda", requires_grad=True)
    _ref_conv(xr, _bf(wt), d).backward(_bf(dy))
    assert _rel(dx, xr.grad) < 2e-3, case


@pytest.mark.parametrize("case", CASES)
def test_conv2d_backward_weights_nchw(case):
    from paper_1810_01993_b200.backend_bf16 import conv2d_backward_weights_device
    n, cin, h, w, cout, k, d = case
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n, cin, h, w, device="cuda", generator=g)
    dy = torch.randn(n, cout, h, w, device="cuda", generator=g)
    dw = conv2d_backward_weights_device(x, dy, (cout, cin, k, k), dilation=d)
    wr = torch.zeros(cout, cin, k, k, dtype=torch.float64, device="cuda", requires_grad=True)
    _ref_conv(_bf(x), wr, d).backward(_bf(dy))
    assert _rel(dw, wr.grad) < 2e-3, case


def test_fprop_fused_epilogue():
    """bias + residual + relu, then accumulate + mask, on channel-slice views."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(0)
    n, h, w, cin, cout = 2, 16, 32, 128, 128
    xb = torch.randn(n, h, w, cin + 64, device="cuda").to(torch.bfloat16)
    x = nhwc.View(xb, 64, cin)
    w_hwio = torch.randn(9, cin, cout, device="cuda") / (9 * cin) ** 0.5
    wp = torch.empty(cout, 9, nhwc.cin_pad(cin), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w_hwio, 3, 3, cin, cout, fprop=wp)
    bias = torch.randn(cout, device="cuda")
    res = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    yb = torch.zeros(n, h, w, cout + 64, dtype=torch.bfloat16, device="cuda")
    y = nhwc.View(yb, 64, cout)
    nhwc.conv_fprop(x, wp, cout, 3, 3, 1, y, bias=bias, residual=nhwc.View(res), relu=True)
    xr = x.tensor().double().permute(0, 3, 1, 2)
    wr = w_hwio.to(torch.bfloat16).double().reshape(3, 3, cin, cout).permute(3, 2, 0, 1)
    ref = F.conv2d(xr, wr, padding=1) + bias.double()[None, :, None, None]
    ref = torch.relu(ref + res.double().permute(0, 3, 1, 2)).permute(0, 2, 3, 1)
    assert _rel(y.tensor(), ref) < 1e-2
    assert yb[..., :64].abs().max() == 0  # untouched neighbours of the slice
    # accumulate + mask
    mask = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    before = y.tensor().double().clone()
    nhwc.conv_fprop(x, wp, cout, 3, 3, 1, y, accumulate=True, mask=nhwc.View(mask))
    conv = F.conv2d(xr, wr, padding=1).permute(0, 2, 3, 1)
    ref2 = before + torch.where(mask.double() > 0, conv, torch.zeros_like(conv))
    assert _rel(y.tensor(), ref2) < 1e-2


@pytest.mark.parametrize("case", [(2, 128, 24, 48, 256, 3, 2), (1, 256, 16, 16, 64, 1, 1), (1, 16, 32, 32, 64, 7, 1),
                                  (2, 64, 18, 12, 48, 3, 12)])
def test_master_layout_weight_modes(case):
    """fprop reading the bf16 HWIO master as an MN-major operand (w_mode 1) and dgrad reading it
    tap-flipped (w_mode 2) equal the packed-weight paths."""
    from paper_1810_01993_b200 import nhwc
    n, cin, h, w, cout, k, d = case
    torch.manual_seed(1)
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    w_hwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    wm = w_hwio.to(torch.bfloat16).contiguous()
    wf = torch.empty(cout, k * k, nhwc.cin_pad(cin), dtype=torch.bfloat16, device="cuda")
    wd = torch.empty(cin, k * k, nhwc.cin_pad(cout), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w_hwio, k, k, cin, cout, fprop=wf, dgrad=wd)
    y0 = torch.zeros(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
    y1 = torch.zeros_like(y0)
    nhwc.conv_fprop(nhwc.View(x), wf, cout, k, k, d, nhwc.View(y0))
    nhwc.conv_fprop(nhwc.View(x), None, cout, k, k, d, nhwc.View(y1), w_master=wm, w_mode=1)
    assert _rel(y1, y0) < 1e-6
    dx0 = torch.zeros(n, h, w, cin, dtype=torch.bfloat16, device="cuda")
    dx1 = torch.zeros_like(dx0)
    nhwc.conv_dgrad(nhwc.View(dy), wd, cin, k, k, d, nhwc.View(dx0))
    nhwc.conv_dgrad(nhwc.View(dy), None, cin, k, k, d, nhwc.View(dx1), w_master=wm)
    # a narrow packed dgrad (cin <= 128) runs on the row-tap kernel: same products, another fp32
    # summation order, so single bf16 output ulps may differ
    assert _rel(dx1, dx0) < (5e-3 if cin <= 128 and k > 1 else 1e-6)


@pytest.mark.parametrize("case", [(1, 256, 36, 24, 256, 3, 4), (2, 128, 24, 48, 512, 3, 2), (1, 64, 9, 13, 320, 1, 1),
                                  (3, 192, 8, 16, 256, 3, 1)])
def test_cta_pair_tiles(case):
    """256-wide N tiles run as CTA pairs (cta_group::2, 256 pixels x 256 channels per pair); odd
    tile counts leave the last odd CTA idle.  All three weight modes plus the fused epilogue."""
    from paper_1810_01993_b200 import nhwc
    n, cin, h, w, cout, k, d = case
    torch.manual_seed(4)
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    w_hwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    wm = w_hwio.to(torch.bfloat16).contiguous()
    wf = torch.empty(cout, k * k, nhwc.cin_pad(cin), dtype=torch.bfloat16, device="cuda")
    wd = torch.empty(cin, k * k, nhwc.cin_pad(cout), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w_hwio, k, k, cin, cout, fprop=wf, dgrad=wd)
    bias = torch.randn(cout, device="cuda")
    res = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    xr = x.double().permute(0, 3, 1, 2)
    wr = wm.double().reshape(k, k, cin, cout).permute(3, 2, 0, 1)
    ref = torch.relu(_ref_conv(xr, wr, d) + bias.double()[None, :, None, None]
                     + res.double().permute(0, 3, 1, 2)).permute(0, 2, 3, 1)
    for mode in (0, 1):
        y = torch.zeros(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
        nhwc.conv_fprop(nhwc.View(x), wf if mode == 0 else None, cout, k, k, d, nhwc.View(y), bias=bias,
                        residual=nhwc.View(res), relu=True, block_n=256, w_master=wm if mode else None, w_mode=mode)
        assert _rel(y, ref) < 1e-2, (case, mode)
    # dgrad (cin >= 256 output channels of the input gradient use pairs too)
    dy = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    xg = torch.zeros(n, cin, h, w, dtype=torch.float64, device="cuda", requires_grad=True)
    _ref_conv(xg, wr, d).backward(dy.double().permute(0, 3, 1, 2))
    gref = xg.grad.permute(0, 2, 3, 1)
    for use_master in (False, True):
        dx = torch.zeros(n, h, w, cin, dtype=torch.float32, device="cuda")
        nhwc.conv_dgrad(nhwc.View(dy), None if use_master else wd, cin, k, k, d, nhwc.View(dx), dx_f32=True,
                        w_master=wm if use_master else None, block_n=256)
        assert _rel(dx, gref) < 2e-3, (case, use_master)


@pytest.mark.parametrize("case", [(2, 16, 32, 48, 64, 7), (1, 16, 20, 24, 64, 7), (1, 8, 16, 16, 32, 5)])
def test_row_window_conv(case):
    """Row-window mode (the 7x7 stem): a haloed NHWC copy of the input, with the kw taps of a
    kernel row folded into K, gives the ordinary conv; wgrad lands in the ordinary HWIO layout."""
    from paper_1810_01993_b200 import nhwc
    n, cin, h, w, cout, k = case
    p = (k - 1) // 2
    torch.manual_seed(5)
    x = torch.randn(n, cin, h, w, device="cuda")
    xw = torch.full((n, h, w + k - 1, cin), 7.0, dtype=torch.bfloat16, device="cuda")  # halo must be zeroed
    nhwc.nchw_to_nhwc_halo(x, xw, p)
    assert torch.equal(xw[:, :, p:p + w].float(), x.to(torch.bfloat16).float().permute(0, 2, 3, 1))
    assert xw[:, :, :p].abs().max() == 0 and xw[:, :, p + w:].abs().max() == 0
    w_hwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    wp = torch.empty(cout, k, nhwc.cin_pad(k * cin), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(w_hwio, k, 1, k * cin, cout, fprop=wp)
    bias = torch.randn(cout, device="cuda")
    y = torch.zeros(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
    nhwc.conv_fprop(nhwc.View(xw), wp, cout, k, 1, 1, nhwc.View(y), bias=bias, relu=True, window=k)
    xr = _bf(x)
    wr = w_hwio.to(torch.bfloat16).double().reshape(k, k, cin, cout).permute(3, 2, 0, 1)
    ref = torch.relu(F.conv2d(xr, wr, padding=p) + bias.double()[None, :, None, None]).permute(0, 2, 3, 1)
    assert _rel(y, ref) < 1e-2
    dy = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    dw = torch.zeros(k * k * cin * cout, device="cuda")
    bg = torch.zeros(cout, device="cuda")
    nhwc.conv_wgrad(nhwc.View(xw), nhwc.View(dy), k, 1, 1, dw, nhwc.Workspace(), bias_grad=bg, window=k)
    wg = torch.zeros(cout, cin, k, k, dtype=torch.float64, device="cuda", requires_grad=True)
    F.conv2d(xr, wg, padding=p).backward(dy.double().permute(0, 3, 1, 2))
    ref_dw = wg.grad.permute(2, 3, 1, 0).reshape(-1)
    assert _rel(dw, ref_dw) < 2e-3
    assert _rel(bg, dy.double().sum((0, 1, 2))) < 1e-4


@pytest.mark.parametrize("cin,cout", [(256, 256), (512, 512), (1024, 256), (2048, 256)])
@pytest.mark.parametrize("d", [1, 2, 4, 12, 18, 24])
def test_atrous_sweep_shapes_vs_oracle(cin, cout, d):
    """Config 5 shapes (tools/atrous_sweep.py times them at full size) against the reference's own
    conv arithmetic (oracle port of _kernels_py.py:44-83) on a cropped 28 x 28 map: fprop, dgrad
    and wgrad through the production NHWC entry points (master-layout weights)."""
    import numpy as np
    from oracle import deskdl_port as ref
    from paper_1810_01993_b200 import nhwc
    n, h, w = 1, 28, 28
    rng = np.random.default_rng(cin + cout + d)
    xq = rng.uniform(-1, 1, (n, cin, h, w)).astype(np.float32)
    dyq = rng.uniform(-1, 1, (n, cout, h, w)).astype(np.float32)
    wq = (rng.uniform(-1, 1, (cout, cin, 3, 3)) / np.sqrt(9 * cin)).astype(np.float32)
    bf = lambda a: torch.from_numpy(a).to(torch.bfloat16)  # noqa: E731
    xb, dyb, wb = bf(xq), bf(dyq), bf(wq)
    x64, dy64, w64 = (t.double().numpy() for t in (xb, dyb, wb))
    y_ref, cols = ref.conv2d_forward(x64, w64, dilation=d)
    dx_ref = ref.conv2d_backward_input(dy64, w64, x64.shape, dilation=d)
    dw_ref = ref.conv2d_backward_weights(cols, dy64, w64.shape, dilation=d)
    x = xb.permute(0, 2, 3, 1).contiguous().cuda()
    dy = dyb.permute(0, 2, 3, 1).contiguous().cuda()
    wm = wb.permute(2, 3, 1, 0).reshape(9, cin, cout).contiguous().cuda()   # HWIO
    y = torch.empty(n, h, w, cout, dtype=torch.float32, device="cuda")
    nhwc.conv_fprop(nhwc.View(x), None, cout, 3, 3, d, nhwc.View(y), y_f32=True, w_master=wm, w_mode=1)
    dx = torch.empty(n, h, w, cin, dtype=torch.float32, device="cuda")
    nhwc.conv_dgrad(nhwc.View(dy), None, cin, 3, 3, d, nhwc.View(dx), dx_f32=True, w_master=wm)
    dw = torch.empty(9 * cin * cout, device="cuda")
    nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), 3, 3, d, dw, nhwc.Workspace())
    y_ref = torch.from_numpy(y_ref).permute(0, 2, 3, 1)
    dx_ref = torch.from_numpy(dx_ref).permute(0, 2, 3, 1)
    dw_ref = torch.from_numpy(dw_ref).permute(2, 3, 1, 0).reshape(-1)
    assert _rel(y.cpu(), y_ref) < 2e-3
    assert _rel(dx.cpu(), dx_ref) < 2e-3
    assert _rel(dw.cpu(), dw_ref) < 2e-3


@pytest.mark.parametrize("cout,k", [(320, 1), (864, 1), (352, 3)])
def test_partial_last_n_tile_many_tiles_per_cta(cout, k):
    """Output channels that leave whole epilogue sub-groups without a chunk in the last N tile,
    with several tiles per persistent CTA and a TMA-loaded operand (mask): the operand prefetch
    chain must skip over tiles a sub-group has no work in (regression: Tiramisu squeeze dgrad)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(9)
    n, h, w, cin = 2, 96, 96, 64
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    wm = (torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5).to(torch.bfloat16)
    mask = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    y = torch.zeros(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
    nhwc.conv_fprop(nhwc.View(x), None, cout, k, k, 1, nhwc.View(y), mask=nhwc.View(mask), w_master=wm, w_mode=1)
    torch.cuda.synchronize()
    xr = x.double().permute(0, 3, 1, 2)
    wr = wm.double().reshape(k, k, cin, cout).permute(3, 2, 0, 1)
    ref = F.conv2d(xr, wr, padding=(k - 1) // 2).permute(0, 2, 3, 1)
    ref = torch.where(mask.double() > 0, ref, torch.zeros_like(ref))
    assert _rel(y, ref) < 1e-2


@pytest.mark.parametrize("n,cin,h,w,cout,k,f", [(2, 64, 9, 12, 64, 3, 4), (1, 256, 8, 6, 256, 3, 4),
                                                 (2, 32, 7, 5, 48, 3, 2), (1, 64, 6, 8, 64, 5, 2)])
def test_upsampled_dgrad_equals_dgrad_plus_block_sum(n, cin, h, w, cout, k, f):
    """Input gradient of a k x k conv over a nearest x f upsampling, block-summed (the upsample VJP),
    computed as one strided conv with merged weights == autograd through upsample + conv (fp64)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(11)
    w_hwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    dy = torch.randn(n, h * f, w * f, cout, device="cuda").to(torch.bfloat16)
    mask = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    kk = k + f - 1
    wm = torch.empty(cin, kk * kk, nhwc.cin_pad(cout), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_upsampled_dgrad(w_hwio, k, cin, cout, f, wm)
    dx = torch.empty(n, h, w, cin, dtype=torch.bfloat16, device="cuda")
    nhwc.upsampled_dgrad(nhwc.View(dy), wm, cin, k, f, nhwc.View(dx), mask=nhwc.View(mask))
    x = torch.zeros(n, cin, h, w, dtype=torch.float64, device="cuda", requires_grad=True)
    xu = x.repeat_interleave(f, 2).repeat_interleave(f, 3)
    wr = w_hwio.double().reshape(k, k, cin, cout).permute(3, 2, 0, 1)
    F.conv2d(xu, wr, padding=(k - 1) // 2).backward(dy.double().permute(0, 3, 1, 2))
    ref = x.grad.permute(0, 2, 3, 1)
    ref = torch.where(mask.double() > 0, ref, torch.zeros_like(ref))
    assert _rel(dx, ref) < 1e-2   # merged weights are rounded to bf16 once


@pytest.mark.gpu
def test_reduce_segments_paths():
    """Split-K partial reduction over a table of segments covering every kernel path (long rows in
    16-byte lanes, short rows with many partials -- vector and scalar -- and unaligned rows):
    equal to the fp64 sum, and bitwise repeatable."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(5)
    cases = [(590_000, 16, 0, 0), (256, 144, 1, 0), (768, 592, 0, 0), (3, 592, 1, 0), (1001, 7, 1, 1),
             (64, 40, 0, 2), (20_000, 3, 1, 0)]
    srcs, segs, ref = [], [], []
    dst = torch.randn(sum(n + 8 for n, *_ in cases), device="cuda")
    dst0 = dst.clone()
    off = 0
    for n, parts, acc, mis in cases:
        buf = torch.randn(parts * n + mis, device="cuda")
        srcs.append(buf)
        src = buf[mis:]
        segs.append((src.data_ptr(), off + mis, n, parts, acc))
        r = src.double().view(parts, n).sum(0)
        if acc:
            r = r + dst0[off + mis:off + mis + n].double()
        ref.append((off + mis, n, r))
        off += n + 8
    table = nhwc.segment_table(segs, "cuda")
    max_n = max(n for n, *_ in cases)
    nhwc.reduce_segments(table, len(segs), max_n, dst)
    first = dst.clone()
    for o, n, r in ref:
        assert torch.allclose(dst[o:o + n].double(), r, rtol=1e-5, atol=1e-4)
    dst.copy_(dst0)
    nhwc.reduce_segments(table, len(segs), max_n, dst)
    assert torch.equal(dst, first)


@pytest.mark.parametrize("n,cin,h,w,cout,k,f", [(1, 64, 6, 8, 64, 3, 4), (2, 256, 9, 12, 256, 3, 4), (1, 128, 8, 8, 64, 3, 2),
                                                (1, 64, 5, 7, 128, 5, 4), (1, 64, 4, 6, 64, 1, 4)])
def test_upsampled_fprop_equals_conv_of_upsampling(n, cin, h, w, cout, k, f):
    """Forward of a k x k conv over a nearest x f upsampling, computed per output phase from the
    low-resolution input with merged weights (stride-f phase views of y) == conv2d(upsample) (fp64)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(12)
    w_hwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    bias = torch.randn(cout, device="cuda")
    wp = torch.empty(nhwc.upsampled_fprop_taps(k, f) * cin * cout, dtype=torch.bfloat16, device="cuda")
    nhwc.pack_upsampled_fprop(w_hwio, k, cin, cout, f, wp)
    y = torch.full((n, h * f, w * f, cout), float("nan"), dtype=torch.bfloat16, device="cuda")
    nhwc.upsampled_fprop(nhwc.View(x), wp, cin, cout, k, f, nhwc.View(y), bias=bias, relu=True)
    xu = x.double().permute(0, 3, 1, 2).repeat_interleave(f, 2).repeat_interleave(f, 3)
    wr = w_hwio.double().reshape(k, k, cin, cout).permute(3, 2, 0, 1)
    ref = torch.relu(F.conv2d(xu, wr, padding=(k - 1) // 2) + bias.double()[None, :, None, None]).permute(0, 2, 3, 1)
    assert not torch.isnan(y).any()
    assert _rel(y, ref) < 1e-2   # merged weights are rounded to bf16 once


@pytest.mark.parametrize("n,cin,h,w,cout,k,f", [(1, 64, 6, 8, 64, 3, 4), (2, 256, 9, 12, 256, 3, 4), (1, 128, 8, 8, 64, 3, 2),
                                                (1, 64, 4, 6, 128, 1, 4), (1, 64, 5, 19, 72, 3, 4),
                                                (2, 64, 3, 40, 256, 3, 4)])
def test_upsampled_wgrad_equals_wgrad_of_upsampling(n, cin, h, w, cout, k, f):
    """Weight + bias gradient of a k x k conv over a nearest x f upsampling from the low-resolution
    input (shifted block sums of dy, a 1x1 wgrad, a permuting reduce) == autograd (fp64)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(13)
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(n, h * f, w * f, cout, device="cuda").to(torch.bfloat16)
    lay = nhwc.upsampled_wgrad_layout(nhwc.View(x), cout, k)
    parts = torch.empty(lay[0], dtype=torch.uint8, device="cuda")
    g = torch.empty(n * h * w * k * k * cout, dtype=torch.bfloat16, device="cuda")
    dw = torch.full((k * k * cin * cout,), float("nan"), device="cuda")
    db = torch.full((cout,), float("nan"), device="cuda")
    nhwc.upsampled_wgrad(nhwc.View(x), nhwc.View(dy), k, f, g, parts, lay, dw, db)
    xu = x.double().permute(0, 3, 1, 2).repeat_interleave(f, 2).repeat_interleave(f, 3)
    wr = torch.zeros(cout, cin, k, k, dtype=torch.float64, device="cuda", requires_grad=True)
    br = torch.zeros(cout, dtype=torch.float64, device="cuda", requires_grad=True)
    F.conv2d(xu, wr, br, padding=(k - 1) // 2).backward(dy.double().permute(0, 3, 1, 2))
    ref_w = wr.grad.permute(2, 3, 1, 0).reshape(-1)   # HWIO
    assert _rel(dw, ref_w) < 1e-2   # block sums are rounded to bf16 once
    assert _rel(db, br.grad) < 1e-2


@pytest.mark.parametrize("c", [6, 64])
def test_upsampled_wgrad_sums_vs_torch(c):
    """Shifted 4 x 4 block sums of dy (2- and 4-channel thread paths): G_t[i] = sum of the padded dy
    over rows / cols [4i + 2 - t, 4i + 6 - t)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(14)
    n, H, W, f, k = 2, 16, 20, 4, 3
    dy = torch.randn(n, H, W, c, device="cuda").to(torch.bfloat16)
    g = torch.empty(n * (H // f) * (W // f) * k * k * c, dtype=torch.bfloat16, device="cuda")
    nhwc.upsampled_wgrad_sums(nhwc.View(dy), k, f, g)
    dyp = F.pad(dy.double().permute(0, 3, 1, 2), (1, 1, 1, 1))
    ref = torch.stack([F.avg_pool2d(dyp[:, :, 2 - ty:2 - ty + H, 2 - tx:2 - tx + W], f) * f * f
                       for ty in range(k) for tx in range(k)], 1)      # [n, taps, c, h, w]
    ref = ref.permute(0, 3, 4, 1, 2)                                   # [n, h, w, taps, c]
    assert _rel(g.view(ref.shape), ref) < 1e-2


@pytest.mark.parametrize("c32,k,cout", [(32, 5, 48), (24, 3, 256), (32, 1, 64)])
def test_kblk32_fprop_and_dgrad_vs_fp64(c32, k, cout):
    """17..32-channel inputs through the master-weight modes use 32-channel K blocks (SW64): the
    forward over a growth-32 tensor and the dgrad over a 32-channel dy (Tiramisu dense layers)."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(5)
    n, h, w = 2, 24, 40
    x = torch.randn(n, h, w, c32, device="cuda").to(torch.bfloat16)
    wm = (torch.randn(k * k, c32, cout, device="cuda") / (k * k * c32) ** 0.5).to(torch.bfloat16)
    y = torch.empty(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
    nhwc.conv_fprop(nhwc.View(x), None, cout, k, k, 1, nhwc.View(y), w_master=wm, w_mode=1)
    xr = x.permute(0, 3, 1, 2).double()
    wr = wm.double().view(k, k, c32, cout).permute(3, 2, 0, 1)
    ref = F.conv2d(xr, wr, padding=(k - 1) // 2)
    assert _rel(y.permute(0, 3, 1, 2), ref) < 1e-2
    # dgrad over a 32-channel dy: this conv maps cout -> c32; dx has c32... use (co=c32, ci=cout)
    dy = torch.randn(n, h, w, c32, device="cuda").to(torch.bfloat16)
    wd = (torch.randn(k * k, cout, c32, device="cuda") / (k * k * c32) ** 0.5).to(torch.bfloat16)  # HWIO cin=cout
    dx = torch.empty(n, h, w, cout, dtype=torch.bfloat16, device="cuda")
    nhwc.conv_dgrad(nhwc.View(dy), None, cout, k, k, 1, nhwc.View(dx), w_master=wd)
    xg = torch.zeros(n, cout, h, w, dtype=torch.float64, device="cuda", requires_grad=True)
    F.conv2d(xg, wd.double().view(k, k, cout, c32).permute(3, 2, 0, 1), padding=(k - 1) // 2).backward(
        dy.permute(0, 3, 1, 2).double())
    assert _rel(dx.permute(0, 3, 1, 2), xg.grad) < 1e-2


@pytest.mark.parametrize("cin,cout,k,d,ops,hw", [(96, 32, 5, 1, "", (37, 45)), (200, 64, 5, 1, "rm", (37, 45)),
                                                  (24, 32, 5, 1, "", (37, 45)), (32, 64, 7, 1, "m", (20, 30)),
                                                  (48, 32, 5, 2, "a", (37, 45)), (40, 24, 5, 1, "", (37, 45)),
                                                  (416, 32, 5, 1, "", (4, 3)), (96, 32, 5, 1, "", (8, 6)),
                                                  (64, 32, 5, 1, "", (16, 12)), (64, 64, 3, 1, "m", (37, 45)),
                                                  (64, 64, 3, 2, "rm", (37, 45)), (48, 32, 3, 1, "a", (20, 30)),
                                                  (32, 96, 5, 1, "m", (37, 45)), (32, 128, 5, 1, "", (20, 30)),
                                                  (128, 128, 3, 1, "rm", (37, 45)), (64, 80, 3, 2, "a", (16, 12)),
                                                  (32, 192, 5, 1, "m", (20, 30)), (32, 256, 3, 1, "", (37, 45)),
                                                  (24, 32, 7, 1, "", (20, 30)), (32, 32, 7, 1, "r", (37, 45))])
def test_rowtap_fprop_vs_fp64(cin, cout, k, d, ops, hw, n=2):
    """Narrow-output convs through the row-tap kernel (one tall input box per column tap and
    channel block, row taps at 1 KB offsets): bias, relu, residual / mask / accumulate epilogue
    operands, dilation, ragged image edges, against fp64 on the same bf16 operands."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(11)
    h, w = hw
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    whwio = torch.randn(k * k, cin, cout, device="cuda") / (k * k * cin) ** 0.5
    wp = torch.empty(cout, k * k, nhwc.cin_pad(cin), dtype=torch.bfloat16, device="cuda")
    nhwc.pack_weights(whwio, k, k, cin, cout, fprop=wp)
    b = torch.randn(cout, device="cuda") * 0.1
    cs = (cout + 7) // 8 * 8
    y = torch.randn(n, h, w, cs, device="cuda").to(torch.bfloat16)
    y0 = y.clone()
    res = torch.randn(n, h, w, cs, device="cuda").to(torch.bfloat16) if "r" in ops else None
    mask = torch.randn(n, h, w, cs, device="cuda").to(torch.bfloat16) if "m" in ops else None
    acc = "a" in ops
    nhwc.conv_fprop(nhwc.View(x), wp, cout, k, k, d, nhwc.View(y, 0, cout), bias=b,
                    residual=nhwc.View(res, 0, cout) if res is not None else None,
                    mask=nhwc.View(mask, 0, cout) if mask is not None else None, relu=True, accumulate=acc)
    wr = whwio.to(torch.bfloat16).double().view(k, k, cin, cout).permute(3, 2, 0, 1)
    ref = F.conv2d(x.permute(0, 3, 1, 2).double(), wr, padding=(k - 1) * d // 2, dilation=d) + b.double()[None, :, None, None]
    if res is not None:
        ref = ref + res[..., :cout].permute(0, 3, 1, 2).double()
    ref = ref.clamp_min(0)
    if mask is not None:
        ref = ref * (mask[..., :cout].permute(0, 3, 1, 2).double() > 0)
    if acc:
        ref = ref + y0[..., :cout].permute(0, 3, 1, 2).double()
    assert _rel(y[..., :cout].permute(0, 3, 1, 2), ref) < 1e-2


@pytest.mark.parametrize("cin,cout,k,d,ops,hw", [(96, 32, 5, 1, "m", (16, 24)), (32, 128, 3, 1, "", (16, 40)),
                                                  (64, 64, 3, 1, "r", (48, 8))])
def test_rowtap_fprop_odd_tile_count(cin, cout, k, d, ops, hw):
    """One image with an odd number of 8 x 16 tiles: the CTA pair's second tile of the last pair is
    past the end (zero-filled loads, no stores)."""
    test_rowtap_fprop_vs_fp64(cin, cout, k, d, ops, hw, n=1)


@pytest.mark.parametrize("cin,cout,k,d,hw", [(96, 32, 5, 1, (37, 45)), (416, 32, 5, 1, (64, 48)),
                                             (200, 64, 5, 2, (33, 29)), (40, 24, 5, 1, (16, 12)),
                                             (64, 32, 5, 1, (4, 3)), (64, 64, 3, 1, (72, 48)),
                                             (64, 64, 3, 2, (33, 29)), (48, 32, 3, 1, (16, 12))])
def test_rowtap_wgrad_vs_fp64(cin, cout, k, d, hw):
    """Narrow-output weight gradient through the row-tap kernel (tall x boxes shared by the kh tap
    rows, one TMEM accumulator per tap row): dW and the bias gradient vs fp64 on bf16 operands."""
    from paper_1810_01993_b200 import nhwc
    torch.manual_seed(13)
    n, (h, w) = 2, hw
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(n, h, w, cout, device="cuda").to(torch.bfloat16)
    dw = torch.empty(k * k * cin * cout, device="cuda")
    db = torch.empty(cout, device="cuda")
    nhwc.conv_wgrad(nhwc.View(x), nhwc.View(dy), k, k, d, dw, nhwc.Workspace(), bias_grad=db)
    wr = torch.zeros(cout, cin, k, k, dtype=torch.float64, device="cuda", requires_grad=True)
    F.conv2d(x.permute(0, 3, 1, 2).double(), wr, padding=(k - 1) * d // 2, dilation=d).backward(
        dy.permute(0, 3, 1, 2).double())
    got = dw.view(k, k, cin, cout).permute(3, 2, 0, 1)
    assert _rel(got, wr.grad) < 1e-3
    assert _rel(db, dy.double().sum(dim=(0, 1, 2))) < 1e-4
