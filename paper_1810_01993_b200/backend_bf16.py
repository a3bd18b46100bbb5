"""bf16 tensor-core convolution backend for the reference's kernel protocol (opt-in).

NOT the precision drop-in: that is `backend` (BACKEND_NAME "b200"), which computes in the
caller's float32 / float64.  This module runs the same protocol on the training step's
arithmetic -- operands rounded to bf16, fp32 accumulation, ~1e-2 relative -- and says so in its
name ("b200-bf16"); float64 callers get bf16-accurate numbers.

The reference selects a module exposing BACKEND_NAME, conv2d_forward,
conv2d_backward_weights and conv2d_backward_input
(pkg/src/deskdl/model/kernels.py:19-40; implementations _kernels_py.py:44-83
and _kernels_cy.py:13-44).  This module has the same names, argument meaning
and error behaviour (stride != 1 -> NotImplementedError, channel mismatch ->
ValueError, _kernels_py.py:46-51) and runs every product on the sm_100a
tensor-core kernels of libb2dl.so via its NCHW fp32 C entry points
(include/b2dl.h group 1).  Arithmetic is bf16 x bf16 -> fp32 ("bf16 mode").

The `*_device` variants take and return CUDA tensors; the protocol functions
take and return NumPy arrays like the reference.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import LIB, check

BACKEND_NAME = "b200-bf16"


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ws(n, cin, h, w, cout, kh, kw):
    nbytes = LIB.b2dl_conv2d_workspace_size(n, cin, h, w, cout, kh, kw)
    return torch.empty(nbytes, dtype=torch.uint8, device="cuda")


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def conv2d_forward_device(x: torch.Tensor, w: torch.Tensor, stride=1, dilation=1) -> torch.Tensor:
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x.shape
    cout, cin_w, kh, kw = w.shape
    if cin != cin_w:
        raise ValueError(f"conv2d: input channels {cin} != weight channels {cin_w}")
    x = x.contiguous().float()
    w = w.contiguous().float()
    y = torch.empty(n, cout, h, wd, dtype=torch.float32, device=x.device)
    ws = _ws(n, cin, h, wd, cout, kh, kw)
    check(LIB.b2dl_conv2d_forward(_p(x), _p(w), _p(y), n, cin, h, wd, cout, kh, kw, stride, dilation,
                                  _p(ws), ws.numel(), _stream()), "conv2d_forward")
    return y


def conv2d_backward_input_device(dy: torch.Tensor, w: torch.Tensor, x_shape, stride=1,
                                 dilation=1) -> torch.Tensor:
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x_shape
    cout, cin_w, kh, kw = w.shape
    if cin != cin_w or tuple(dy.shape) != (n, cout, h, wd):
        raise ValueError(f"conv2d_backward_input: shapes {tuple(dy.shape)} / {tuple(w.shape)} / {x_shape}")
    dy = dy.contiguous().float()
    w = w.contiguous().float()
    dx = torch.empty(n, cin, h, wd, dtype=torch.float32, device=dy.device)
    ws = _ws(n, cin, h, wd, cout, kh, kw)
    check(LIB.b2dl_conv2d_backward_input(_p(dy), _p(w), _p(dx), n, cin, h, wd, cout, kh, kw, stride,
                                         dilation, _p(ws), ws.numel(), _stream()),
          "conv2d_backward_input")
    return dx


def conv2d_backward_weights_device(x: torch.Tensor, dy: torch.Tensor, w_shape, dilation=1) -> torch.Tensor:
    cout, cin, kh, kw = w_shape
    n, cin_x, h, wd = x.shape
    if cin_x != cin or tuple(dy.shape) != (n, cout, h, wd):
        raise ValueError(f"conv2d_backward_weights: shapes {tuple(x.shape)} / {tuple(dy.shape)} / {w_shape}")
    x = x.contiguous().float()
    dy = dy.contiguous().float()
    dw = torch.empty(cout, cin, kh, kw, dtype=torch.float32, device=x.device)
    ws = _ws(n, cin, h, wd, cout, kh, kw)
    check(LIB.b2dl_conv2d_backward_weights(_p(x), _p(dy), _p(dw), n, cin, h, wd, cout, kh, kw,
                                           dilation, _p(ws), ws.numel(), _stream()),
          "conv2d_backward_weights")
    return dw


# ---------------------------------------------------------------- reference protocol (NumPy)

def _to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def conv2d_forward(x, w, stride=1, dilation=1):
    """Same-padded 2D convolution; returns (output, cache for backward)."""
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    x = np.asarray(x)
    if x.shape[1] != np.shape(w)[1]:
        raise ValueError(f"conv2d: input channels {x.shape[1]} != weight channels {np.shape(w)[1]}")
    y = conv2d_forward_device(_to_dev(x), _to_dev(w), stride, dilation)
    return y.cpu().numpy().astype(x.dtype, copy=False), x


def conv2d_backward_weights(cache, dy, w_shape, dilation=1):
    x = cache
    dw = conv2d_backward_weights_device(_to_dev(x), _to_dev(dy), tuple(w_shape), dilation)
    return dw.cpu().numpy().astype(np.asarray(dy).dtype, copy=False)


def conv2d_backward_input(dy, w, x_shape, stride=1, dilation=1):
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    dx = conv2d_backward_input_device(_to_dev(dy), _to_dev(w), tuple(x_shape), stride, dilation)
    return dx.cpu().numpy().astype(np.asarray(dy).dtype, copy=False)
