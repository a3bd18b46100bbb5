"""Drop-in convolution backend for the reference's kernel protocol, at the caller's precision.

The reference selects a module exposing BACKEND_NAME, conv2d_forward, conv2d_backward_weights
and conv2d_backward_input (pkg/src/deskdl/model/kernels.py:19-40; implementations
_kernels_py.py:44-83 and _kernels_cy.py:13-44).  This module has the same names, argument
meaning, output dtypes and error behaviour (stride != 1 -> NotImplementedError, channel mismatch
-> ValueError, _kernels_py.py:46-51) and runs every product on the GPU through the
reference-precision C entry points of libb2dl.so (include/b2dl.h, b2dl_conv2d_*_typed;
csrc/refconv.cu): float64 arrays are convolved in fp64, everything else in fp32, like the
Cython core's fused type (_convkernels.pyx:11-13).  The reference's own kernel tests therefore
apply unchanged (1e-12 against the loop oracle in float64, 1e-7 finite differences, 1e-5
agreement with the other backends in float32: pkg/tests/test_kernels.py:28-82).

The `*_device` variants take and return CUDA tensors (torch float32 / float64); the protocol
functions take and return NumPy arrays like the reference.  The bf16 tensor-core arithmetic of
the training step is the separate, explicitly named backend `backend_bf16` ("b200-bf16").
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import LIB, check

BACKEND_NAME = "b200"

B2DL_DTYPE_F32, B2DL_DTYPE_F64 = 0, 1


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _compute_dtype(*dtypes) -> torch.dtype:
    return torch.float64 if any(d == torch.float64 for d in dtypes) else torch.float32


def _code(dt: torch.dtype) -> int:
    return B2DL_DTYPE_F64 if dt == torch.float64 else B2DL_DTYPE_F32


def conv2d_forward_device(x: torch.Tensor, w: torch.Tensor, stride=1, dilation=1) -> torch.Tensor:
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x.shape
    cout, cin_w, kh, kw = w.shape
    if cin != cin_w:
        raise ValueError(f"conv2d: input channels {cin} != weight channels {cin_w}")
    dt = _compute_dtype(x.dtype, w.dtype)
    x = x.to(dt).contiguous()
    w = w.to(device=x.device, dtype=dt).contiguous()
    y = torch.empty(n, cout, h, wd, dtype=dt, device=x.device)
    check(LIB.b2dl_conv2d_forward_typed(_code(dt), _p(x), _p(w), _p(y), n, cin, h, wd, cout, kh, kw, stride,
                                        dilation, _stream()), "conv2d_forward")
    return y


def conv2d_backward_input_device(dy: torch.Tensor, w: torch.Tensor, x_shape, stride=1,
                                 dilation=1) -> torch.Tensor:
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x_shape
    cout, cin_w, kh, kw = w.shape
    if cin != cin_w or tuple(dy.shape) != (n, cout, h, wd):
        raise ValueError(f"conv2d_backward_input: shapes {tuple(dy.shape)} / {tuple(w.shape)} / {tuple(x_shape)}")
    dt = _compute_dtype(dy.dtype, w.dtype)
    dy = dy.to(dt).contiguous()
    w = w.to(device=dy.device, dtype=dt).contiguous()
    dx = torch.empty(n, cin, h, wd, dtype=dt, device=dy.device)
    check(LIB.b2dl_conv2d_backward_input_typed(_code(dt), _p(dy), _p(w), _p(dx), n, cin, h, wd, cout, kh, kw,
                                               stride, dilation, _stream()), "conv2d_backward_input")
    return dx


def conv2d_backward_weights_device(x: torch.Tensor, dy: torch.Tensor, w_shape, dilation=1) -> torch.Tensor:
    cout, cin, kh, kw = w_shape
    n, cin_x, h, wd = x.shape
    if cin_x != cin or tuple(dy.shape) != (n, cout, h, wd):
        raise ValueError(f"conv2d_backward_weights: shapes {tuple(x.shape)} / {tuple(dy.shape)} / {tuple(w_shape)}")
    dt = _compute_dtype(x.dtype, dy.dtype)
    x = x.to(dt).contiguous()
    dy = dy.to(device=x.device, dtype=dt).contiguous()
    dw = torch.empty(cout, cin, kh, kw, dtype=dt, device=x.device)
    check(LIB.b2dl_conv2d_backward_weights_typed(_code(dt), _p(x), _p(dy), _p(dw), n, cin, h, wd, cout, kh, kw,
                                                 dilation, _stream()), "conv2d_backward_weights")
    return dw


# ---------------------------------------------------------------- reference protocol (NumPy)

def _to_dev(a):
    a = np.asarray(a)
    if a.dtype != np.float64:
        a = a.astype(np.float32, copy=False)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def conv2d_forward(x, w, stride=1, dilation=1):
    """Same-padded 2D convolution; returns (output, cache for backward).  The cache is the input
    itself (like the Cython backend's padded input, it is backend-private)."""
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    x = np.asarray(x)
    w = np.asarray(w)
    if x.shape[1] != w.shape[1]:
        raise ValueError(f"conv2d: input channels {x.shape[1]} != weight channels {w.shape[1]}")
    y = conv2d_forward_device(_to_dev(x), _to_dev(w), stride, dilation)
    return y.cpu().numpy().astype(np.result_type(x, w), copy=False), x


def conv2d_backward_weights(cache, dy, w_shape, dilation=1):
    x = np.asarray(cache)
    dy = np.asarray(dy)
    dw = conv2d_backward_weights_device(_to_dev(x), _to_dev(dy), tuple(w_shape), dilation)
    return dw.cpu().numpy().astype(np.result_type(x, dy), copy=False)


def conv2d_backward_input(dy, w, x_shape, stride=1, dilation=1):
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    dy = np.asarray(dy)
    w = np.asarray(w)
    dx = conv2d_backward_input_device(_to_dev(dy), _to_dev(w), tuple(x_shape), stride, dilation)
    return dx.cpu().numpy().astype(np.result_type(dy, w), copy=False)


def install(kernels_module=None):
    """Make this backend the one the reference's executor calls: rebinds the protocol functions
    and BACKEND of `deskdl.model.kernels` (what a DESKDL_KERNELS=b200 branch at kernels.py:24-32
    would do at import).  Returns the previous bindings for `uninstall`."""
    if kernels_module is None:
        from deskdl.model import kernels as kernels_module
    names = ("BACKEND", "conv2d_forward", "conv2d_backward_input", "conv2d_backward_weights")
    prev = {k: getattr(kernels_module, k) for k in names}
    kernels_module.BACKEND = BACKEND_NAME
    kernels_module.conv2d_forward = conv2d_forward
    kernels_module.conv2d_backward_input = conv2d_backward_input
    kernels_module.conv2d_backward_weights = conv2d_backward_weights
    return kernels_module, prev


def uninstall(handle):
    mod, prev = handle
    for k, v in prev.items():
        setattr(mod, k, v)
