"""ctypes binding of libb2dl.so (the C ABI in include/b2dl.h).

This is the only place Python touches the native library.  There is no
fallback: if the shared library is missing or was built without sm_100a code,
importing the package fails loudly (the product never silently runs on CPU).
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# B2DL_LIB_PATH: load another build of the same ABI (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("B2DL_LIB_PATH") or os.path.join(HERE, "libb2dl.so")

B2DL_OK = 0
B2DL_E_NOT_IMPLEMENTED = 1
B2DL_E_VALUE = 2
B2DL_E_CUDA = 3
B2DL_E_ALIGN = 4
B2DL_E_NONFINITE = 5


class Act(ctypes.Structure):
    """b2dl_act: NHWC view (ptr at channel offset, c channels, pitch c_stride)."""
    _fields_ = [("ptr", ctypes.c_void_p), ("n", ctypes.c_int), ("h", ctypes.c_int),
                ("w", ctypes.c_int), ("c", ctypes.c_int), ("c_stride", ctypes.c_int)]


NULL_ACT = Act(None, 0, 0, 0, 0, 0)


class ConvArgs(ctypes.Structure):
    _fields_ = [("x", Act), ("w_packed", ctypes.c_void_p), ("cout", ctypes.c_int),
                ("kh", ctypes.c_int), ("kw", ctypes.c_int), ("dilation", ctypes.c_int),
                ("pad_top", ctypes.c_int), ("pad_left", ctypes.c_int), ("y", Act),
                ("y_f32", ctypes.c_int), ("bias", ctypes.c_void_p), ("residual", Act),
                ("relu", ctypes.c_int), ("accumulate", ctypes.c_int), ("mask", Act),
                ("block_n", ctypes.c_int), ("w_master", ctypes.c_void_p), ("w_mode", ctypes.c_int),
                ("window", ctypes.c_int), ("in_stride", ctypes.c_int), ("out_stride", ctypes.c_int),
                ("out_phase_h", ctypes.c_int), ("out_phase_w", ctypes.c_int), ("bn_partial", ctypes.c_void_p),
                ("bnb_stats", ctypes.c_void_p), ("bnb_partial", ctypes.c_void_p)]


class WgradArgs(ctypes.Structure):
    _fields_ = [("x", Act), ("dy", Act), ("kh", ctypes.c_int), ("kw", ctypes.c_int),
                ("dilation", ctypes.c_int), ("pad_top", ctypes.c_int), ("pad_left", ctypes.c_int),
                ("dw", ctypes.c_void_p), ("bias_grad", ctypes.c_void_p),
                ("accumulate", ctypes.c_int), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("splits", ctypes.c_int),
                ("defer_reduce", ctypes.c_int), ("window", ctypes.c_int)]


class Segment(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst_off", ctypes.c_int64), ("n", ctypes.c_int64),
                ("parts", ctypes.c_int32), ("accumulate", ctypes.c_int32)]


class LarcArgs(ctypes.Structure):
    _fields_ = [("w", ctypes.c_void_p), ("m", ctypes.c_void_p), ("g", ctypes.c_void_p),
                ("offsets", ctypes.c_void_p), ("ntensors", ctypes.c_int),
                ("lr", ctypes.c_float), ("momentum", ctypes.c_float), ("trust", ctypes.c_float),
                ("weight_decay", ctypes.c_float), ("eps", ctypes.c_float),
                ("grad_scale", ctypes.c_float), ("lr_out", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("mode", ctypes.c_int), ("w_bf16", ctypes.c_void_p)]


# every symbol include/b2dl.h declares, with its ctypes signature
_c_int, _vp, _sz = ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
_SIGS = {
    "b2dl_conv2d_workspace_size": (_sz, [_c_int] * 7),
    "b2dl_conv2d_forward": (_c_int, [_vp, _vp, _vp] + [_c_int] * 9 + [_vp, _sz, _vp]),
    "b2dl_conv2d_backward_input": (_c_int, [_vp, _vp, _vp] + [_c_int] * 9 + [_vp, _sz, _vp]),
    "b2dl_conv2d_backward_weights": (_c_int, [_vp, _vp, _vp] + [_c_int] * 8 + [_vp, _sz, _vp]),
    "b2dl_conv2d_forward_typed": (_c_int, [_c_int, _vp, _vp, _vp] + [_c_int] * 9 + [_vp]),
    "b2dl_conv2d_backward_input_typed": (_c_int, [_c_int, _vp, _vp, _vp] + [_c_int] * 9 + [_vp]),
    "b2dl_conv2d_backward_weights_typed": (_c_int, [_c_int, _vp, _vp, _vp] + [_c_int] * 8 + [_vp]),
    "b2dl_ewise": (_c_int, [Act, Act, Act, Act, _vp, ctypes.c_float, _c_int, _c_int, _c_int, _vp]),
    "b2dl_matmul_w": (_c_int, [Act, _vp, _c_int, _c_int, Act, Act, _c_int, _c_int, _vp]),
    "b2dl_matmul_w_grad": (_c_int, [Act, Act, _vp, _c_int, _c_int, _vp]),
    "b2dl_channel_sum": (_c_int, [Act, _vp, _c_int, _c_int, _vp]),
    "b2dl_conv_fprop_bn_rows": (_c_int, [ctypes.POINTER(ConvArgs)]),
    "b2dl_bn_forward_partials": (_c_int, [_vp, _c_int, Act, _vp, _vp, ctypes.c_float, Act, _c_int, Act, _vp,
                                          _vp, _sz, _c_int, _vp]),
    "b2dl_bn_backward_partials": (_c_int, [_vp, _c_int, Act, Act, _vp, _vp, _vp, _vp, _c_int, Act, _c_int, _vp, _sz,
                                           _c_int, _vp]),
    "b2dl_cin_pad": (_c_int, [_c_int]),
    "b2dl_conv_fprop": (_c_int, [ctypes.POINTER(ConvArgs), _vp]),
    "b2dl_wgrad_workspace_size": (_sz, [ctypes.POINTER(WgradArgs)]),
    "b2dl_conv_wgrad": (_c_int, [ctypes.POINTER(WgradArgs), _vp]),
    "b2dl_wgrad_partials": (_c_int, [ctypes.POINTER(WgradArgs), ctypes.POINTER(_c_int), ctypes.POINTER(_c_int),
                                     ctypes.POINTER(_sz)]),
    "b2dl_reduce_segments": (_c_int, [_vp, _c_int, ctypes.c_int64, _vp, _vp]),
    "b2dl_pack_weights": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "b2dl_nchw_to_nhwc": (_c_int, [_vp, Act, _c_int, _vp]),
    "b2dl_bn_workspace_size": (ctypes.c_size_t, [_c_int]),
    "b2dl_bn_forward": (_c_int, [Act, _vp, _vp, ctypes.c_float, Act, _c_int, Act, _vp, _vp, ctypes.c_size_t,
                                 _c_int, _vp]),
    "b2dl_bn_backward": (_c_int, [Act, Act, _vp, _vp, _vp, _vp, _c_int, Act, _c_int, _vp, ctypes.c_size_t, _c_int,
                                  _vp]),
    "b2dl_bilinear_fwd": (_c_int, [Act, Act, _c_int, _c_int, _vp]),
    "b2dl_bilinear_workspace_size": (ctypes.c_size_t, [Act, _c_int]),
    "b2dl_bilinear_bwd": (_c_int, [Act, Act, _c_int, _c_int, Act, _c_int, _vp, ctypes.c_size_t, _vp]),
    "b2dl_f32_conv_fprop": (_c_int, [ctypes.POINTER(ConvArgs), _vp]),
    "b2dl_f32_wgrad_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(WgradArgs)]),
    "b2dl_f32_conv_wgrad": (_c_int, [ctypes.POINTER(WgradArgs), _vp]),
    "b2dl_f32_avgpool_fwd": (_c_int, [Act, Act, _c_int, _vp]),
    "b2dl_f32_avgpool_bwd": (_c_int, [Act, Act, _c_int, _c_int, Act, _vp]),
    "b2dl_f32_upsample_fwd": (_c_int, [Act, Act, _c_int, _vp]),
    "b2dl_f32_upsample_bwd": (_c_int, [Act, Act, _c_int, _c_int, Act, _vp]),
    "b2dl_f32_add": (_c_int, [Act, Act, _c_int, Act, _vp]),
    "b2dl_head_backward_parts": (_c_int, []),
    "b2dl_head_backward": (_c_int, [Act, _vp, Act, Act, _c_int, _c_int, _vp, _vp, _vp]),
    "b2dl_pack_upsampled_dgrad": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "b2dl_pack_upsampled_fprop": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "b2dl_upsampled_fprop_taps": (_c_int, [_c_int, _c_int]),
    "b2dl_upsampled_wgrad_sums": (_c_int, [Act, _c_int, _c_int, _vp, _vp]),
    "b2dl_upsampled_wgrad_reduce": (_c_int, [_vp, _c_int, _c_int, ctypes.c_size_t, _c_int, _c_int, _c_int, _vp, _vp,
                                             _vp]),
    "b2dl_nchw_to_nhwc_halo": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _vp]),
    "b2dl_nhwc_to_nchw": (_c_int, [Act, _c_int, _vp, _vp]),
    "b2dl_avgpool_fwd": (_c_int, [Act, Act, _c_int, _vp]),
    "b2dl_avgpool_bwd": (_c_int, [Act, Act, _c_int, _c_int, Act, _vp]),
    "b2dl_upsample_fwd": (_c_int, [Act, Act, _c_int, _vp]),
    "b2dl_upsample_bwd": (_c_int, [Act, Act, _c_int, _c_int, Act, _vp]),
    "b2dl_add": (_c_int, [Act, Act, _c_int, Act, _vp]),
    "b2dl_relu_mask": (_c_int, [Act, Act, _vp]),
    "b2dl_dgrad_1x1_small": (_c_int, [Act, _vp, Act, _c_int, Act, _vp]),
    "b2dl_bias_grad": (_c_int, [Act, _vp, _c_int, _vp, _sz, _vp]),
    "b2dl_bias_grad_workspace_size": (_sz, [Act]),
    "b2dl_wce": (_c_int, [Act, _vp, _vp, _c_int, _vp, _vp, Act, _c_int, ctypes.c_float, _vp, _vp, _vp, _sz, _vp]),
    "b2dl_wce_workspace_size": (_sz, [_c_int] * 4),
    "b2dl_larc_workspace_size": (_sz, [ctypes.c_int64, _c_int]),
    "b2dl_larc_update": (_c_int, [ctypes.POINTER(LarcArgs), _vp]),
    "b2dl_version": (ctypes.c_char_p, []),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def _load(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_1810_01993_b200._build` "
            "(this package has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB_F16_PATH = os.path.join(HERE, "libb2dl_f16.so")
_LIBS = {"bf16": _load()}
_current = threading.local()


def library(half: str = "bf16"):
    """The build whose 16-bit storage type is `half` ("bf16": libb2dl.so, "fp16": libb2dl_f16.so)."""
    if half not in _LIBS:
        if half != "fp16":
            raise ValueError(f"no {half!r} build")
        _LIBS[half] = _load(LIB_F16_PATH)
    return _LIBS[half]


class _Dispatch:
    """`LIB`: the bf16 build, or inside `use(\"fp16\")` the fp16 build (same symbols)."""

    def __getattr__(self, name):
        return getattr(getattr(_current, "lib", None) or _LIBS["bf16"], name)


LIB = _Dispatch()


class use:
    """Context: route LIB calls of this thread to the build of the given 16-bit type (re-entrant)."""

    def __init__(self, half: str):
        self.lib = library(half) if half == "fp16" else _LIBS["bf16"]

    def __enter__(self):
        self.prev = getattr(_current, "lib", None)
        _current.lib = self.lib
        return self.lib

    def __exit__(self, *exc):
        _current.lib = self.prev


class B2DLError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    """Map a b2dl return code onto the reference's exception types."""
    if rc == B2DL_OK:
        return
    if rc == B2DL_E_NOT_IMPLEMENTED:
        raise NotImplementedError(f"{what}: execution kernels support stride 1 only")
    if rc in (B2DL_E_VALUE, B2DL_E_ALIGN):
        raise ValueError(f"{what}: invalid arguments (b2dl code {rc})")
    if rc == B2DL_E_NONFINITE:
        raise FloatingPointError(f"{what}: non-finite norm in LARC")
    raise B2DLError(f"{what}: CUDA error (b2dl code {rc})")
