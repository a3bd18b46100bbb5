"""SGD with momentum, LARC and lag-1 application (pkg/src/deskdl/optimizer.py), on the GPU.

Same names, fields, validation and semantics as the reference:
  larc_effective_lr  min(trust*|w|/(|g|+wd*|w|), lr); lr when |w| == 0 or the
                     denominator < eps; FloatingPointError on a non-finite norm
  sgd_step           m <- beta*m + g + wd*w ; w <- w - f32(lr_eff)*m   (in place)
  larc_sgd_step      LARC rate then sgd_step; returns the rate
  lagged_apply       lag 0: apply now; lag 1: apply the previous gradient
Per-tensor calls run the multi-tensor LARC kernel (b2dl_larc_update) on one
segment; the trainer calls it once for all tensors of the model.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import nhwc


@dataclass(frozen=True)
class OptimConfig:
    lr: float = 1.0
    momentum: float = 0.9
    trust: float = 0.02
    weight_decay: float = 0.0
    eps: float = 1e-8
    lag: int = 0

    def __post_init__(self):
        if self.lr <= 0 or self.trust <= 0:
            raise ValueError("lr and trust must be positive")
        if not 0 <= self.momentum < 1:
            raise ValueError("momentum must be in [0, 1)")
        if self.weight_decay < 0 or self.eps <= 0:
            raise ValueError("weight_decay must be >= 0 and eps > 0")
        if self.lag not in (0, 1):
            raise ValueError("only lag 0 and 1 are supported")


def _as_dev(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).cuda()


class LayerParam:
    """One tensor's weights + optimizer state on the device (reference optimizer.py:36-45)."""
    __slots__ = ("name", "w", "m", "g_prev", "_shape")

    def __init__(self, name: str, w):
        self.name = name
        self._shape = tuple(w.shape) if isinstance(w, torch.Tensor) else tuple(np.shape(w))
        self.w = _as_dev(w).reshape(-1).clone()
        self.m = torch.zeros_like(self.w)
        self.g_prev = None


_WS = None


def _run(param, g, cfg, mode, lr_given=None):
    global _WS
    if _WS is None:
        _WS = nhwc.Workspace("cuda")
    gd = _as_dev(g).reshape(-1)
    if gd.numel() != param.w.numel():
        raise ValueError(f"{param.name}: gradient shape {tuple(np.shape(g))} != {param._shape}")
    off = torch.tensor([0, param.w.numel()], dtype=torch.int64, device="cuda")
    lr_out = torch.empty(1, dtype=torch.float32, device="cuda")
    if lr_given is not None:
        lr_out.fill_(float(np.float32(lr_given)))
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    nhwc.larc_update(param.w, param.m, gd, off, cfg.lr, cfg.momentum, cfg.trust, cfg.weight_decay, cfg.eps,
                     1.0, lr_out, status, _WS, mode=mode)
    if int(status.item()):
        raise FloatingPointError("non-finite norm in LARC")
    return float(lr_out.item())


def larc_effective_lr(w, g, cfg: OptimConfig) -> float:
    p = LayerParam("w", w)
    return _run(p, g, cfg, mode=1)


def sgd_step(param: LayerParam, g, lr_eff: float, cfg: OptimConfig) -> None:
    _run(param, g, cfg, mode=2, lr_given=lr_eff)


def larc_sgd_step(param: LayerParam, g, cfg: OptimConfig) -> float:
    return _run(param, g, cfg, mode=0)


def lagged_apply(param: LayerParam, g_current, cfg: OptimConfig) -> bool:
    if cfg.lag == 0:
        larc_sgd_step(param, g_current, cfg)
        return True
    g = param.g_prev
    param.g_prev = _as_dev(g_current).reshape(-1).clone()
    if g is None:
        return False
    larc_sgd_step(param, g, cfg)
    return True
