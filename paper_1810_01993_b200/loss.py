"""Class weighting and the weighted softmax cross-entropy (pkg/src/deskdl/model/loss.py).

`weighted_ce_loss` keeps the reference signature and validation (loss.py:47-74)
and runs the fused cross-entropy kernel (b2dl_wce): exact per-sample class
histograms, per-sample weight normalisation, loss and fp32 dlogits in one pass.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import nhwc


@dataclass(frozen=True)
class ClassWeights:
    """Inverse-square-root class weights from label frequencies (loss.py:18-40)."""
    frequencies: tuple

    def __post_init__(self):
        f = self.frequencies
        if len(f) < 2 or any(v <= 0 for v in f):
            raise ValueError(f"frequencies must be positive: {f}")
        if abs(sum(f) - 1.0) > 1e-6:
            raise ValueError(f"frequencies must sum to 1, got {sum(f)}")

    @property
    def weights(self) -> np.ndarray:
        return 1.0 / np.sqrt(np.asarray(self.frequencies, dtype=np.float64))

    def vector(self, dtype=np.float32) -> np.ndarray:
        return self.weights.astype(dtype)

    @classmethod
    def uniform(cls, classes: int) -> "ClassWeights":
        return cls(tuple(1.0 / classes for _ in range(classes)))


def uniform_weights(classes: int, dtype=np.float32) -> np.ndarray:
    return np.ones(classes, dtype=dtype)


def expected_uniform_loss(classes: int) -> float:
    return math.log(classes)


_WS = None


def weighted_ce_loss(logits, labels, weights, return_device=False):
    """(loss, dlogits [N,C,H,W]) for logits [N,C,H,W] and integer labels [N,H,W]."""
    global _WS
    lg = logits if isinstance(logits, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(logits))
    c = lg.shape[1]
    w = np.asarray(weights, dtype=np.float32)
    if w.shape != (c,):
        raise ValueError(f"weights shape {w.shape} does not match {c} classes")
    if np.any(w <= 0):
        raise ValueError("class weights must be positive")
    lab = labels if isinstance(labels, torch.Tensor) else torch.from_numpy(np.asarray(labels))
    if tuple(lab.shape) != (lg.shape[0],) + tuple(lg.shape[2:]):
        raise ValueError(f"labels shape {tuple(lab.shape)} does not match logits {tuple(lg.shape)}")
    if lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= c):
        raise ValueError(f"labels outside [0, {c})")
    if lg.dim() != 4:
        raise ValueError("logits must be [N, C, H, W]")
    n, _, h, wd = lg.shape
    dev = torch.device("cuda")
    lg32 = lg.to(device=dev, dtype=torch.float32).contiguous()
    z = torch.empty((n, h, wd, c), dtype=torch.float32, device=dev)
    nhwc.nchw_to_nhwc(lg32, nhwc.View(z), dst_f32=True)
    dl = torch.empty((n, h, wd, c), dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    counts = torch.empty(n * c, dtype=torch.int32, device=dev)
    if _WS is None:
        _WS = nhwc.Workspace(dev)
    nhwc.wce(nhwc.View(z), lab.to(device=dev, dtype=torch.uint8).contiguous().reshape(-1),
             torch.from_numpy(w).to(dev), loss, counts, nhwc.View(dl), None, _WS, dlogits_f32=True)
    out = torch.empty((n, c, h, wd), dtype=torch.float32, device=dev)
    nhwc.nhwc_to_nchw(nhwc.View(dl), out, src_f32=True)
    if return_device:
        return loss, out
    return float(loss.item()), out.cpu().numpy()
