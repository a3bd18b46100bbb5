"""Model objects with the reference's network surface (pkg/src/deskdl/model/net.py:44-174).

`MiniDenseNet` and `DeepLabV3Plus` expose .graph, .params, .param_order,
forward, forward_loss -> (loss, logits, tape), backward(tape) -> grads,
grads_as_named, predictions, state_dict / load_state, num_parameters — with
the same argument meaning and exceptions — and execute every step on the GPU
engine (engine.py).  Inputs may be NumPy arrays (reference-style, copied to the
device) or CUDA tensors.  Parameter and gradient dicts are NumPy in the
reference's OIHW layout; the engine keeps its own device copies (HWIO fp32
master + bf16 packed operands).
"""

from __future__ import annotations

import numpy as np
import torch

from . import models
from .engine import Engine
from .graph import ShapeError
from .models import DeepLabConfig, NetConfig


class NamedTensor:
    """Flat float32 gradient with a shape and a stable name (reference core.py:16-45)."""
    __slots__ = ("name", "shape", "data")

    def __init__(self, name, shape, data):
        if not name:
            raise ValueError("tensor name must be non-empty")
        shape = tuple(int(s) for s in shape)
        data = np.ascontiguousarray(data, dtype=np.float32).reshape(-1)
        if data.size != int(np.prod(shape)):
            raise ShapeError(f"{name}: data length {data.size} != prod{shape}")
        self.name, self.shape, self.data = name, shape, data

    @property
    def size(self):
        return self.data.size

    def reshaped(self):
        return self.data.reshape(self.shape)


class Tape:
    """Handle on the engine state of one forward pass (the reference's ops.Tape)."""

    def __init__(self, engine: Engine, step: int):
        self.engine, self.step = engine, step


def _dev(a, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class SegmentationNet:
    """Shared implementation: seeded graph + params, one GPU engine per input shape."""

    def __init__(self, cfg, seed: int = 0, precision: str = "bf16"):
        """precision: "bf16" (tensor-core path) or "fp32" (parity mode, b2dl.h group 3)."""
        self.cfg = cfg
        self.precision = precision
        self.graph, params, self.logits_name, self.loss_name = models.build(cfg, seed)
        self.param_order = list(params)
        self._params = params
        self._engines = {}
        self._active = None
        self._steps = 0

    # -- parameter state (NumPy OIHW, like the reference) -----------------------
    @property
    def params(self) -> dict:
        if self._active is not None:
            self._params = self._active.export_params()
        return self._params

    def state_dict(self) -> dict:
        return {k: v.copy() for k, v in self.params.items()}

    def load_state(self, state: dict) -> None:
        cur = self.params
        new = {}
        for name in self.param_order:
            if name not in state:
                raise KeyError(f"missing parameter {name!r}")
            v = np.asarray(state[name], dtype=np.float32)
            if v.shape != cur[name].shape:
                raise ShapeError(f"{name}: shape {v.shape} != {cur[name].shape}")
            new[name] = v.copy()
        self._params = new
        for eng in self._engines.values():
            eng.load_params(new)

    def num_parameters(self) -> int:
        return int(sum(v.size for v in self._params.values()))

    # -- execution -----------------------------------------------------------------
    def _check_batch(self, shape):
        d = self.cfg.downsample_factor
        if len(shape) != 4 or shape[1] != self.cfg.channels_in:
            raise ShapeError(f"batch {tuple(shape)} does not match [N,{self.cfg.channels_in},H,W]")
        if shape[2] % d or shape[3] % d:
            raise ShapeError(f"spatial extent {tuple(shape[2:])} not divisible by {d}")

    def engine(self, shape) -> Engine:
        shape = tuple(int(s) for s in shape)
        self._check_batch(shape)
        eng = self._engines.get(shape)
        if eng is None:
            params = self.params
            eng = Engine(self.graph, params, self.param_order, shape, self.loss_name, self.logits_name,
                         precision=self.precision)
            self._engines[shape] = eng
        elif self._active is not None and self._active is not eng:
            eng.load_params(self.params)
        self._active = eng
        return eng

    def _run(self, batch, labels, class_weights, params):
        if params is not None:
            self.load_state(params)
        eng = self.engine(tuple(batch.shape))
        if labels is None:
            labels = torch.zeros((batch.shape[0],) + tuple(batch.shape[2:]), dtype=torch.uint8)
        lab = np.asarray(labels) if not isinstance(labels, torch.Tensor) else labels
        if not isinstance(lab, torch.Tensor) and lab.size and (lab.min() < 0 or lab.max() >= self.cfg.classes):
            raise ValueError(f"labels outside [0, {self.cfg.classes})")
        eng.set_batch(_dev(batch, torch.float32), _dev(lab, torch.uint8))
        eng.set_class_weights(np.ones(self.cfg.classes) if class_weights is None else class_weights)
        eng.forward()
        if isinstance(lab, torch.Tensor) and int(eng.label_status.item()):   # device labels: kernel check
            raise ValueError(f"labels outside [0, {self.cfg.classes})")
        self._steps += 1
        return eng

    def forward(self, batch, params=None):
        """Logits [N, classes, H, W] (CUDA fp32)."""
        return self._run(batch, None, None, params).logits_nchw()

    def forward_loss(self, batch, labels, class_weights, params=None):
        """Returns (loss scalar, logits [N,C,H,W] CUDA fp32, tape for backward)."""
        w = np.asarray(class_weights, dtype=np.float32)
        if w.shape != (self.cfg.classes,) or np.any(w <= 0):
            raise ValueError("class weights must be a positive vector of length classes")
        eng = self._run(batch, labels, w, params)
        return float(eng.loss.item()), eng.logits_nchw(), Tape(eng, self._steps)

    def backward(self, tape: Tape) -> dict:
        tape.engine.backward()
        return tape.engine.export_grads()

    def grads_as_named(self, grads: dict) -> list:
        return [NamedTensor(n, self._params[n].shape, grads[n]) for n in self.param_order]

    def predictions(self, logits):
        if isinstance(logits, torch.Tensor):
            return torch.argmax(logits, dim=1)
        return np.argmax(logits, axis=1)


class MiniDenseNet(SegmentationNet):
    """The reference's FC-DenseNet / Tiramisu-style network (net.py:44-174)."""

    def __init__(self, cfg: NetConfig = NetConfig(), seed: int = 0, precision: str = "bf16"):
        super().__init__(cfg, seed, precision)


class DeepLabV3Plus(SegmentationNet):
    """DeepLabV3+ (OS8, ASPP 12/18/24, full-resolution decoder) of the headline benchmark."""

    def __init__(self, cfg: DeepLabConfig = DeepLabConfig(), seed: int = 0, precision: str = "bf16"):
        super().__init__(cfg, seed, precision)
