"""Seeded synthetic climate scenes: the training step's input source.

`make_scene` restates pkg/src/deskdl/model/synthetic.py:140-173 draw for draw
(same generator calls in the same order), so a seed yields the reference's
exact field and label bytes (pinned by tests/golden/scenes.npz).  It is host
NumPy, like the reference's; the GPU step only consumes its tensors.
`scene_rng(seed, step, j)` is the trainer's stream (trainer.py:70-79): sample j
of step t comes from default_rng((seed, 0, t, j)) whatever the rank split.

`device_scene_pool` builds a pool of statistically similar tiles directly on
the GPU (noise + coarse field + painted blob / streak labels) for throughput
runs, where make_scene's 0.84 s per full-size tile would dominate.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TRAIN_NS = 0


@dataclass(frozen=True)
class SceneConfig:
    """Scene shape and class mix (reference synthetic.py:31-65)."""
    count: int = 1000
    channels: int = 16
    height: int = 64
    width: int = 48
    frequencies: tuple = (0.982, 0.017, 0.001)
    noise_sigma: float = 1.0
    amplitude: float = 3.0
    streak_channels: tuple = (0, 1, 2, 3)
    blob_channels: tuple = (4, 5, 6, 7)

    def __post_init__(self):
        if min(self.count, self.channels, self.height, self.width) < 1:
            raise ValueError("count, channels, height and width must be positive")
        f = self.frequencies
        if len(f) != 3 or any(v < 0 for v in f) or abs(sum(f) - 1.0) > 1e-9:
            raise ValueError(f"frequencies must be 3 non-negatives summing to 1: {f}")
        sig = self.streak_channels + self.blob_channels
        if sig and max(sig) >= self.channels:
            raise ValueError("signal channel index out of range")


def scene_rng(seed: int, step: int, j: int):
    return np.random.default_rng((seed, TRAIN_NS, step, j))


def _round_prob(rng, x: float) -> int:
    lo = math.floor(x)
    return lo + int(rng.random() < x - lo)


def _blob(rng, lab, count, value):
    if count == 0:
        return
    h, w = lab.shape
    cy, cx = rng.uniform(0, h), rng.uniform(0, w)
    yy, xx = np.mgrid[0:h, 0:w]
    key = (yy - cy) ** 2 + (xx - cx) ** 2 + rng.uniform(0, 2.0, size=(h, w))
    order = np.argsort(key.reshape(-1), kind="stable")
    flat = lab.reshape(-1)
    pick = order[flat[order] == 0][:count]
    if pick.size < count:
        raise ValueError("not enough free pixels for the blob")
    flat[pick] = value


def _stroke(rng, h, w):
    y0, x0 = rng.uniform(0, h), rng.uniform(0, w)
    ang = rng.uniform(0, math.pi)
    sy, sx = math.sin(ang), math.cos(ang)
    n = int(rng.uniform(0.3, 1.0) * max(h, w))
    thick = rng.integers(1, 3)
    pts = []
    for t in range(n):
        r0, c = int(y0 + t * sy), int(x0 + t * sx)
        for k in range(thick):
            r = r0 + k
            if 0 <= r < h and 0 <= c < w:
                pts.append((r, c))
    return pts


def _streaks(rng, lab, count, value):
    left, idle = count, 0
    while left > 0:
        placed = 0
        for r, c in _stroke(rng, *lab.shape):
            if lab[r, c] == 0:
                lab[r, c] = value
                placed += 1
                left -= 1
                if left == 0:
                    break
        idle = idle + 1 if placed == 0 else 0
        if idle > 1000:
            raise ValueError("could not place requested streak pixels")


def make_scene(cfg: SceneConfig, rng):
    """Returns (field [C,H,W] float32, labels [H,W] uint8)."""
    h, w, c = cfg.height, cfg.width, cfg.channels
    hw = h * w
    n_blob = _round_prob(rng, cfg.frequencies[2] * hw)
    n_streak = _round_prob(rng, cfg.frequencies[1] * hw)
    if n_blob + n_streak > hw:
        raise ValueError("requested class pixels exceed the image")
    lab = np.zeros((h, w), np.uint8)
    _blob(rng, lab, n_blob, 2)
    _streaks(rng, lab, n_streak, 1)
    field = rng.standard_normal((c, h, w)).astype(np.float32) * cfg.noise_sigma
    coarse = rng.standard_normal((h // 8 + 1, w // 8 + 1)).astype(np.float32)
    field += coarse.repeat(8, 0).repeat(8, 1)[:h, :w] * cfg.noise_sigma
    amp = np.float32(cfg.amplitude)
    for ch in cfg.streak_channels:
        field[ch][lab == 1] += amp
    for ch in cfg.blob_channels:
        field[ch][lab == 2] += amp
    signal = set(cfg.streak_channels) | set(cfg.blob_channels)
    fake = np.zeros((h, w), np.uint8)
    for ch in range(c):
        if ch in signal:
            continue
        fake[:] = 0
        _streaks(rng, fake, min(n_streak + n_blob, hw), 1)
        field[ch][fake == 1] += amp
    return field, lab


def class_counts(labels, classes: int = 3):
    return np.bincount(np.asarray(labels).reshape(-1), minlength=classes)


def generated_batch(cfg: SceneConfig, seed: int, step: int, rank: int, local_batch: int):
    """Rank's slice of the global batch of step t (reference trainer.py:70-79)."""
    fields, labels = [], []
    for j in range(rank * local_batch, (rank + 1) * local_batch):
        f, lab = make_scene(cfg, scene_rng(seed, step, j))
        fields.append(f)
        labels.append(lab)
    return np.stack(fields), np.stack(labels)


def device_scene_pool(count: int, cfg: SceneConfig, seed: int, device="cuda"):
    """`count` tiles generated on the GPU: (fields [K,C,H,W] fp32, labels [K,H,W] uint8).

    Same recipe as make_scene (N(0, sigma) noise, 8x8-block coarse field,
    +amplitude on signal channels, one compact blob of class 2 and thin
    streaks of class 1 at the configured frequencies) but not the same bytes.
    """
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    k, c, h, w = count, cfg.channels, cfg.height, cfg.width
    f = torch.randn(k, c, h, w, generator=g, device=device) * cfg.noise_sigma
    coarse = torch.randn(k, 1, h // 8 + 1, w // 8 + 1, generator=g, device=device)
    f += coarse.repeat_interleave(8, 2).repeat_interleave(8, 3)[..., :h, :w] * cfg.noise_sigma
    yy = torch.arange(h, device=device).view(1, h, 1).float()
    xx = torch.arange(w, device=device).view(1, 1, w).float()
    lab = torch.zeros(k, h, w, dtype=torch.uint8, device=device)
    # streaks: thin oriented bands whose width is set to hit the class-1 budget
    ang = torch.rand(k, 1, 1, generator=g, device=device) * math.pi
    cy = torch.rand(k, 1, 1, generator=g, device=device) * h
    cx = torch.rand(k, 1, 1, generator=g, device=device) * w
    dist = ((yy - cy) * torch.cos(ang) - (xx - cx) * torch.sin(ang)).abs()
    half = cfg.frequencies[1] * h * w / (2.0 * max(h, w))
    lab[dist < half] = 1
    # blob: disc with the class-2 pixel budget
    by = torch.rand(k, 1, 1, generator=g, device=device) * h
    bx = torch.rand(k, 1, 1, generator=g, device=device) * w
    rad = math.sqrt(cfg.frequencies[2] * h * w / math.pi)
    lab[((yy - by) ** 2 + (xx - bx) ** 2) < rad * rad] = 2
    amp = cfg.amplitude
    for ch in cfg.streak_channels:
        f[:, ch] += amp * (lab == 1)
    for ch in cfg.blob_channels:
        f[:, ch] += amp * (lab == 2)
    return f.contiguous(), lab.contiguous()
