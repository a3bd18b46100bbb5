"""CKP1 checkpoint files (reference model/checkpoint.py:18-56) and training-state resume.

Format, all little-endian: magic b"CKP1" (u32 0x31504B43), version u32 = 1, count u32, then per
tensor: u16 name length + UTF-8 name, u8 ndim, ndim x u32 dims, float32 payload.  Files written
here load with the reference's `load_checkpoint` and vice versa (tests/golden/ckp1_reference.bin).

`save_train_state` / `load_train_state` extend a parameter checkpoint with everything a resumed
run needs: per-tensor momentum ("momentum:<name>"), the reduced gradient a lag-1
run still has to apply ("lag_grad:<name>", stored as the rank MEAN, so a run may resume on a
different number of ranks), and counters ("meta:steps" as two exact 16-bit halves [lo, hi],
"meta:have_prev", "meta:world" = the writer's rank count) -- still a plain CKP1 file, so the
reference's reader sees the weights plus extra named tensors.
"""

from __future__ import annotations

import struct

import numpy as np

CKPT_MAGIC = 0x31504B43
CKPT_VERSION = 1


def save_checkpoint(path: str, params: dict) -> None:
    """Write named float32 tensors in insertion order."""
    out = [struct.pack("<III", CKPT_MAGIC, CKPT_VERSION, len(params))]
    for name, value in params.items():
        a = np.ascontiguousarray(value, dtype="<f4")
        nb = name.encode("utf-8")
        if len(nb) > 0xFFFF or a.ndim > 0xFF:
            raise ValueError(f"{name}: name or rank too large for CKP1")
        out.append(struct.pack("<H", len(nb)) + nb + struct.pack("<B", a.ndim)
                   + struct.pack(f"<{a.ndim}I", *a.shape) + a.tobytes())
    with open(path, "wb") as fh:
        fh.write(b"".join(out))


def load_checkpoint(path: str) -> dict:
    """Read a CKP1 file into {name: float32 ndarray}; ValueError on a malformed file."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 12:
        raise ValueError(f"{path}: truncated checkpoint header")
    magic, version, count = struct.unpack_from("<III", raw, 0)
    if magic != CKPT_MAGIC:
        raise ValueError(f"{path}: bad checkpoint magic {magic:#x}")
    if version != CKPT_VERSION:
        raise ValueError(f"{path}: unsupported checkpoint version {version}")
    pos, out = 12, {}
    try:
        for _ in range(count):
            (ln,) = struct.unpack_from("<H", raw, pos)
            name = raw[pos + 2:pos + 2 + ln].decode("utf-8")
            pos += 2 + ln
            (nd,) = struct.unpack_from("<B", raw, pos)
            dims = struct.unpack_from(f"<{nd}I", raw, pos + 1)
            pos += 1 + 4 * nd
            cnt = int(np.prod(dims)) if nd else 1
            out[name] = np.frombuffer(raw, dtype="<f4", count=cnt, offset=pos).reshape(dims).copy()
            pos += 4 * cnt
    except struct.error as e:
        raise ValueError(f"{path}: truncated checkpoint ({e})") from None
    if pos != len(raw):
        raise ValueError(f"{path}: {len(raw) - pos} trailing bytes")
    return out


def save_train_state(path: str, trainer) -> None:
    """Weights, momentum, pending lag-1 gradient and counters of a DataParallelTrainer."""
    st = trainer.export_state()
    tensors = dict(st["params"])
    tensors.update({f"momentum:{k}": v for k, v in st["momentum"].items()})
    if st["lag_grad"] is not None:
        tensors.update({f"lag_grad:{k}": v for k, v in st["lag_grad"].items()})
    steps = int(st["steps"])
    if not 0 <= steps < 2 ** 32:
        raise ValueError(f"step count {steps} out of range")
    tensors["meta:steps"] = np.array([steps & 0xFFFF, steps >> 16], dtype=np.float32)   # exact halves
    tensors["meta:have_prev"] = np.array([1.0 if st["have_prev"] else 0.0], dtype=np.float32)
    tensors["meta:world"] = np.array([st.get("world", 1)], dtype=np.float32)
    save_checkpoint(path, tensors)


def load_train_state(path: str, trainer) -> None:
    """Restore a state written by save_train_state into a trainer of the same model / lag."""
    t = load_checkpoint(path)
    order = trainer.net.param_order
    missing = [k for k in order if k not in t or f"momentum:{k}" not in t]
    if missing:
        raise KeyError(f"{path}: missing tensors for {missing[:3]}")
    have_prev = bool(t.get("meta:have_prev", np.zeros(1))[0])
    lag = {k: t[f"lag_grad:{k}"] for k in order} if have_prev else None
    ms = t["meta:steps"]
    steps = int(ms[0]) + (int(ms[1]) << 16 if ms.size > 1 else 0)
    trainer.import_state({"params": {k: t[k] for k in order}, "momentum": {k: t[f"momentum:{k}"] for k in order},
                          "lag_grad": lag, "steps": steps, "have_prev": have_prev})
