"""CKP1 checkpoint files (reference model/checkpoint.py:18-56): our reader loads a file the
reference wrote, our writer reproduces it byte for byte, malformed files raise ValueError."""

import os
import struct

import numpy as np
import pytest

from paper_1810_01993_b200.checkpoint import load_checkpoint, save_checkpoint

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _ref_arrays():
    d = np.load(os.path.join(G, "ckp1_reference_arrays.npz"))
    names = list(d["names"])
    return {n: d[f"a{i}"] for i, n in enumerate(names)}


def test_reads_reference_written_file():
    got = load_checkpoint(os.path.join(G, "ckp1_reference.bin"))
    ref = _ref_arrays()
    assert list(got) == list(ref)
    for k in ref:   # (the format stores at least one dimension: a scalar comes back as shape (1,))
        r = np.ascontiguousarray(ref[k], dtype=np.float32)
        assert got[k].dtype == np.float32 and got[k].shape == r.shape
        assert got[k].tobytes() == r.tobytes()


def test_writer_is_byte_identical_to_reference(tmp_path):
    p = tmp_path / "ours.ckpt"
    save_checkpoint(str(p), _ref_arrays())
    assert p.read_bytes() == open(os.path.join(G, "ckp1_reference.bin"), "rb").read()


def test_malformed_files_raise(tmp_path):
    good = open(os.path.join(G, "ckp1_reference.bin"), "rb").read()
    cases = {"magic": b"XXXX" + good[4:], "version": good[:4] + struct.pack("<I", 2) + good[8:],
             "trailing": good + b"\0", "truncated": good[:-3], "header": good[:6]}
    for name, raw in cases.items():
        p = tmp_path / f"{name}.ckpt"
        p.write_bytes(raw)
        with pytest.raises(ValueError):
            load_checkpoint(str(p))
