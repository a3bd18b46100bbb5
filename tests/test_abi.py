"""The C ABI boundary (include/b2dl.h): every declared symbol is exported by libb2dl.so
with a ctypes binding, and the ctypes struct layouts equal the C ones (gcc sizeof/offsetof).
Also the host-side planner on CPU: fused ops, zero-copy concats, relu masks folded."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "b2dl.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"B2DL_API\s+[\w\s\*]+?\b(b2dl_\w+)\s*\(", src)))


def test_every_declared_symbol_is_bound_and_exported():
    from paper_1810_01993_b200 import _lib
    names = declared()
    assert len(names) >= 20
    assert sorted(_lib.EXPORTED_SYMBOLS) == names
    for n in names:
        assert hasattr(_lib.LIB, n), n
    assert _lib.LIB.b2dl_version().startswith(b"b2dl")
    # the fp16 build (libb2dl_f16.so) exports the same ABI, and _lib.use routes LIB to it
    f16 = _lib.library("fp16")
    for n in names:
        assert hasattr(f16, n), n
    with _lib.use("fp16") as lib:
        assert lib is f16 and _lib.LIB.b2dl_cin_pad is f16.b2dl_cin_pad
    assert _lib.LIB.b2dl_cin_pad is _lib.library("bf16").b2dl_cin_pad


def test_struct_layouts_match_c(tmp_path):
    from paper_1810_01993_b200 import _lib
    structs = {"b2dl_act": _lib.Act, "b2dl_conv_args": _lib.ConvArgs, "b2dl_wgrad_args": _lib.WgradArgs,
               "b2dl_larc_args": _lib.LarcArgs}
    fields = {"b2dl_conv_args": ["y", "bias", "mask", "block_n", "bn_partial", "bnb_stats", "bnb_partial"], "b2dl_wgrad_args": ["dw", "workspace", "splits"],
              "b2dl_larc_args": ["lr", "lr_out", "workspace_bytes", "mode"], "b2dl_act": ["c", "c_stride"]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HDR}"', "int main(void){"]
    for s in structs:
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f in fields[s]:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                           check=True).stdout.split("\n") if l)
    for s, cls in structs.items():
        assert int(out[s]) == ctypes.sizeof(cls), s
        for f in fields[s]:
            assert int(out[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_error_codes_map_to_reference_exceptions():
    from paper_1810_01993_b200._lib import B2DLError, check
    with pytest.raises(NotImplementedError):
        check(1, "x")
    with pytest.raises(ValueError):
        check(2, "x")
    with pytest.raises(FloatingPointError):
        check(5, "x")
    with pytest.raises(B2DLError):
        check(3, "x")
    check(0, "x")


@pytest.mark.parametrize("which", ["deeplab", "deeplab_small", "minidensenet"])
def test_plan_fuses_everything(which):
    from paper_1810_01993_b200 import models
    from paper_1810_01993_b200.engine import Plan
    cfg = {"deeplab": models.DeepLabConfig(), "deeplab_small": models.deeplab_small(),
           "minidensenet": models.NetConfig()}[which]
    g, p, head, loss = models.build(cfg, 0)
    shape = (2, 16, 64, 64) if which != "deeplab" else (2, 16, 1152, 768)
    pl = Plan(g, {k: v.shape for k, v in p.items()}, shape, loss, head)
    convs = [o for o in pl.ops if o.kind == "conv"]
    assert len(convs) == sum(nd.kind == "conv2d" for nd in g.nodes)   # one launch per conv
    assert not any(o.copy_ins for o in pl.ops if o.kind == "concat")   # all concats zero-copy
    assert pl.relu_passes == 0                                        # relu VJP folded
    assert all(o.kind != "add" for o in pl.ops)                       # residual adds fused
    # every live conv output has a gradient buffer; the data input has none
    assert "x" not in pl.live and all(o.out in pl.live for o in convs)
