"""Build libb2dl.so in-tree with nvcc for sm_100a (no torch JIT cache).

`python -m paper_1810_01993_b200._build` or `__graft_entry__.build()`.
Object files go to build/; the shared library lands next to this file so the
gpurun snapshot carries it to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libb2dl.so")
BUILD = os.path.join(ROOT, "build", "b2dl")
# the same sources with IEEE fp16 as the 16-bit storage / MMA operand type (csrc/half.cuh)
OUT_F16 = os.path.join(HERE, "libb2dl_f16.so")
BUILD_F16 = os.path.join(ROOT, "build", "b2dl_f16")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["conv_tc.cu", "host.cu", "elementwise.cu", "loss.cu", "larc.cu", "fp32.cu", "norm.cu", "refconv.cu", "generic.cu"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I" + os.path.join(ROOT, "include"),
]


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "b2dl.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, verbose: bool, f16: bool = False) -> str:
    obj = os.path.join(BUILD_F16 if f16 else BUILD, src.replace(".cu", ".o"))
    cmd = [NVCC, *FLAGS, *(["-DB2DL_F16"] if f16 else []), "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def _link(objs, out):
    tmp = out + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link libb2dl.so (bf16) and libb2dl_f16.so (fp16
    storage); returns the bf16 library's path."""
    dep = _deps_mtime()
    todo = [(f16, out) for f16, out in ((False, OUT), (True, OUT_F16))
            if force or not os.path.exists(out) or os.path.getmtime(out) < dep]
    if not todo:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(BUILD_F16, exist_ok=True)
    jobs = [(src, f16) for f16, _ in todo for src in SOURCES]
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        objs = list(ex.map(lambda j: _compile(j[0], verbose, j[1]), jobs))
    for k, (f16, out) in enumerate(todo):
        _link(objs[k * len(SOURCES):(k + 1) * len(SOURCES)], out)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
