"""Build the in-tree CUDA library libfsyrk_b200.so for sm_100a.

Explicit nvcc, no JIT cache: the .so lands next to this file so it travels
to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfsyrk_b200.so")
SOURCES = ["driver.cu", "tc_modmm.cu", "elementwise.cu", "host_io.cu"]
HEADERS = ["host_io.h", "modp.cuh", "sm100.cuh", "tc_modmm.h", "elementwise.cuh", "field_host.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "fsyrk_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True, out: str = LIB, defines=()) -> str:
    """Compile the library; `out` / `defines` (-D flags) build tuning variants for experiments
    (loaded with FSYRK_B200_LIB=<path>), the default is the shipped library."""
    if out == LIB and not defines and not force and not needs_build():
        return LIB
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           *[f"-D{d}" for d in defines], "-o", out] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    # python -m paper_2001_04109_b200.build [--force] [--out PATH -DNAME=VAL ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB
    build(force="--force" in argv, out=out, defines=[a[2:] for a in argv if a.startswith("-D")])
