"""Build libdg (C ABI + sm_100a kernels) in-tree with nvcc.

The shared library lands in paper_2404_16648_b200/lib/libdg.so so it travels
with the repo snapshot to the GPU box (no JIT cache, no pip install).
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", "dg_host.cpp"), os.path.join(HERE, "csrc", "dg_kernels.cu"),
        os.path.join(HERE, "csrc", "dg_stage.cu"), os.path.join(HERE, "csrc", "dg_regrid.cpp"),
        os.path.join(HERE, "csrc", "dg_visc.cu"), os.path.join(HERE, "csrc", "dg_tracer.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", "dg_internal.h"), os.path.join(ROOT, "include", "dg.h")]
LIB = os.path.join(HERE, "lib", "libdg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libdg; `out`/`defines` build development variants (e.g. lib/libdg_exp.so, ["-DDG_EXP=1"])."""
    if force or out != LIB or needs_build():
        os.makedirs(os.path.dirname(out), exist_ok=True)
        cmd = [NVCC] + FLAGS + list(defines) + (["-Xptxas", "-v"] if verbose else []) + SRCS + ["-o", out + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force=True))
