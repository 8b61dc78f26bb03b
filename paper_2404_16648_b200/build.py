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
        os.path.join(HERE, "csrc", "dg_stage.cu"), os.path.join(HERE, "csrc", "dg_stage_h4.cu"), os.path.join(HERE, "csrc", "dg_regrid.cpp"),
        os.path.join(HERE, "csrc", "dg_visc.cu"), os.path.join(HERE, "csrc", "dg_tracer.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", "dg_internal.h"), os.path.join(HERE, "csrc", "dg_device.cuh"), os.path.join(ROOT, "include", "dg.h")]
LIB = os.path.join(HERE, "lib", "libdg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177,1886"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libdg; `out`/`defines` build development variants (e.g. lib/libdg_exp.so, ["-DDG_EXP=1"]).

    Each source is compiled to its own object in parallel (nvcc -c; the stage kernels dominate),
    then linked into one shared library."""
    if force or out != LIB or needs_build():
        import concurrent.futures as cf
        import tempfile
        os.makedirs(os.path.dirname(out), exist_ok=True)
        tmp = tempfile.mkdtemp(prefix="libdg_")
        objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in SRCS]
        cflags = [f for f in FLAGS if f != "-shared"] + list(defines) + (["-Xptxas", "-v"] if verbose else [])

        def one(src_obj):
            subprocess.check_call([NVCC] + cflags + ["-c", src_obj[0], "-o", src_obj[1]])
        with cf.ThreadPoolExecutor(max_workers=len(SRCS)) as ex:
            list(ex.map(one, zip(SRCS, objs)))
        subprocess.check_call([NVCC] + ["-gencode", "arch=compute_100a,code=sm_100a", "-shared"] + objs
                              + ["-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
        for o in objs:
            os.remove(o)
        os.rmdir(tmp)
    return out


if __name__ == "__main__":
    print(build(force=True))
