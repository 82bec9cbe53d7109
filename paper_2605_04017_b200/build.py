"""Build libplt.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2605_04017_b200.build [--force]

Every .cu/.cpp under csrc/ is compiled with nvcc (-gencode arch=compute_100a,
code=sm_100a, -lineinfo, -O3) and linked into paper_2605_04017_b200/libplt.so with
the CUDA runtime linked statically (no dependency on the torch-bundled cudart).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libplt.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", *ARCH,
          "-I", os.path.join(HERE, "..", "include")]
SOURCES = ["lens.cpp", "map.cpp", "abi.cpp", "trace.cu", "splat.cu", "eval_map.cu"]
HEADERS = ["plt_internal.h", "host.h", "splat_dev.cuh", "trace_dev.cuh"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """Build libplt.so.  `defines`/`out` are for developer instrumentation builds only."""
    obj_dir, out_path = OBJ, OUT
    if defines:
        tag = "_".join(d.lower() for d in defines)
        obj_dir = os.path.join(HERE, "build_" + tag)
        out_path = out or os.path.join(HERE, "libplt_" + tag + ".so")
    os.makedirs(obj_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "plt.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            extra = ["-Xptxas", "-v"] if verbose and src.endswith(".cu") else []
            cmd = [NVCC, *COMMON, *extra, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
            subprocess.check_call(cmd)
    if force or _stale(out_path, objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out_path, *objs,
                               "-Xlinker", "--exclude-libs,ALL"])
    return out_path


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs))
