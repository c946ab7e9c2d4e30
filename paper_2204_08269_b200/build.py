"""Build libjtfs.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun).

    python -m paper_2204_08269_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libjtfs.so")
SOURCES = ["plan.cpp", "kernels.cu", "kernels_tc.cu", "knn.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
    "-prec-sqrt=true", "-prec-div=true", "-ftz=false", "-cudart", "static",
    "-I" + os.path.join(ROOT, "include"),
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "jtfs.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile libjtfs.so (or, for A/B measurements of a compile-time variant, `lib` with
    extra -D `defines`; select it at run time with JTFS_LIB=<path>)."""
    if not force and not _stale(lib):
        return lib
    objs, procs = [], []
    tag = "" if lib == LIB else "." + os.path.basename(lib)
    for src in SOURCES:  # the translation units compile concurrently
        obj = os.path.join(CSRC, src + tag + ".o")
        cmd = [NVCC, *FLAGS, *("-D" + d for d in defines), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           *objs, "-o", lib + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    # python -m paper_2204_08269_b200.build [--force] [-DNAME=VALUE ... --lib PATH]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = sys.argv[sys.argv.index("--lib") + 1] if "--lib" in sys.argv else LIB
    print(build(force="--force" in sys.argv, verbose=True, defines=defs, lib=out))
