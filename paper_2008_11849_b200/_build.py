"""Build libsparsert.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2008_11849_b200._build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsparsert.so")
SOURCES = ["inspector.cpp", "capi.cpp", "kernels.cu", "jit.cpp", "tune.cu"]
HEADERS = [os.path.join(CSRC, "plan.h"), os.path.join(ROOT, "include", "sparsert.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-cudart", "static",
         "--expt-relaxed-constexpr", "-Xptxas", "-v,-warn-spills"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + HEADERS + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libsparsert.so (or, for A/B experiments, a variant with extra -D defines
    into `out`)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    objs = []
    tmpdir = os.path.join(PKG, "build" if out is None else "build_variant")
    os.makedirs(tmpdir, exist_ok=True)
    procs = []
    for s in SOURCES:
        obj = os.path.join(tmpdir, s + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, s), "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    logs = []
    for s, pr in procs:
        out, _ = pr.communicate()
        logs.append(out.decode(errors="replace"))
        if pr.returncode != 0:
            sys.stderr.write(out.decode(errors="replace"))
            raise RuntimeError(f"nvcc failed on {s}")
    if verbose:
        sys.stderr.write("\n".join(logs))
    with open(os.path.join(tmpdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
                           "-L/usr/local/cuda/lib64", "-lnvptxcompiler_static", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
