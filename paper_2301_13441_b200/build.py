"""Build ``libcmlb.so`` (sm_100a) in-tree with nvcc; no torch dependency.

    python -m paper_2301_13441_b200.build          # or __graft_entry__.build()

The library is loaded with ctypes (``_native.py``); the built ``.so`` stays
inside the package directory so it travels to the GPU box with the repo.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcmlb.so")
SOURCES = ["capi.cu", "forest.cu", "linear.cu", "scaler.cu", "svm.cu", "cols.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("common.cuh", "sm100.cuh")] + [os.path.join(ROOT, "include", "cmlb.h")]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(deps):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include")] + ARCH
    if verbose:
        flags += ["-Xptxas", "-v"]
    objs = []
    procs = []
    headers = deps[len(srcs):]
    for s in srcs:
        obj = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(obj)
        # per-object rebuild: a source is recompiled when it or a header is newer
        if not force and not verbose and os.path.exists(obj) and os.path.getmtime(obj) >= _newest([s] + headers):
            continue
        procs.append((s, subprocess.Popen([NVCC, *flags, "-c", s, "-o", obj],
                                          stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    logs = []
    for s, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{out}")
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"], check=True)
    os.replace(tmp, LIB)
    if verbose:
        sys.stdout.write("".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
