"""Build liblabuf.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2605_19049_b200.build [--force]

The shared library exports exactly the C ABI of include/la.h.  The CUDA
runtime is linked statically; NCCL is dlopen'ed at run time (csrc/tp.cpp).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblabuf.so")

CU_SOURCES = ["chunk.cu", "chunk_f32_direct.cu", "chunk_f32_state.cu", "chunk_bf16_direct.cu",
              "chunk_bf16_state.cu", "chunk_bf16h_direct.cu", "chunk_bf16h_state.cu", "fold.cu", "fold_ut.cu", "recurrent.cu"]
CPP_SOURCES = ["la.cpp", "tp.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES]


def _deps():
    out = _sources() + [os.path.join(CSRC, f) for f in ("device.cuh", "internal.h", "chunk.cuh")]
    out.append(os.path.join(ROOT, "include", "la.h"))
    return out


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden",
             f"-I{os.path.join(ROOT, 'include')}",
             "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"]
    if verbose:
        flags.append("-Xptxas=-v")
    # one object per source, compiled in parallel (no relocatable device code:
    # every kernel is launched from its own translation unit), then one link
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    headers = [p for p in _deps() if not p.endswith((".cu", ".cpp"))]
    for src in _sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        # incremental: an object is rebuilt when it is older than its source
        # or any shared header (always with force)
        if not force and os.path.exists(obj) and \
                os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in [src, *headers]):
            continue
        procs.append((src, subprocess.Popen([nvcc, *flags, "-c", "-o", obj, src])))
    bad = [src for src, p in procs if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, f"nvcc {' '.join(bad)}")
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl", "-lpthread"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
