"""In-tree build of the sm_100a library (libplse_b200.so) with nvcc.

The .so lands next to this file so that it travels with the repo snapshot to
the GPU box (git-ignored, not gpurun-ignored).  No JIT cache, no torch
extension machinery: the C ABI has no torch types.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libplse_b200.so")
SOURCES = ["capi.cu", "improve.cu", "improve_hw.cu", "population.cu", "distance.cu", "similarity_tc.cu", "host_graph.cu", "plits.cu", "improve_ref.cu", "plits_ref.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "plse_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


CLI = os.path.join(HERE, "plse_b200")
CLI_SRC = os.path.join(ROOT, "tools", "plse_b200.cpp")
CXX = os.environ.get("PLSE_CXX", "g++")


def build_cli(force: bool = False) -> str:
    """tools/plse_b200.cpp -> plse_b200 (the C++ front-end over include/plse_b200.hpp), linked to the
    in-tree library with an $ORIGIN rpath so it travels with the snapshot."""
    deps = [CLI_SRC, LIB, os.path.join(ROOT, "include", "plse_b200.hpp"), os.path.join(ROOT, "include", "plse_b200.h")]
    if not force and os.path.exists(CLI) and all(os.path.getmtime(d) <= os.path.getmtime(CLI) for d in deps
                                                  if os.path.exists(d)):
        return CLI
    cmd = [CXX, "-O2", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI + ".tmp",
           "-L" + HERE, "-lplse_b200", "-Wl,-rpath,$ORIGIN", "-pthread"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("c++ failed:\n" + " ".join(cmd) + "\n" + out.stdout + out.stderr)
    os.replace(CLI + ".tmp", CLI)
    return CLI


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        build_cli()
        return LIB
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-I" + os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *sources()]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out.stdout + out.stderr)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        sys.stderr.write(out.stderr)
    build_cli(force=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
