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
SOURCES = ["capi.cu", "improve.cu", "population.cu", "pool.cu", "distance.cu", "similarity_tc.cu", "host_graph.cu", "plits.cu", "improve_ref.cu", "plits_ref.cu"]
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


def _compile(src: str, obj: str) -> subprocess.CompletedProcess:
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O3",
           "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc -c per translation unit (in parallel; only the sources newer than their object unless
    forced), then one shared-library link."""
    if not force and not needs_build():
        build_cli()
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "plse_b200.h"))
    newest_header = max(os.path.getmtime(h) for h in headers if os.path.exists(h))
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_header)
        jobs.append((src, obj, stale))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        results = {src: ex.submit(_compile, src, obj) for src, obj, stale in jobs if stale}
        log = []
        for src, fut in results.items():
            out = fut.result()
            if out.returncode != 0:
                raise RuntimeError("nvcc failed on " + src + ":\n" + out.stdout + out.stderr)
            log.append(out.stderr)
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *[obj for _, obj, _ in jobs]]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + " ".join(cmd) + "\n" + out.stdout + out.stderr)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        sys.stderr.write("".join(log))
    build_cli(force=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
