"""Build libtdpipe.so (the C-ABI library) in-tree with nvcc for sm_100a.

Usage: python -m paper_2506_10470_b200.build [-j N] [--force]
Objects go to build/; the shared library lands next to this file so that it
travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libtdpipe.so")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    """nccl.h from the torch-bundled nvidia-nccl wheel (types only; the library
    is dlopen'ed at run time, so nothing links against libnccl)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for loc in (spec.submodule_search_locations or []):
            inc = os.path.join(loc, "nccl", "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return None


NCCL_INC = _nccl_include()
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + (["-I" + NCCL_INC] if NCCL_INC else ["-DTDP_NO_NCCL"])
CU_FLAGS = ARCH + ["-Xptxas", "-v", "--expt-relaxed-constexpr", "-diag-suppress", "177"]
# extra -D flags for A/B builds of compile-time tuning constants (measurement only)
COMMON += os.environ.get("TDP_NVCC_DEFINES", "").split()


def sources():
    out = []
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(d, f))
    return sorted(out)


def headers():
    hs = [os.path.join(ROOT, "include", "tdpipe.h")]
    for d, _, files in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in files if f.endswith((".h", ".cuh"))]
    return hs


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def _compile(src, force, hdr_mtime):
    obj = _obj(src)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, ""
    flags = COMMON + (CU_FLAGS if src.endswith(".cu") else ["-x", "cu"] + ARCH)
    cmd = [NVCC] + flags + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(jobs: int = 8, force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in headers())
    srcs = sources()
    logs = {}
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = {ex.submit(_compile, s, force, hdr_mtime): s for s in srcs}
        objs = []
        for f in cf.as_completed(futs):
            o, log = f.result()
            objs.append(o)
            logs[futs[f]] = log
    objs = sorted(objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        for s, l in logs.items():
            if l.strip():
                print(f"== {os.path.relpath(s, ROOT)}\n{l}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.j, a.force, a.v))
