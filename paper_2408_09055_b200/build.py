"""Build libatlas_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2408_09055_b200.build [--force] [--verbose]

Sources: paper_2408_09055_b200/csrc/*.cu (nvcc) and *.cpp (nvcc as host
compiler driver); linked with -shared, cudart static.  Object files go to
build/ (git-ignored); the .so lands next to this file so it travels with the
repository snapshot to the GPU box.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libatlas_b200.so")
BUILD = os.path.join(ROOT, "build", "atlas")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include")]
CU_FLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "atlas.h")])


def _digest(path, flags):
    h = hashlib.sha1()
    for p in [path] + _headers():
        h.update(open(p, "rb").read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()[:16]


def _compile(src, verbose):
    flags = COMMON + (CU_FLAGS if src.endswith(".cu") else ["-x", "cu"] + CU_FLAGS
                      if False else COMMON[:0])
    if src.endswith(".cu"):
        flags = COMMON + CU_FLAGS
    else:
        flags = COMMON + ["-x", "c++"]
    obj = os.path.join(BUILD, os.path.basename(src) + "." + _digest(src, flags) + ".o")
    if os.path.exists(obj):
        return obj
    cmd = [NVCC] + flags + ["-c", src, "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    if force:
        for f in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(f)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if (not force and os.path.exists(OUT)
            and all(os.path.getmtime(o) <= os.path.getmtime(OUT) for o in objs)):
        return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
