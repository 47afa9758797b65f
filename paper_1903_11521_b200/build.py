"""Build libydg.so in-tree (sm_100a), with parallel nvcc/g++ jobs and a stamp cache.

    python -m paper_1903_11521_b200.build [--force]

The generated sources (csrc/generated/) are committed; regenerate them with
``python -m paper_1903_11521_b200.gen.tables`` (slow, mpmath) and
``python -m paper_1903_11521_b200.gen.kernels``.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.environ.get("YDG_BUILD_DIR") or os.path.join(HERE, "_build")
LIB = os.environ.get("YDG_LIB") or os.path.join(HERE, "libydg.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
                  "-I", CSRC, "--expt-relaxed-constexpr"] + os.environ.get("YDG_NVFLAGS", "").split()
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-fopenmp", "-I", CSRC, "-I", os.path.join(CUDA, "include")]
# -D defines of YDG_NVFLAGS apply to the host translation units as well (shared headers)
CXXFLAGS += [f for f in os.environ.get("YDG_NVFLAGS", "").split() if f.startswith("-D")]


def sources():
    cu = [os.path.join(CSRC, f) for f in ("kernels.cu", "halo.cu", "generic.cu", "visco.cu", "lina.cu")]
    cu += [os.path.join(CSRC, "generated", f"kernels_N{n}.cu") for n in range(1, 7)]
    cpp = [os.path.join(CSRC, f) for f in ("setup.cpp", "api.cpp")]
    return cu, cpp


def _deps_hash(src):
    h = hashlib.sha256()
    for root in (CSRC, os.path.join(HERE, "..", "include")):
        for dp, _, fs in os.walk(root):
            for f in sorted(fs):
                if f.endswith((".h", ".cuh")):
                    with open(os.path.join(dp, f), "rb") as fh:
                        h.update(fh.read())
    with open(src, "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(NVFLAGS + CXXFLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src, force):
    name = os.path.basename(src)
    obj = os.path.join(BUILD, name + ".o")
    stamp = obj + ".stamp"
    key = _deps_hash(src)
    if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == key:
        return obj, False
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as fh:
        fh.write(key)
    return obj, True


def build(force=False, verbose=True):
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp = sources()
    srcs = cu + cpp
    # biggest translation units first
    srcs.sort(key=lambda s: -os.path.getsize(s))
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    rebuilt = any(c for _, c in results) or not os.path.exists(LIB)
    if rebuilt:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-Xcompiler", "-fopenmp", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(("built " if rebuilt else "up to date ") + LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
