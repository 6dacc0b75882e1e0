"""Build libfea.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2204_03893_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfea.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["fea_kernels.cu", "fea_kernels5.cu", "fea_kernels6.cu", "fea_kernels_t.cu", "fea_kernels_t5.cu", "fea_kernels_x.cu", "fea_host.cpp"]
DEPS = SOURCES + ["fea_internal.h", "fea_device.cuh"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    srcs = [os.path.join(CSRC, s) for s in DEPS] + [os.path.join(ROOT, "include", "fea.h"), __file__]
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    inc += os.environ.get("FEA_BUILD_DEFS", "").split()  # experiment switches, e.g. "-DFEA5_MMA=0"

    hdrs = [os.path.join(CSRC, h) for h in ("fea_internal.h", "fea_device.cuh")] + [os.path.join(ROOT, "include", "fea.h")]
    defs_key = os.environ.get("FEA_BUILD_DEFS", "") + ("|diag" if os.environ.get("FEA_BUILD_DIAG") else "")
    stamp = os.path.join(OBJ, "defs.txt")
    same_defs = os.path.exists(stamp) and open(stamp).read() == defs_key

    def compile_one(src):
        obj = os.path.join(OBJ, src + ".o")
        deps = [os.path.join(CSRC, src), __file__] + hdrs
        if not force and same_defs and os.path.exists(obj) and os.path.getmtime(obj) > max(map(os.path.getmtime, deps)):
            return obj  # up to date (per-object: only changed sources recompile)
        if src.endswith(".cu"):
            diag = ["-DFEA5_DIAG"] if os.environ.get("FEA_BUILD_DIAG") else []
            cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", *diag, *inc, "-c",
                   os.path.join(CSRC, src), "-o", obj]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function", "-pthread", "-fopenmp",
                   "-I", "/usr/local/cuda/include", *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    with open(stamp, "w") as f:
        f.write(defs_key)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", *ARCH, "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
