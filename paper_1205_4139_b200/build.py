"""Build libfmp_cuda.so (sm_100a) in-tree with nvcc.

    python -m paper_1205_4139_b200.build [--force]

Objects are compiled in parallel into ``paper_1205_4139_b200/_build`` and
linked into ``paper_1205_4139_b200/libfmp_cuda.so`` (cudart linked
statically, so the library needs nothing beyond the driver).  Sources are
rebuilt only when newer than their object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# FMP_BUILD_DEFS / FMP_BUILD_OUT: an experimental variant (extra -D flags)
# built into its own object directory and library, e.g. _variants/x.so
DEFS = os.environ.get("FMP_BUILD_DEFS", "").split()
_VOUT = os.environ.get("FMP_BUILD_OUT")
OBJ = os.path.join(PKG, "_build") if not _VOUT else os.path.abspath(_VOUT) + "_obj"
LIB = os.path.join(PKG, "libfmp_cuda.so") if not _VOUT else os.path.abspath(_VOUT) + ".so"
FACADE = os.path.join(PKG, "libfastmp_b200.so")
DRIVER = os.path.join(PKG, "fmp_driver")
CXX = os.environ.get("CXX", "g++")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"), *DEFS]
SOURCES = ["fmp_omp_c128.cu", "fmp_omp_c64.cu", "fmp_omp_f64.cu", "fmp_omp_f32.cu", "fmp_omp.cu", "fmp_cosamp.cu", "fmp_large.cu", "fmp_large_host.cu", "fmp_fast_update.cu", "fmp_qr.cu", "fmp_transform.cu", "fmp_transform_4s.cu", "fmp_transform_fold.cu", "fmp_capi.cu", "fmp_gen.cu", "fmp_host_gen.cpp"]
HEADERS = ["fmp_device.cuh", "fmp_kernels.cuh", "fmp_kcommon.cuh", "fmp_omp_impl.cuh", "fmp_capi_internal.cuh"]


def _newest_dep(src: str) -> float:
    # fmp_omp_impl.cuh is included by the fmp_omp_<dtype>.cu units only
    hs = [h for h in HEADERS if h != "fmp_omp_impl.cuh" or src.startswith("fmp_omp_")]
    deps = [os.path.join(CSRC, h) for h in hs] + [os.path.join(ROOT, "include", "fmp.h")]
    return max(os.path.getmtime(d) for d in deps)


def _compile(src: str, force: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _newest_dep(src)):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *COMMON, "-x", "c++", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if _VOUT:
        return LIB
    # the C++ drop-in facade over the C ABI
    src = os.path.join(PKG, "host", "fastmp_facade.cpp")
    if force or not os.path.exists(FACADE) or os.path.getmtime(FACADE) < max(
            os.path.getmtime(src), os.path.getmtime(LIB),
            os.path.getmtime(os.path.join(ROOT, "include", "fastmp_b200", "fastmp.hpp"))):
        cmd = [CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
               "-I" + os.path.join(ROOT, "include"), "-o", FACADE, src, LIB,
               "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"facade build failed:\n{r.stderr}")
    # the seeded multi-GPU driver (C ABI only)
    dsrc = os.path.join(PKG, "host", "fmp_driver.cpp")
    if force or not os.path.exists(DRIVER) or os.path.getmtime(DRIVER) < max(
            os.path.getmtime(dsrc), os.path.getmtime(LIB)):
        cmd = [CXX, "-std=c++17", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
               "-o", DRIVER, dsrc, LIB, "-lpthread", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"driver build failed:\n{r.stderr}")
    if verbose:
        print("built", LIB, "and", FACADE, "and", DRIVER)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
