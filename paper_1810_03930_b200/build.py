"""Build recipe of the native library (sm_100a only, in-tree).

``python -m paper_1810_03930_b200.build`` compiles every CUDA/C++ source under
``csrc/`` with nvcc for ``-gencode arch=compute_100a,code=sm_100a`` into
``paper_1810_03930_b200/libpcal_b200.so`` (objects under ``build/``), the
C++ header-mirror example ``build/pcal_cpp_example`` and the caller-defined
device model example ``build/libpcal_device_model_example.so``.  Sources are rebuilt
only when they (or any header) are newer than their object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "pcal_b200")
LIB = os.path.join(PKG, "libpcal_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "--expt-relaxed-constexpr", "-diag-suppress", "177"]
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra"]


def _headers() -> list:
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*", "*.hpp")))


def _stale(obj: str, src: str, deps: list) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def _compile(src: str, verbose: bool) -> str:
    base = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(BUILD, base + ".o")
    if not _stale(obj, src, _headers()):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, *CUFLAGS, "-c", src, "-o", obj]
    else:
        cmd = ["g++", *CXXFLAGS, "-I/usr/local/cuda/include", "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    ex_src = os.path.join(ROOT, "examples", "pcal_cpp_example.cpp")
    if os.path.exists(ex_src):
        exe = os.path.join(os.path.dirname(BUILD), "pcal_cpp_example")
        if _stale(exe, ex_src, _headers() + [LIB]):
            cmd = ["g++", "-O2", "-std=c++17", f"-I{ROOT}/include", ex_src, "-o", exe,
                   f"-L{PKG}", "-lpcal_b200", f"-Wl,-rpath,{PKG}"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"example build failed\n{r.stdout}\n{r.stderr}")
    dm_src = os.path.join(ROOT, "examples", "device_model_example.cu")
    if os.path.exists(dm_src):  # a caller-defined device model (PCAL_MODEL_DEVICE_CALLBACK)
        so = os.path.join(os.path.dirname(BUILD), "libpcal_device_model_example.so")
        if _stale(so, dm_src, _headers()):
            cmd = [NVCC, *ARCH, *CUFLAGS, f"-I{ROOT}/include", "-shared", dm_src, "-o", so]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"device-model example build failed\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
