"""In-tree build of the native libraries (nvcc for sm_100a, g++ for the host layer).

Outputs (git-ignored, shipped to the GPU box with the snapshot):
  paper_1702_05854_b200/lib/libhsaw_gpu.so    CUDA kernels + the C-ABI of include/hsaw_gpu.h
  paper_1702_05854_b200/lib/libhsaw_host.so   C++ host layer mirroring the reference's hsaw:: API
  paper_1702_05854_b200/bin/hsaw              drop-in CLI (interdict / sample / bench)
"""
from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
LIB = os.path.join(PKG, "lib")
BIN = os.path.join(PKG, "bin")
OBJ = os.path.join(PKG, "lib", "obj")

GPU_SO = os.path.join(LIB, "libhsaw_gpu.so")
HOST_SO = os.path.join(LIB, "libhsaw_host.so")
CLI = os.path.join(BIN, "hsaw")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
CXX = "/usr/bin/g++"  # the environment's $CXX wrapper links libstdc++ statically; see oracle/Makefile

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-ccbin", CXX,
    "-Xcompiler", "-fPIC",
    "-diag-suppress", "128",
]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _sources(directory: str, exts: tuple[str, ...]) -> list[str]:
    if not os.path.isdir(directory):
        return []
    return sorted(os.path.join(directory, f) for f in os.listdir(directory) if f.endswith(exts))


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a for every .cu under csrc/, linked into one .so."""
    cus = _sources(CSRC, (".cu",))
    cpps = _sources(CSRC, (".cpp",))
    headers = _sources(CSRC, (".cuh", ".h")) + [os.path.join(ROOT, "include", "hsaw_gpu.h")]
    if not force and _newer(GPU_SO, cus + cpps + headers):
        return GPU_SO
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(cu: str) -> str:
        obj = os.path.join(OBJ, os.path.basename(cu)[:-3] + ".o")
        if not force and _newer(obj, [cu] + headers):
            return obj
        cmd = [NVCC, *NVCC_FLAGS, "-c", cu, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        return obj

    def compile_cpp(cpp: str) -> str:  # host-only helpers of the same library (plain g++)
        obj = os.path.join(OBJ, os.path.basename(cpp)[:-4] + ".o")
        if force or not _newer(obj, [cpp] + headers):
            subprocess.check_call([CXX, "-std=c++17", "-O3", "-fPIC", "-pthread", "-c", cpp, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=4) as ex:
        objs = list(ex.map(compile_one, cus))
    objs += [compile_cpp(c) for c in cpps]
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-ccbin", CXX,
                           "-o", GPU_SO, *objs, "-lcudart"])
    return GPU_SO


def build_host(force: bool = False) -> str | None:
    """g++ build of the C++ host layer + CLI on top of the C-ABI."""
    cpps = [c for c in _sources(HOST, (".cpp",)) if not c.endswith("_main.cpp")]
    if not cpps:
        return None
    headers = _sources(HOST, (".hpp", ".h")) + [os.path.join(ROOT, "include", "hsaw_gpu.h")]
    flags = ["-std=c++20", "-O2", "-fPIC", "-pthread", "-Wall", "-Wextra", "-I",
             os.path.join(ROOT, "include"), "-I", HOST]
    if force or not _newer(HOST_SO, cpps + headers + [GPU_SO]):
        subprocess.check_call([CXX, *flags, "-shared", "-o", HOST_SO, *cpps, "-L", LIB,
                               "-lhsaw_gpu", "-ldl", "-pthread", "-Wl,-rpath,$ORIGIN"])
    mains = [c for c in _sources(HOST, (".cpp",)) if c.endswith("_main.cpp")]
    if mains and (force or not _newer(CLI, mains + headers + [HOST_SO])):
        os.makedirs(BIN, exist_ok=True)
        subprocess.check_call([CXX, *flags, "-o", CLI, *mains, "-L", LIB, "-lhsaw_host",
                               "-lhsaw_gpu", "-Wl,-rpath,$ORIGIN/../lib"])
    return HOST_SO


def build_all(force: bool = False, verbose: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    build_gpu(force, verbose)
    build_host(force)


def clean() -> None:
    shutil.rmtree(LIB, ignore_errors=True)
    shutil.rmtree(BIN, ignore_errors=True)


if __name__ == "__main__":
    import sys

    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(GPU_SO)
