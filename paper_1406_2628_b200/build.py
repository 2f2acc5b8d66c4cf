"""Build recipe for the native library (sm_100a only).

`build()` compiles paper_1406_2628_b200/csrc/mp_capi.cu into the in-tree
shared library paper_1406_2628_b200/libmergepath_b200.so with

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo ...

nvcc cross-compiles without a GPU, so this runs in the CPU container and the
resulting .so travels to the GPU box with the repository snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmergepath_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libmergepath_b200.so")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [
        ROOT / "include" / "mergepath_b200.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in sources())


TOOL_SRC = PKG / "tools" / "mergebench_b200.cpp"
TOOL = PKG / "bin" / "mergebench_b200"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def build_tool(verbose: bool = False) -> Path:
    """mergebench_b200: the reference tool's CLI contract over the drop-in
    headers and the C ABI (g++ -std=c++20, linked to the in-tree library)."""
    TOOL.parent.mkdir(exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", "-pthread",
           "-I", str(ROOT / "include"), "-I", str(CUDA_HOME / "include"),
           "-o", str(TOOL) + ".tmp", str(TOOL_SRC),
           "-L", str(PKG), "-lmergepath_b200", "-Wl,-rpath,$ORIGIN/..",
           "-L", str(CUDA_HOME / "lib64"), "-lcudart_static", "-ldl", "-lrt"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=ROOT)
    os.replace(str(TOOL) + ".tmp", TOOL)
    return TOOL


MULTI_SRC = ROOT / "tests" / "cpp" / "test_multi_gpu.cpp"
MULTI_TEST = PKG / "bin" / "test_multi_gpu"


def build_multi_test(verbose: bool = False) -> Path:
    """The C++ caller of mp_multi_merge / mp_multi_sort (no Python)."""
    MULTI_TEST.parent.mkdir(exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-Wall", "-Wextra",
           "-I", str(ROOT / "include"), "-I", str(CUDA_HOME / "include"),
           "-o", str(MULTI_TEST) + ".tmp", str(MULTI_SRC),
           "-L", str(PKG), "-lmergepath_b200", "-Wl,-rpath,$ORIGIN/..",
           "-L", str(CUDA_HOME / "lib64"), "-lcudart_static", "-ldl", "-lrt", "-pthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=ROOT)
    os.replace(str(MULTI_TEST) + ".tmp", MULTI_TEST)
    return MULTI_TEST


def build(force: bool = False, verbose: bool = False) -> Path:
    if force or not up_to_date():
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(LIB) + ".tmp", str(CSRC / "mp_capi.cu")]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=ROOT)
        os.replace(str(LIB) + ".tmp", LIB)
    if force or not TOOL.exists() or TOOL.stat().st_mtime < max(
            LIB.stat().st_mtime, TOOL_SRC.stat().st_mtime,
            *(p.stat().st_mtime for p in (ROOT / "include").rglob("*.h*"))):
        build_tool(verbose)
    if force or not MULTI_TEST.exists() or MULTI_TEST.stat().st_mtime < max(
            LIB.stat().st_mtime, MULTI_SRC.stat().st_mtime):
        build_multi_test(verbose)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
