"""Build libfbx.so in-tree with nvcc for sm_100a (the driver's build() check).

The plan kernels themselves are generated per plan and compiled at prepare
time by NVRTC through ``fbx_compile``; this builds the C-ABI runtime and its
precompiled kernels.
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "libfbx.so"
SOURCES = [PKG / "csrc" / "fbx_runtime.cu", PKG / "csrc" / "fbx_engine.cu",
           PKG / "csrc" / "fbx_table.cu"]
HEADERS = [ROOT / "include" / "fbx.h", ROOT / "include" / "fbx_abi.h"]
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def nvcc_command() -> list[str]:
    return [str(CUDA / "bin" / "nvcc"), "-gencode", "arch=compute_100a,code=sm_100a",
            "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
            "-cudart", "static", f"-I{ROOT / 'include'}", "-o", str(LIB),
            *map(str, SOURCES), f"-L{CUDA / 'lib64'}", "-lnvrtc", "-ldl",
            "-Xlinker", f"-rpath,{CUDA / 'lib64'}"]


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


GEN_LIB = PKG / "libfbxgen.so"
GEN_SRC = PKG / "csrc" / "corpus_gen.c"


def build_corpus_gen(force: bool = False) -> Path:
    """gcc build of the bulk corpus generator (measurement input)."""
    if force or not GEN_LIB.exists() or GEN_SRC.stat().st_mtime > GEN_LIB.stat().st_mtime:
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", str(GEN_LIB), str(GEN_SRC)],
                       check=True)
    return GEN_LIB


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if force or stale():
        cmd = nvcc_command()
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build_library(force=True, verbose=True)
    build_corpus_gen(force=True)
