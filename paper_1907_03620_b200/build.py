"""In-tree build of the native libraries (sm_100a only).

    libraster_b200.so    CUDA kernels + C-ABI (include/raster_gpu.h) — the product
    libraster_datagen.so seeded synthetic workloads (include/raster_datagen.h)

Both land next to this file so they travel with the repository snapshot to
the GPU box. The CPU checkers under oracle/ are built by oracle/build_ref.sh
(test infrastructure; see oracle/raster_oracle.h).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
GPU_LIB = PKG / "libraster_b200.so"
GEN_LIB = PKG / "libraster_datagen.so"

CUDA_SOURCES = ["contract.cu", "agglomerate.cu", "agglomerate_sorted.cu", "label.cu", "points.cu", "dedupe.cu", "partition.cu", "api.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_gpu(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in CUDA_SOURCES]
    deps = srcs + [CSRC / "common.cuh", CSRC / "internal.h", ROOT / "include" / "raster_gpu.h"]
    if force or _stale(GPU_LIB, deps):
        tmp = GPU_LIB.with_suffix(".so.tmp")
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(tmp), *map(str, srcs)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=str(CSRC))
        tmp.replace(GPU_LIB)
    return GPU_LIB


def build_datagen(force: bool = False, verbose: bool = False) -> Path:
    src = CSRC / "datagen.cpp"
    if force or _stale(GEN_LIB, [src, ROOT / "include" / "raster_datagen.h"]):
        tmp = GEN_LIB.with_suffix(".so.tmp")
        cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", str(tmp), str(src)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        tmp.replace(GEN_LIB)
    return GEN_LIB


def build_oracle(verbose: bool = False) -> None:
    """Compile the CPU checkers (the C restatement; and the reference itself
    when /root/reference is present)."""
    out = subprocess.run(["bash", str(ROOT / "oracle" / "build_ref.sh")], check=True,
                         capture_output=not verbose, text=True)
    if verbose and out.stdout:
        print(out.stdout)


def build_cpp_tests(verbose: bool = False) -> None:
    """C++ drop-in parity test (needs the reference headers; skipped if absent)."""
    out = subprocess.run(["bash", str(ROOT / "tests" / "cpp" / "build.sh")], check=True,
                         capture_output=not verbose, text=True)
    if verbose and out.stdout:
        print(out.stdout)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_gpu(force, verbose)
    build_datagen(force, verbose)
    build_oracle(verbose)
    build_cpp_tests(verbose)


if __name__ == "__main__":
    build_all(force=True, verbose=True)
