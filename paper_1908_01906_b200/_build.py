"""In-tree build of libtetray_b200.so (nvcc, sm_100a) and the parity oracle.

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box; nothing is installed into site-packages.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtetray_b200.so"
SOURCES = ["render.cu", "synth.cu", "pbuild.cu", "meta.cu", "epilogue.cu", "host_build.cpp", "common.cpp"]
HEADERS = [ROOT / "include" / "tetray_b200.h", CSRC / "tr_internal.h", CSRC / "glibc_pow.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit-exact fp64 contract: never contract a*b+c
    "-fmad=false",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-fno-fast-math,-O2",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libtetray_b200.so")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    from . import _glibc_pow
    _glibc_pow.write_header()  # glibc pow tables from the installed libm
    deps = [CSRC / s for s in SOURCES] + HEADERS + [CSRC / "glibc_pow_data.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, "-ccbin", "/usr/bin/g++",
           "-I", str(ROOT / "include"), "-I", str(CSRC),
           *[str(CSRC / s) for s in SOURCES],
           "-o", str(tmp), "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    (PKG / "ptxas_info.txt").write_text(res.stderr)
    os.replace(tmp, LIB)
    return LIB


def build_oracle(force: bool = False) -> Path:
    """The C parity oracle (test infrastructure; see oracle/oracle.c)."""
    target = ROOT / "oracle" / "liboracle.so"
    srcs = [ROOT / "oracle" / f for f in ("oracle.c", "build.c", "Makefile")]
    if force or _stale(target, srcs):
        res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-B" if force else "-s"],
                             capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    return target


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
    print(build_oracle(force=True))
