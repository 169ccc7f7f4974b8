"""Builds libmetldpc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

host code : g++ -O2 -ffp-contract=off (phi tables are fp64 closed forms, N2)
kernels   : nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
            (no FMA contraction: the fp32 sequence is DESIGN.md N1-N5; explicit
            __fmaf_rn only in the phi table evaluation)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libmetldpc.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["host_code.cpp", "kernels.cu", "decoder.cu"]
EXTRA = os.environ.get("METLDPC_NVCC_EXTRA", "").split()
HEADERS = ["internal.h", "kernels.cuh"]


def _cmd(src: Path, obj: Path) -> list[str]:
    if src.suffix == ".cpp":
        return ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                f"-I{INCLUDE}", "-c", str(src), "-o", str(obj)]
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xptxas", "-v", *EXTRA,
            "-Xcompiler", "-fPIC,-ffp-contract=off", f"-I{INCLUDE}", "-c", str(src), "-o", str(obj)]


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    deps_mtime = max((CSRC / h).stat().st_mtime for h in HEADERS)
    deps_mtime = max(deps_mtime, (INCLUDE / "metldpc.h").stat().st_mtime)
    objs = []
    relinked = force or not LIB.exists()
    for s in SOURCES:
        src = CSRC / s
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, deps_mtime):
            cmd = _cmd(src, obj)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or r.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"compile failed: {s}")
            (OBJ / (src.stem + ".ptxas.txt")).write_text(r.stderr)
            relinked = True
    if relinked or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
