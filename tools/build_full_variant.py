#!/usr/bin/env python
"""Builds a full-library variant (host code and kernels with the same -D flags; not product code).

    python tools/build_full_variant.py NAME -DMACRO=VALUE ...  ->  scratch/variants/NAME/libmetldpc.so
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1711_01783_b200 import build as B  # noqa: E402


def main(name, defines):
    out = ROOT / "scratch" / "variants" / name
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    for s in B.SOURCES:
        src = B.CSRC / s
        obj = out / (src.stem + ".o")
        cmd = B._cmd(src, obj)
        cmd[1:1] = defines
        r = subprocess.run(cmd, capture_output=True, text=True)
        (out / (src.stem + ".ptxas.txt")).write_text(r.stderr)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(obj)
    lib = out / "libmetldpc.so"
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart", "static"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    return lib


if __name__ == "__main__":
    print(main(sys.argv[1], sys.argv[2:]))
