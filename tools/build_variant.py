#!/usr/bin/env python
"""Builds a kernel-variant copy of libmetldpc.so for A/B measurements (not product code).

    python tools/build_variant.py NAME -DMACRO=VALUE ...   ->  scratch/variants/NAME/libmetldpc.so
    python tools/build_variant.py NAME --rev GITREV ...    (kernels.cu as of a git revision)

kernels.cu is recompiled with the given -D flags; the host objects come from the normal
in-tree build.  Select a variant at run time with METLDPC_LIB=<path> (binding.py).
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1711_01783_b200 import build as B  # noqa: E402


def main(name: str, defines: list[str]) -> Path:
    B.build()
    out = ROOT / "scratch" / "variants" / name
    out.mkdir(parents=True, exist_ok=True)
    obj = out / "kernels.o"
    src = B.CSRC / "kernels.cu"
    tmp = None
    if "--rev" in defines:
        i = defines.index("--rev")
        rev = defines[i + 1]
        defines = defines[:i] + defines[i + 2:]
        tmp = B.CSRC / f"_variant_{name}.cu"   # next to the headers it includes
        tmp.write_text(subprocess.run(["git", "show", f"{rev}:paper_1711_01783_b200/csrc/kernels.cu"], cwd=ROOT,
                                      capture_output=True, text=True, check=True).stdout)
        src = tmp
    cmd = B._cmd(src, obj)
    cmd[1:1] = defines
    r = subprocess.run(cmd, capture_output=True, text=True)
    if tmp:
        tmp.unlink()
    (out / "ptxas.txt").write_text(r.stderr)
    if r.returncode:
        sys.exit(r.stderr)
    objs = [obj if o.stem == "kernels" else o for o in (B.OBJ / (Path(s).stem + ".o") for s in B.SOURCES)]
    lib = out / "libmetldpc.so"
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart", "static"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    return lib


if __name__ == "__main__":
    print(main(sys.argv[1], sys.argv[2:]))
