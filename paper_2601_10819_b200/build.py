"""Build the in-tree C-ABI library ``paper_2601_10819_b200/lib/libmsda_b200.so``.

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu source pages map to the kernels.  The library has no
torch dependency: its interface is ``include/msda_b200.h``.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "lib" / "obj"
LIB = PKG / "lib" / "libmsda_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         "-I", str(PKG.parent / "include"), *os.environ.get("MSDA_EXTRA_NVCC_FLAGS", "").split()]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), PKG.parent / "include" / "msda_b200.h"]
    return obj.stat().st_mtime < max(d.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    # objects built with other flags (e.g. a builder-only MSDA_EXTRA_NVCC_FLAGS
    # timeline build) are stale whatever their mtimes
    stamp = OBJ / "flags.txt"
    flags = " ".join([*ARCH, *FLAGS])
    if not stamp.exists() or stamp.read_text() != flags:
        force = True
    srcs = sources()
    objs = [OBJ / (s.stem + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if force or _stale(obj, src):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
            return True
        return False

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        changed = any(list(ex.map(compile_one, zip(srcs, objs))))
    if force or changed or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        subprocess.run(cmd, check=True)
    stamp.write_text(flags)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
