"""Build libb200lobpcg.so in-tree with nvcc for sm_100a.

    python -m paper_0705_2626_b200.build

The shared library lands next to this file (paper_0705_2626_b200/lib/) so it
travels with the repo snapshot to the GPU box.  No torch extension machinery:
the boundary is a plain C ABI (include/b200lobpcg.h) loaded with ctypes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIBNAME = "libb200lobpcg.so"
SOURCES = ["abi.cu", "stencil.cu", "stencil_gram.cu", "blockops.cu", "fused.cu", "rr.cu", "rng.cu", "pcg.cu", "iterate.cu", "slab.cu"]
HEADERS = ["common.cuh", "gram_tile.cuh", "stencil.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def lib_path() -> Path:
    return LIBDIR / LIBNAME


def _stale(out: Path) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "b200lobpcg.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr)


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None) -> Path:
    """One object per translation unit (compiled in parallel), then one
    shared-library link; no relocatable device code crosses files."""
    from concurrent.futures import ThreadPoolExecutor

    out = lib_path()
    if not force and not _stale(out):
        return out
    LIBDIR.mkdir(exist_ok=True)
    objdir = LIBDIR / "obj"
    objdir.mkdir(exist_ok=True)
    objs = [objdir / (Path(s).stem + ".o") for s in SOURCES]
    cmds = [[nvcc(), *NVCC_FLAGS, *(extra or []), "-c", "-o", str(o), str(CSRC / s)]
            for s, o in zip(SOURCES, objs)]
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda c: _run(c, verbose), cmds))
    tmp = out.with_suffix(".so.tmp")
    _run([nvcc(), *NVCC_FLAGS, "-shared", "-o", str(tmp), *map(str, objs), "-ldl"], verbose)
    tmp.replace(out)
    return out


if __name__ == "__main__":
    force = "--force" in sys.argv
    verbose = "-v" in sys.argv
    extra = ["-Xptxas", "-v"] if "--ptxas" in sys.argv else None
    print(build(force=force, verbose=verbose or bool(extra), extra=extra))
