"""Build an A/B variant of libb200lobpcg.so with extra nvcc defines into
scratch/variants/<name>.so (git-ignored; travels to the GPU box), to be
selected with B2L_LIB_PATH.  Diagnostic only.

    python tools/build_variant.py name -DB2L_PAIR_BALANCE=0 [...]
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0705_2626_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = b.ROOT / "scratch" / "variants"
objdir = out / (name + "_obj")
objdir.mkdir(parents=True, exist_ok=True)
objs = [objdir / (Path(s).stem + ".o") for s in b.SOURCES]


def cc(so):
    s, o = so
    r = subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *extra, "-c", "-o", str(o), str(b.CSRC / s)],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)


with ThreadPoolExecutor(8) as ex:
    list(ex.map(cc, zip(b.SOURCES, objs)))
lib = out / (name + ".so")
subprocess.run([b.nvcc(), *b.NVCC_FLAGS, "-shared", "-o", str(lib), *map(str, objs), "-ldl"],
               check=True)
print(lib)
