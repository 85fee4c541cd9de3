"""Phase timeline of F1's compute warps (library built with -DB2L_TRACE, see
fused.cu): per warp and chunk the clocks spent waiting for an output buffer,
waiting for the stage, in the update, at the pair barrier, in the Gram, and
releasing.  Diagnostic only:
    python tools/build_variant.py trace -DB2L_TRACE
    B2L_LIB_PATH=scratch/variants/trace.so python tools/trace_f1.py"""
import ctypes
import runpy
import sys
from pathlib import Path

import numpy as np

sys.argv = [sys.argv[0]]
runpy.run_path(str(Path(__file__).with_name("time_f1.py")), run_name="__main__")
from paper_0705_2626_b200 import _lib  # noqa: E402

lib = _lib.load()
buf = (ctypes.c_longlong * (16 * 48 * 8))()
rc = lib.b2l_debug_trace(buf)
assert rc == 0, rc
t = np.ctypeslib.as_array(buf).reshape(16, 48, 8)[:14].astype(np.float64)
names = ["wait out-buffer", "wait stage", "update", "pair barrier", "Gram", "release"]
chunks = slice(8, 40)
d = np.diff(t[:, chunks, :7], axis=2)           # (warp, chunk, 6 phases)
period = np.diff(t[:, chunks, 0], axis=1)       # loop top to loop top
print("chunk period (clocks): mean %.0f  per warp %s" % (period.mean(), np.round(period.mean(1))))
half = np.array([(cw & 1) ^ ((cw >> 2) & 1) for cw in range(14)])   # pair_half (fused.cu)
for h, nm in ((0, "half 0 (columns 0-7, DMMA)"), (1, "half 1 (columns 8-9, DFMA tail)")):
    print(nm)
    sel = half == h
    for k, n in enumerate(names):
        print("  %-16s mean %7.0f   (per warp %s)" % (n, d[sel][:, :, k].mean(),
                                                      np.round(d[sel][:, :, k].mean(1))))
