"""Steady-state timing of one BASELINE-like config on one GPU: ms per
iteration of the native loop (CUDA events over a window) and the per-kernel
CUDA-event means of a timer pass (the Python-driven path), with each
kernel's algorithmic GB/s.  Diagnostic only.

    python tools/time_config.py N m [--b] [--warm W] [--steps K]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("N", type=int)
ap.add_argument("m", type=int)
ap.add_argument("--b", action="store_true")
ap.add_argument("--warm", type=int, default=5)
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
N, m = args.N, args.m
n = N ** 3
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
b = (pk.DiagonalOperator(np.random.Generator(np.random.PCG64(1000)).uniform(1.0, 2.0, n))
     if args.b else None)
cfg = pk.SolverConfig(block_size=m, tol=1e-6, max_iter=args.warm + 2 * args.steps + 10, seed=0)
run = pk.LOBPCGRun(a, b=b, t=pk.jacobi_preconditioner(a), config=cfg)
for _ in range(args.warm):
    run.step()
torch.cuda.synchronize()
import ctypes  # noqa: E402
from paper_0705_2626_b200 import _lib  # noqa: E402
_buf = (ctypes.c_double * 8)()
_lib.load().b2l_iter_profile(_buf, 1)   # reset the host phase timers (B2L_ITER_PROFILE=1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    run.step()
e1.record()
torch.cuda.synchronize()
ms_it = e0.elapsed_time(e1) / args.steps
_on = _lib.load().b2l_iter_profile(_buf, 0)
kt = {}


def timer(name, fn):
    x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x.record()
    r = fn()
    y.record()
    kt.setdefault(name, []).append((x, y))
    return r


with pk.device_options(timer=timer):
    for _ in range(args.steps):
        run.step()
torch.cuda.synchronize()
alg = ({"step": 8.0 * n * 11 * m, "stencil": 16.0 * n * m + 8.0 * n * m} if m <= 16
       else {"stencil": 16.0 * n * m})   # above 16 columns: the plain stencil
out = {"N": N, "m": m, "ms_per_it": ms_it, "it_s": 1e3 / ms_it,
       "iteration_gbs": 104.0 * n * m / (ms_it / 1e3) / 1e9}
for k, v in kt.items():
    d = float(np.mean([x.elapsed_time(y) for x, y in v]))
    out[k] = {"ms": d, "calls": len(v)}
    if k in alg:
        out[k]["gbs"] = alg[k] / (d / 1e3) / 1e9
if _on:
    c = max(_buf[0], 1.0)
    out["host_phase_us"] = {"native_steps": int(_buf[0]), "fetch_enqueue": _buf[1] / c,
                            "sync_wait": _buf[2] / c, "drift_lock": _buf[3] / c,
                            "rr_first_half": _buf[6] / c, "wait_g2": _buf[7] / c,
                            "rr_second_half": _buf[4] / c, "uploads_launches": _buf[5] / c}
print(json.dumps(out))
