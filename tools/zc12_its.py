"""Iterations of the chaotic generic-B case zc12 (tests/test_gpu_generic_b.py)
and of the golden 20^3 case under the current Rayleigh-Ritz form.  Diagnostic."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m, plane = 12, 6, 144


def bz(v):
    y = 2.5 * v
    y[plane:] -= 0.5 * v[:-plane]
    y[:-plane] -= 0.5 * v[plane:]
    return y


out = []
for k in range(-3, 4):
    a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2) * (1.0 + k * 2.0 ** -52))
    rep = pk.solve(a, b=lambda v: bz(v.clone()), config=pk.SolverConfig(block_size=m, tol=1e-7, max_iter=300, seed=0))
    out.append((rep.iterations_used, rep.status))
print("zc12 k=-3..3:", out)
a = pk.laplacian3d((20, 20, 20))
rep = pk.solve(a, t=pk.jacobi_preconditioner(a), config=pk.SolverConfig(block_size=10, tol=1e-6, max_iter=200, seed=2))
print("golden20:", rep.iterations_used, rep.status, sorted(int(x) for x in rep.lock_iterations))
