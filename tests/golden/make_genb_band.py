#!/usr/bin/env python3
"""A wider reference iteration band for the chaotic generic-B case zc12
(12^3, m = 6, B couples z-neighbours, tol 1e-7, no T): the REAL reference with
its operator scaled by (1 + k ulp), k = +-1..32 (make_golden.py's fixture has
k = +-1..4).  Build container only:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_genb_band.py
-> genb_zc12_band64.npz (ulps, iterations, status)."""
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
from blockeig import MatrixFreeOperator, SolverConfig, laplacian3d, solve  # noqa: E402

OUT = Path(__file__).parent
N, m, tol = 12, 6, 1e-7
n, plane = N ** 3, N * N
s = float((N + 1) ** 2)
L = laplacian3d((N, N, N))


def b_zcouple(v):
    y = 2.5 * v
    y[plane:] -= 0.5 * v[:-plane]
    y[:-plane] -= 0.5 * v[plane:]
    return y


B = MatrixFreeOperator(n, b_zcouple, spd=True)
ulps, its, status = [], [], []
for k in [k for k in range(-32, 33) if k]:
    s1 = 1.0 + k * 2.0 ** -52
    A = MatrixFreeOperator(n, lambda v, s1=s1: s1 * (s * L(v)), spd=True,
                           diag=np.full(n, 6.0 * s1 * s))
    rep = solve(A, b=B, config=SolverConfig(block_size=m, tol=tol, max_iter=300, seed=0))
    ulps.append(k)
    its.append(rep.iterations_used)
    status.append(rep.status)
print(sorted(set(its)), {x: status.count(x) for x in set(status)})
np.savez_compressed(OUT / "genb_zc12_band64.npz", ulps=np.array(ulps), iterations=np.array(its),
                    status=np.array(status))
