#!/usr/bin/env python3
"""Seeds 0..15 of two shapes run to convergence by the REAL reference: status,
iterations, fallbacks (-> seed_sweep.npz).  The GPU test holds the B200 path's
failure / stall behaviour to these (tests/test_gpu_solve.py::test_seed_sweep_*).
Build container only:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_seed_sweep.py"""
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
from blockeig import (  # noqa: E402
    MatrixFreeOperator, SolverConfig, jacobi_preconditioner, laplacian3d, solve)

OUT = Path(__file__).parent
out = {}
for name, N, m, tol in [("n20", 20, 10, 1e-6), ("n16", 16, 8, 1e-8)]:
    s = float((N + 1) ** 2)
    L = laplacian3d((N, N, N))
    A = MatrixFreeOperator(N ** 3, lambda v, L=L, s=s: s * L(v), spd=True,
                           diag=np.full(N ** 3, 6.0 * s))
    its, status, fb = [], [], []
    for seed in range(16):
        rep = solve(A, t=jacobi_preconditioner(A),
                    config=SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
        its.append(rep.iterations_used)
        status.append(rep.status)
        fb.append(rep.basis_fallbacks)
    print(name, its, status, flush=True)
    out[name + "_iterations"] = np.array(its)
    out[name + "_status"] = np.array(status)
    out[name + "_fallbacks"] = np.array(fb)
np.savez_compressed(OUT / "seed_sweep.npz", **out)
