"""A few iterations of an N^3, block-m Laplacian solve (optionally with the
C5 diagonal B), for ncu captures of one kernel.  Diagnostic only.
Usage: python tools/run_small.py N m [B]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
use_b = len(sys.argv) > 3 and sys.argv[3] == "B"
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
b = pk.DiagonalOperator(np.random.Generator(np.random.PCG64(1000)).uniform(1.0, 2.0, N ** 3)) if use_b else None
with pk.device_options(return_device=True):
    rep = pk.solve(a, b=b, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=1e-6, max_iter=8, seed=0))
print(rep.status, rep.eigenvalues[:3])
