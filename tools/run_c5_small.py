"""A few C5-shaped iterations (m = 64, diagonal B, Jacobi) on a 128^3 grid,
for ncu captures of the large-block kernels.  Diagnostic only."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
b = pk.DiagonalOperator(np.random.Generator(np.random.PCG64(1000)).uniform(1.0, 2.0, N ** 3))
with pk.device_options(return_device=True):
    rep = pk.solve(a, b=b, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=64, tol=1e-6, max_iter=6, seed=0))
print(rep.status, rep.eigenvalues[:3])
