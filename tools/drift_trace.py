"""Drift (max |X^T B X - I|) per iteration and the drift repairs of a C2
solve on the native loop.  Diagnostic only: python tools/drift_trace.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m = 128, 10
a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=300, seed=0))
drift, reps = [], []
while True:
    r0 = run.drift_repairs
    ok = run.step()
    if run._native is not None:
        drift.append(float(run._native.drift))
    if run.drift_repairs > r0:
        reps.append(run.it)
    if not ok:
        break
d = np.array(drift)
print(f"repairs {run.drift_repairs} at {reps}; drift median {np.median(d):.2e}, "
      f"p90 {np.quantile(d, 0.9):.2e}, max {d.max():.2e}")
