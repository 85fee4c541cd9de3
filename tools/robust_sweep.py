"""Convergence sweep over seeds and sizes with the current Rayleigh-Ritz form:
status, iterations, eigenvalue error against the closed form.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

rows = []
for N, m, jac, tol in [(32, 4, False, 1e-6), (20, 10, True, 1e-6), (24, 6, True, 1e-7),
                       (16, 8, True, 1e-8), (40, 12, True, 1e-6)]:
    s = float((N + 1) ** 2)
    a = pk.Laplacian3D((N, N, N), scale=s)
    exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
    st, its, worst = Counter(), [], 0.0
    for seed in range(16):
        rep = pk.solve(a, t=pk.jacobi_preconditioner(a) if jac else None,
                       config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
        key = rep.status if not rep.status.startswith("BasisFallback") else "BasisFallback"
        st[key] += 1
        its.append(rep.iterations_used)
        if rep.all_converged:
            worst = max(worst, float(np.max(np.abs(rep.eigenvalues - exact) / exact)))
    print(f"N={N} m={m} jac={jac} tol={tol:g}: {dict(st)} iterations {min(its)}..{max(its)} "
          f"median {int(np.median(its))} worst rel err {worst:.1e}", flush=True)
