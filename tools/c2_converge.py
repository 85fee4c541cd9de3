"""C2 (128^3, m = 10, Jacobi, tol 1e-8) run to convergence (max_iter 1500) over
a few 1-ulp perturbations of the operator scale: status, iterations, lock
iterations -- to compare Rayleigh-Ritz forms (B2L_RR_EIG / B2L_RR_ALIGN).
Diagnostic only:  python tools/c2_converge.py [K]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_0705_2626_b200 as pk  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
N, m = 128, 10
base = float((N + 1) ** 2)
rows = []
for k in range(-K, K + 1):
    s = base * (1.0 + k * 2.0 ** -52)
    a = pk.Laplacian3D((N, N, N), scale=s)
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=1500, seed=0))
    exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
    err = float(np.max(np.abs(rep.eigenvalues - exact) / exact))
    rows.append((k, rep.status, int(rep.iterations_used), int(rep.converged.sum()), err))
    print(k, rep.status, rep.iterations_used, int(rep.converged.sum()), f"{err:.1e}",
          sorted(int(x) for x in rep.lock_iterations), flush=True)
its = [r[2] for r in rows]
print(json.dumps({"converged": sum(r[1] == "Converged" for r in rows), "runs": len(rows),
                  "median_it": int(np.median(its)), "min_it": min(its), "max_it": max(its)}))
