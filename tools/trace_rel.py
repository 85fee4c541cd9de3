"""Relative-tolerance case: find failing seeds and trace the end.  Diagnostic."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m, tol = 20, 10, 1e-8
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
np.set_printoptions(linewidth=220, precision=2)
for seed in range(16):
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed,
                                          relative_tol=True))
    if rep.status.startswith("Failed") or rep.basis_fallbacks:
        print("seed", seed, rep.status, rep.iterations_used, list(int(x) for x in rep.lock_iterations))
        for h in rep.history[-25:]:
            act = np.flatnonzero(h.active)
            print(" ", h.iteration, "active", list(act), "resid", h.residual_norms[act],
                  "thr", (tol * exact)[act], "ritz-exact", (h.ritz - exact)[act], "fb", h.fallbacks)
