"""Residual / Ritz trace of the late iterations of one case.  Diagnostic.
python tools/trace_case.py N m tol seed [from_it]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m, tol, seed = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
it0 = int(sys.argv[5]) if len(sys.argv) > 5 else 0
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
               config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
print(rep.status, rep.iterations_used, list(int(x) for x in rep.lock_iterations))
exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
np.set_printoptions(linewidth=220, precision=2)
for h in rep.history:
    if h.iteration >= it0 and (h.iteration % 10 == 0 or h.fallbacks or h.locked_now
                               or h.iteration >= rep.iterations_used - 3):
        act = np.flatnonzero(h.active)
        print(h.iteration, "active", list(act), "resid", h.residual_norms[act],
              "ritz-exact", (h.ritz - exact)[act], "fb", h.fallbacks, "locked", h.locked_now)
