"""One scaled-Laplacian case, all seeds: status / iterations / lock iterations
/ fallbacks.  python tools/one_case.py N m tol [jac=1] [seeds=16]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m, tol = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
jac = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
seeds = int(sys.argv[5]) if len(sys.argv) > 5 else 16
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
for seed in range(seeds):
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a) if jac else None,
                   config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
    fb = [h.iteration for h in rep.history if h.fallbacks]
    print(seed, rep.status, rep.iterations_used, sorted(int(x) for x in rep.lock_iterations),
          "fallback its", fb[:6], "..." if len(fb) > 6 else "", len(fb),
          "resid max %.1e" % float(np.max(rep.residual_norms)), flush=True)
