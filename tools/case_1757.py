"""The fuzz case that stalled before the stall watch (24^3, m = 9, tol 1e-8,
seeds 1757..1760): status, iterations, refreshes.  Diagnostic."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk
N, m = 24, 9
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
for seed in (1757, 1758, 1759, 1760):
    run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a), config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=3000, seed=seed))
    while run.step():
        pass
    rep = run.report()
    print("   refreshes", run.ax_refreshes, "repairs", run.drift_repairs)
    h = rep.history[-1]
    act = np.flatnonzero(h.active)
    print(seed, rep.status, rep.iterations_used, int(rep.converged.sum()), sorted(int(x) for x in rep.lock_iterations),
          "last resid", h.residual_norms[act], "ritz-exact", (h.ritz - exact)[act])
