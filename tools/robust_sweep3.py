"""Third sweep: relative-tolerance mode on degenerate spectra (16 seeds).
`python tools/robust_sweep3.py [oracle]`.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ORACLE = len(sys.argv) > 1 and sys.argv[1] == "oracle"
if ORACLE:
    from oracle import lobpcg_oracle as orc
else:
    import paper_0705_2626_b200 as pk
for N, m, tol in [(20, 10, 1e-8), (16, 8, 1e-9), (24, 7, 1e-7)]:
    st, its = Counter(), []
    for seed in range(16):
        if ORACLE:
            r = orc.laplacian_case(N, m, precond="jacobi", tol=tol, max_iter=1500, seed=seed,
                                   record=False, relative_tol=True) \
                if "relative_tol" in orc.laplacian_case.__code__.co_varnames else None
            if r is None:
                n = N ** 3
                s = float((N + 1) ** 2)
                r = orc.run_lobpcg(lambda v: orc.stencil7(v, N, N, N, s), n, m,
                                   tinv=1.0 / np.full(n, 6.0 * s), tol=tol, max_iter=1500,
                                   seed=seed, relative_tol=True, record=False)
        else:
            a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
            r = pk.solve(a, t=pk.jacobi_preconditioner(a),
                         config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed,
                                                relative_tol=True))
        key = r.status if not r.status.startswith("BasisFallback") else "BasisFallback"
        st[key] += 1
        its.append(int(r.iterations_used))
    print(f"N={N} m={m} rel tol={tol:g}: {dict(st)} iterations {min(its)}..{max(its)} "
          f"median {int(np.median(its))}", flush=True)
