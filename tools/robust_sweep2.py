"""Second convergence sweep (16 seeds each): an anisotropic grid with distinct
clustered eigenvalues, a diagonal-B pencil, an unpreconditioned unscaled cube.
`python tools/robust_sweep2.py` on the GPU; `python tools/robust_sweep2.py oracle`
runs the CPU oracle on the same cases (build container).  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ORACLE = len(sys.argv) > 1 and sys.argv[1] == "oracle"
CASES = [  # name, dims, m, jacobi, diag_b seed, scaled, tol
    ("aniso 12x14x16 m=6 tol 1e-8", (12, 14, 16), 6, True, None, False, 1e-8),
    ("diagB 20^3 m=6 tol 1e-6", (20, 20, 20), 6, True, 77, True, 1e-6),
    ("noT 12^3 m=5 tol 1e-7", (12, 12, 12), 5, False, None, False, 1e-7),
    ("aniso 10x20x30 m=8 tol 1e-6 scaled", (10, 20, 30), 8, True, None, True, 1e-6),
]
if ORACLE:
    from oracle import lobpcg_oracle as orc
else:
    import paper_0705_2626_b200 as pk
for name, dims, m, jac, bseed, scaled, tol in CASES:
    nx, ny, nz = dims
    n = nx * ny * nz
    s = float((max(dims) + 1) ** 2) if scaled else 1.0
    bd = np.random.Generator(np.random.PCG64(bseed)).uniform(1.0, 2.0, n) if bseed else None
    st, its = Counter(), []
    for seed in range(16):
        if ORACLE:
            r = orc.run_lobpcg(lambda v: orc.stencil7(v, nx, ny, nz, s if scaled else None), n, m,
                               bdiag=bd, tinv=(1.0 / np.full(n, 6.0 * s)) if jac else None,
                               tol=tol, max_iter=1500, seed=seed, record=False)
        else:
            a = pk.Laplacian3D(dims, scale=s)
            r = pk.solve(a, b=pk.DiagonalOperator(bd) if bd is not None else None,
                         t=pk.jacobi_preconditioner(a) if jac else None,
                         config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
        key = r.status if not r.status.startswith("BasisFallback") else "BasisFallback"
        st[key] += 1
        its.append(int(r.iterations_used))
    print(f"{name}: {dict(st)} iterations {min(its)}..{max(its)} median {int(np.median(its))}",
          flush=True)
