"""Cubic grids (degenerate spectra), random m / tol / seed: status counts and
any Failed / non-orthonormal / inaccurate result.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
st = Counter()
slow = []
for i in range(count):
    N = int(r.integers(8, 25))
    m = int(r.integers(3, 17))
    s = float((N + 1) ** 2)
    rel = bool(r.integers(0, 2))
    tol = float(10.0 ** -r.integers(6, 10)) * (1.0 if rel else 1.0)
    if not rel:
        tol = max(tol, 1e-8)
    seed = int(r.integers(0, 10000))
    a = pk.Laplacian3D((N, N, N), scale=s)
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=tol, max_iter=3000, seed=seed,
                                          relative_tol=rel))
    key = rep.status.split("(")[0]
    st[key] += 1
    x = rep.eigenvectors
    bad = key == "Failed" or np.abs(x.T @ x - np.eye(m)).max() > 1e-8
    if rep.all_converged:
        exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
        bad = bad or np.max(np.abs(rep.eigenvalues - exact) / exact) > 1e-7
    if bad or key == "MaxIterReached":
        print("NOTE", (N, m, rel, f"{tol:.0e}", seed), rep.status, rep.iterations_used,
              int(rep.converged.sum()), flush=True)
print(dict(st))
