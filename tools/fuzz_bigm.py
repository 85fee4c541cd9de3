"""Large blocks (m = 17..48: the unfused path, LAPACK above a 64 x 64 pencil)
on small cubes with and without diagonal B.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
st = Counter()
for i in range(count):
    N = int(r.integers(10, 21))
    m = int(r.integers(17, 49))
    s = float((N + 1) ** 2)
    useb = bool(r.integers(0, 2))
    seed = int(r.integers(0, 10000))
    n = N ** 3
    bd = r.uniform(1.0, 2.0, n) if useb else None
    a = pk.Laplacian3D((N, N, N), scale=s)
    rep = pk.solve(a, b=pk.DiagonalOperator(bd) if useb else None, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=1e-6, max_iter=1500, seed=seed))
    key = rep.status.split("(")[0]
    st[key] += 1
    x = rep.eigenvectors
    bx = x * bd[:, None] if useb else x
    bad = key == "Failed" or np.abs(x.T @ bx - np.eye(m)).max() > 1e-8
    if rep.all_converged and not useb:
        exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
        bad = bad or np.max(np.abs(rep.eigenvalues - exact) / exact) > 1e-7
    if bad or key == "MaxIterReached":
        print("NOTE", (N, m, useb, seed), rep.status, rep.iterations_used,
              int(rep.converged.sum()), flush=True)
print(dict(st))
