"""solve_staged (hard locking) on random small grids: union of the stages'
eigenvalues against the closed form, B-orthonormal union.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 30
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
st = Counter()
for i in range(count):
    dims = tuple(int(v) for v in r.integers(6, 17, 3))
    total = int(r.integers(4, 13))
    blk = int(r.integers(1, 5))
    seed = int(r.integers(0, 1000))
    print('case', dims, total, blk, seed, flush=True)
    a = pk.laplacian3d(dims)
    rep = pk.solve_staged(a, t=pk.jacobi_preconditioner(a), total_wanted=total, stage_block=blk,
                          config=pk.SolverConfig(tol=1e-7, max_iter=600, seed=seed))
    key = rep.status.split("(")[0]
    st[key] += 1
    exact = pk.exact_eigenvalues(dims, total)
    vals = np.sort(rep.eigenvalues)
    x = rep.eigenvectors
    bad = key == "Failed" or np.abs(x.T @ x - np.eye(x.shape[1])).max() > 1e-7
    if rep.all_converged and vals.size == total:
        bad = bad or np.max(np.abs(vals - exact) / exact) > 1e-6
    if bad or key not in ("Converged", "BasisFallback"):
        print("NOTE", (dims, total, blk, seed), rep.status, vals.size, flush=True)
print(dict(st))
