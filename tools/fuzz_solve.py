"""Random small problems through solve(): no exception, no Failed status,
converged pairs match the closed form (identity B) and the residual /
B-orthonormality bounds.  Diagnostic:  python tools/fuzz_solve.py [count] [seed]"""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
st = Counter()
for i in range(count):
    dims = tuple(int(v) for v in r.integers(3, 26, 3))
    n = int(np.prod(dims))
    m = int(r.integers(1, min(16, n // 4) + 1))
    scaled = bool(r.integers(0, 2))
    s = float((max(dims) + 1) ** 2) if scaled else 1.0
    jac = bool(r.integers(0, 2))
    useb = bool(r.integers(0, 4) == 0)
    rel = bool(r.integers(0, 3) == 0)
    tol = float(10.0 ** -r.integers(5, 9)) * (1.0 if rel else s)
    seed = int(r.integers(0, 1000))
    a = pk.Laplacian3D(dims, scale=s)
    bd = r.uniform(0.5, 2.0, n) if useb else None
    cfg = pk.SolverConfig(block_size=m, tol=tol, max_iter=2500, seed=seed, relative_tol=rel)
    tag = (dims, m, scaled, jac, useb, rel, f"{tol:.1e}", seed)
    try:
        rep = pk.solve(a, b=pk.DiagonalOperator(bd) if useb else None,
                       t=pk.jacobi_preconditioner(a) if jac else None, config=cfg)
    except Exception as e:  # noqa: BLE001
        st["exception"] += 1
        print("EXC", tag, type(e).__name__, str(e)[:100], flush=True)
        continue
    key = rep.status.split("(")[0]
    st[key] += 1
    ok = True
    if key == "Failed":
        ok = False
    x = rep.eigenvectors
    bx = x * bd[:, None] if useb else x
    if np.abs(x.T @ bx - np.eye(m)).max() > 1e-8:
        ok = False
    if rep.all_converged and not useb:
        exact = pk.exact_eigenvalues(dims, m, scale=s)
        if np.max(np.abs(rep.eigenvalues - exact) / exact) > 1e-7:
            ok = False
    if not ok:
        print("BAD", tag, rep.status, rep.iterations_used, flush=True)
print(dict(st))
