"""Random small problems through the callback / constraint / inner-PCG paths
of solve(): no exception, sane status, B-orthonormal result.  Diagnostic."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
st = Counter()
for i in range(count):
    dims = tuple(int(v) for v in r.integers(4, 15, 3))
    n = int(np.prod(dims))
    m = int(r.integers(1, 9))
    mode = int(r.integers(0, 5))
    seed = int(r.integers(0, 1000))
    a = pk.laplacian3d(dims)
    cfg = pk.SolverConfig(block_size=m, tol=1e-6, max_iter=800, seed=seed)
    tag = (dims, m, mode, seed)
    try:
        kw = {}
        bmat = None
        if mode == 0:      # generic B callback (tridiagonal SPD)
            def b(v):
                y = 3.0 * v
                y[1:] -= v[:-1]
                y[:-1] -= v[1:]
                return y
            kw["b"] = b
            bmat = b
        elif mode == 1:    # generic T callback
            kw["t"] = lambda w: w / 6.0
        elif mode == 2:    # inner PCG preconditioner
            kw["t"] = pk.inner_pcg_preconditioner(a, None, steps=int(r.integers(1, 6)))
        elif mode == 3:    # constraints
            nc = int(r.integers(1, 7))
            kw["y"] = pk.Constraints.from_basis(r.standard_normal((n, nc)))
            kw["t"] = pk.jacobi_preconditioner(a)
        else:              # MatrixFreeOperator harness around the stencil
            L = pk.laplacian3d(dims)
            a = pk.MatrixFreeOperator(n, lambda v: 2.5 * L(v), spd=True,
                                      diag=np.full(n, 15.0))
            kw["t"] = pk.jacobi_preconditioner(a)
        rep = pk.solve(a, config=cfg, **kw)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        st["exception"] += 1
        print("EXC", tag, type(e).__name__, str(e)[:120], flush=True)
        continue
    key = rep.status.split("(")[0]
    st[key] += 1
    st[(mode, key)] += 1
    x = rep.eigenvectors
    if bmat is not None:
        bx = bmat(torch.from_numpy(x).cuda()).cpu().numpy()
    else:
        bx = x
    if key == "Failed" or np.abs(x.T @ bx - np.eye(m)).max() > 1e-7:
        print("BAD", tag, rep.status, rep.iterations_used, flush=True)
print({k: v for k, v in st.items() if isinstance(k, str)})
print(sorted((k, v) for k, v in st.items() if not isinstance(k, str)))
