"""pcg_solve / InnerPCGPreconditioner on random small operators against a
plain numpy PCG of the same recurrences (operators.py:341-392).  Diagnostic."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200.pcg import pcg_solve  # noqa: E402
from paper_0705_2626_b200.problems import dense_matrix  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0


def np_pcg(A, tinv, b, steps):
    x = np.zeros_like(b)
    res = b.copy()
    z = tinv * res
    p = z.copy()
    rz = res @ z
    for _ in range(steps):
        ap = A @ p
        alpha = rz / (p @ ap)
        x += alpha * p
        res -= alpha * ap
        z = tinv * res
        rz2 = res @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return x


for i in range(count):
    dims = tuple(int(v) for v in r.integers(2, 11, 3))
    n = int(np.prod(dims))
    a = pk.laplacian3d(dims)
    A = dense_matrix(a)
    steps = int(r.integers(1, 12))
    b = r.standard_normal(n)
    use_t = bool(r.integers(0, 2))
    t = pk.jacobi_preconditioner(a) if use_t else None
    try:
        x = pcg_solve(a, t, b, steps)
        ref = np_pcg(A, (1.0 / 6.0) if use_t else 1.0, b, steps)
        np.testing.assert_allclose(x, ref, rtol=1e-9, atol=1e-11 * np.abs(ref).max())
        # the block preconditioner on k columns = column-wise pcg_solve
        k = int(r.integers(1, 7))
        Bk = r.standard_normal((n, k))
        T = pk.inner_pcg_preconditioner(a, t, steps=steps)
        Y = T(Bk)
        for j in range(k):
            np.testing.assert_allclose(Y[:, j], np_pcg(A, (1.0 / 6.0) if use_t else 1.0, Bk[:, j], steps),
                                       rtol=1e-9, atol=1e-11 * np.abs(Y[:, j]).max())
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL", dims, steps, use_t, type(e).__name__, str(e)[:150], flush=True)
print(f"{count - bad} / {count} cases pass")
