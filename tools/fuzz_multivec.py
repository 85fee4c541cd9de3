"""multivec API (gram / multiply / tri_solve_right / column_norms) on random
shapes against numpy.  Diagnostic."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0705_2626_b200 import multivec as mv  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 80
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = total = 0


def check(name, fn):
    global bad, total
    total += 1
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL", name, type(e).__name__, str(e)[:120], flush=True)


for i in range(count):
    n = int(r.choice([1, 5, 333, 4099, 30011]))
    kx, ky = int(r.integers(1, 65)), int(r.integers(1, 65))
    x, y = r.standard_normal((n, kx)), r.standard_normal((n, ky))
    c = r.standard_normal((kx, ky))
    tri = np.triu(r.standard_normal((kx, kx))) + kx * np.eye(kx)

    def f_gram():
        np.testing.assert_allclose(mv.gram(x, y), x.T @ y, rtol=1e-11, atol=1e-11 * n)

    def f_mul():
        np.testing.assert_allclose(mv.multiply(x, c), x @ c, rtol=1e-11, atol=1e-11 * kx)

    def f_tri():
        z = mv.tri_solve_right(x, tri)
        np.testing.assert_allclose(z @ tri, x, rtol=0, atol=1e-10 * max(1.0, np.abs(x).max()))

    def f_norm():
        np.testing.assert_allclose(mv.column_norms(x), np.linalg.norm(x, axis=0), rtol=1e-12)

    check(f"gram {n} {kx} {ky}", f_gram)
    check(f"multiply {n} {kx}x{ky}", f_mul)
    check(f"tri {n} {kx}", f_tri)
    check(f"norms {n} {kx}", f_norm)
print(f"{total - bad} / {total} checks pass")
