"""Host Rayleigh-Ritz timing (b2l_rayleigh_ritz) on C2-shaped Grams (m = 10,
all columns active, P present).  Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0705_2626_b200.small import NativeRitz  # noqa: E402
from tests.test_rr_native import _case  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10
G1, G2, lam = _case(400, m, m, True, 0)
J = np.arange(m)
nat = NativeRitz(m)
out = nat(m, m, True, G1, G2, lam, J, J, 1e-8)
for _ in range(200):
    nat(m, m, True, G1, G2, lam, J, J, 1e-8)
reps = 2000
t0 = time.perf_counter()
for _ in range(reps):
    nat(m, m, True, G1, G2, lam, J, J, 1e-8)
dt = (time.perf_counter() - t0) / reps
print(f"m={m}: {1e6 * dt:.1f} us per call (incl. ctypes wrapper)")
print("lam", out[0][:4] if isinstance(out, tuple) else out)

if "--dump" in sys.argv:
    # case file for tools/rr_harness.cu: 5 int64 (m, G1 rows, G1 cols, G2 rows,
    # G2 cols) then G1, G2, lam as float64
    d = Path(__file__).resolve().parent / "data"
    d.mkdir(exist_ok=True)
    with open(d / f"case{m}.bin", "wb") as f:
        np.array([m, G1.shape[0], G1.shape[1], G2.shape[0], G2.shape[1]], dtype=np.int64).tofile(f)
        np.ascontiguousarray(G1, dtype=np.float64).tofile(f)
        np.ascontiguousarray(G2, dtype=np.float64).tofile(f)
        np.ascontiguousarray(lam, dtype=np.float64).tofile(f)
    print("wrote", d / f"case{m}.bin")
