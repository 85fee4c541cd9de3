#!/usr/bin/env python3
"""Full-size matched-iteration fixtures for the BASELINE configs too big for
the build container (62 GiB RAM): C4 (464^3, m=8, Jacobi) and C5 (192^3,
m=64, diagonal B, Jacobi), from the CPU oracle port (oracle/lobpcg_oracle.py,
pinned bit-exact to the reference's golden trajectory) run on the GPU host
(196 GiB, 16 cores):

    gpurun --timeout 3600 -- 'python tests/golden/make_bigconfigs.py gpurun_out/'

then copy gpurun_out/{c4,c5}_*.npz to tests/golden/.  C3 (256^3, m=16) comes
from the REAL reference in the build container (make_golden.py --full-size).

Test infrastructure only (tests/golden/); the product never imports oracle/.
Harness as SURVEY 8c: A = s L7, s = (N+1)^2, Jacobi 1/(6s), X0 = PCG64(0)
uniform(-1, 1), B = diag(U[1,2]) from PCG64(1000).
"""

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import lobpcg_oracle as orc  # noqa: E402


def record(r):
    return dict(
        eigenvalues=r.eigenvalues, residual_norms=r.residual_norms,
        iterations_used=np.int64(r.iterations_used), converged=r.converged,
        lock_iterations=r.lock_iterations, status=np.array(r.status),
        basis_fallbacks=np.int64(r.basis_fallbacks), hist_ritz=np.array(r.hist_ritz),
        hist_resid=np.array(r.hist_resid), hist_active=np.array(r.hist_active),
        drift_repairs=np.int64(r.drift_repairs))


def main(out):
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    which = os.environ.get("BIG", "c5,c4").split(",")
    t0 = time.time()
    if "c5" in which:
        r = orc.laplacian_case(192, 64, bseed=1000, tol=1e-6, max_iter=5, seed=0)
        np.savez_compressed(out / "c5_192cubed_m64_diagB_5it.npz", **record(r))
        print(f"C5@5 {r.status} {time.time() - t0:.1f} s", flush=True)
    if "c4" in which:
        r = orc.laplacian_case(464, 8, tol=1e-6, max_iter=5, seed=0)
        np.savez_compressed(out / "c4_464cubed_m8_5it.npz", **record(r))
        print(f"C4@5 {r.status} {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "tests" / "golden"))
