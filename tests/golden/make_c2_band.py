#!/usr/bin/env python3
"""The C2 trajectory band: the oracle port (bit-exact to the reference on the
golden trajectory) re-run on C2 (128^3, m=10, Jacobi, tol 1e-8, 300 it) with
its operator scaled by (1 + k 2^-52), k = +-1 -- the reference's own
sensitivity of the Ritz trajectory inside the degenerate clusters (1+3+3+3)
of this spectrum.  ~8 min per run on the GPU host's 16 cores:

    gpurun --timeout 3000 -- 'python tests/golden/make_c2_band.py gpurun_out/'

then copy gpurun_out/c2_band.npz to tests/golden/.  Test infrastructure only.
"""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import lobpcg_oracle as orc  # noqa: E402


def main(out):
    N, m = 128, 10
    n = N ** 3
    s = float((N + 1) ** 2)
    ritz, its, stat = [], [], []
    for k in (1, -1):
        t0 = time.time()
        s1 = s * (1.0 + k * 2.0 ** -52)
        r = orc.run_lobpcg(lambda v, s1=s1: orc.stencil7(v, N, N, N, s1), n, m,
                           tinv=1.0 / np.full(n, 6.0 * s1), tol=1e-8, max_iter=300, seed=0)
        ritz.append(np.array(r.hist_ritz))
        its.append(r.iterations_used)
        stat.append(r.status)
        print(k, r.status, r.iterations_used, r.drift_repairs, f"{time.time() - t0:.0f} s", flush=True)
    Path(out).mkdir(parents=True, exist_ok=True)
    np.savez_compressed(Path(out) / "c2_band.npz", ulps=np.array([1, -1]), pert_ritz=np.stack(ritz),
                        iterations=np.array(its), status=np.array(stat))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "tests" / "golden"))
