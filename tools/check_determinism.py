"""Run the C2 solve several times and report bitwise (in)equality of the
final eigenvalues and the first iteration where the Ritz history diverges.
Diagnostic only."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, m, its = 128, 10, int(sys.argv[1]) if len(sys.argv) > 1 else 300
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=its, seed=0)
hists = []
for r in range(3):
    with pk.device_options(return_device=True):
        rep = pk.solve(a, t=pk.jacobi_preconditioner(a), config=cfg)
    h = np.array([e.ritz for e in rep.history])
    hists.append(h)
    print(r, rep.status, hashlib.sha1(h.tobytes()).hexdigest()[:12], rep.eigenvalues[:3], flush=True)
for r in (1, 2):
    d = np.flatnonzero(np.any(hists[r] != hists[0], axis=1))
    print(f"run {r} vs 0: first differing iteration {d[0] if d.size else None}")
