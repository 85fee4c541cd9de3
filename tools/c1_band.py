"""C1@1000 under the reference band's operator perturbations on the GPU,
native loop vs the unfused Python path: iterations, status and where the
basis fallbacks happened.  Diagnostic only."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N = 32
base = float((N + 1) ** 2)
for fused in (True, False):
    rows = []
    for k in (1, -1, 2, -2, 3, -3, 4, -4, 5, 8, -8):
        a = pk.Laplacian3D((N, N, N), scale=base * (1.0 + k * 2.0 ** -52))
        with pk.device_options(fused=fused):
            rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=1000, seed=0))
        fb = [(h.iteration, h.fallbacks) for h in rep.history if h.fallbacks]
        rows.append((k, rep.iterations_used, rep.status, fb[:4], list(rep.lock_iterations)))
    print("fused" if fused else "python", flush=True)
    for r in rows:
        print("  ", r, flush=True)
