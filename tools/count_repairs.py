"""Drift repairs (lobpcg.py:419-428) in the C2 run and the time they take.
Diagnostic only."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200 import lobpcg as lb  # noqa: E402

N, m = 128, 10
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
T = pk.jacobi_preconditioner(a)
cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=300, seed=0)
for rep in range(2):
    r = lb.LOBPCGRun(a, t=T, config=cfg)
    times = []
    reps_before = 0
    while True:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        more = r.step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        times.append((dt, r.drift_repairs > reps_before))
        reps_before = r.drift_repairs
        if not more:
            break
    rep_t = [t for t, d in times if d]
    norm_t = sorted(t for t, d in times if not d)
    print(f"run {rep}: {r.drift_repairs} drift repairs in {r.it} iterations; repair steps "
          f"{[round(1e3 * t, 2) for t in rep_t]} ms; median normal step {1e3 * norm_t[len(norm_t) // 2]:.3f} ms "
          f"(synchronised per step)")
