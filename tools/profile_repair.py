"""Where a C2 drift-repair step spends its time (cProfile of the Python
path + device time).  Diagnostic only."""
import cProfile
import pstats
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
    prof = cProfile.Profile()
    reps = 0
    while True:
        torch.cuda.synchronize()
        before = r.drift_repairs
        # profile only steps that repair (re-run detection: profile every step, keep repair ones)
        p = cProfile.Profile()
        t0 = time.perf_counter()
        p.enable()
        more = r.step()
        torch.cuda.synchronize()
        p.disable()
        dt = time.perf_counter() - t0
        if r.drift_repairs > before:
            reps += 1
            if rep == 1 and reps == 2:
                print(f"repair step {1e3 * dt:.2f} ms")
                pstats.Stats(p).sort_stats("cumulative").print_stats(25)
        if not more:
            break
