"""Re-run bench.py's timed region (C2, warm-up 5, steps 5..300) and report the
slowest steps (host time between step returns; each native step synchronises
at its start, so this tracks the device).  Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N, M = 128, 10
s = float((N + 1) ** 2)
A = pk.Laplacian3D((N,) * 3, scale=s)
x0 = np.random.Generator(np.random.PCG64(0)).uniform(-1.0, 1.0, size=(N ** 3, M))
T = pk.jacobi_preconditioner(A)
cfg = pk.SolverConfig(block_size=M, tol=1e-8, max_iter=300, seed=0)
run = pk.LOBPCGRun(A, t=T, x0=x0, config=cfg)
sampler = None
if len(sys.argv) > 1 and sys.argv[1] == "nvml":
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from bench import ClockSampler  # noqa: E402
    sampler = ClockSampler(0)
for _ in range(5):
    run.step()
torch.cuda.synchronize()
if sampler:
    sampler.__enter__()
ts = [time.perf_counter()]
reps = []
for _ in range(295):
    before = run.drift_repairs
    run.step()
    ts.append(time.perf_counter())
    reps.append(run.drift_repairs > before)
torch.cuda.synchronize()
if sampler:
    sampler.__exit__(None, None, None)
dt = np.diff(ts) * 1e3
order = np.argsort(dt)[::-1][:6]
print(f"total {sum(dt):.1f} ms; slowest steps (index, ms, repair): " +
      ", ".join(f"({i + 5}, {dt[i]:.2f}, {reps[i]})" for i in order), flush=True)
