"""Per-step device time of the C2 run (CUDA events around each step on the
launching stream) with the steps that ran a drift repair marked.
Diagnostic only: python tools/step_times.py [N m steps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 120
a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
for rep in range(2):
    run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a),
                       config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=300, seed=0))
    evs, marks = [], []
    for i in range(steps):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append(e)
        r0 = run.drift_repairs
        if not run.step():
            break
        marks.append(run.drift_repairs > r0)
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    evs.append(e)
    torch.cuda.synchronize()
    dt = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)])
    marks = np.array(marks[:len(dt)])
    rep_idx = np.flatnonzero(marks)
    normal = dt[5:][~marks[5:]]
    print(f"pass {rep}: normal step median {np.median(normal):.4f} ms, mean {normal.mean():.4f}; "
          f"repair steps {[(int(i), round(float(dt[i]), 4), round(float(dt[i + 1]), 4)) for i in rep_idx]}")
