"""Time the pieces of the drift-repair path on their first and second
execution in a fresh process (C2 shapes).  Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200 import device as dv  # noqa: E402
from paper_0705_2626_b200 import lobpcg as lb  # noqa: E402
from paper_0705_2626_b200.small import scaled_cholesky, sym_eig  # noqa: E402

N, m = 128, 10
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
T = pk.jacobi_preconditioner(a)
cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=300, seed=0)
r = lb.LOBPCGRun(a, t=T, config=cfg)
for _ in range(3):
    r.step()
torch.cuda.synchronize()


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return out


for rep in range(2):
    print(f"-- pass {rep}")
    gxx = t("gram_xx", r._gram_xx)
    _, minv = t("scaled_cholesky", lambda: scaled_cholesky(gxx))
    Md = t("to_device", lambda: dv.to_device(minv, r.dev))
    t("update (rotation)", lambda: dv.update(r.n, m, r.X, r.AX, Md, r.X2, r.AX2))
    g = t("gram X^T AX", lambda: r._gram(r.n, [(r.X, m)], [(r.AX, m)], pair_mode=lb._UPPER))
    gh = t("to_host", lambda: dv.to_host(g))
    t("sym_eig", lambda: sym_eig(gh))
