"""Find which buffer differs between the first and the second C2 run of a
process after each of the first steps.  Diagnostic only."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200 import lobpcg as lb  # noqa: E402

N, m = 128, 10
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
T = pk.jacobi_preconditioner(a)
cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=20, seed=0)


def snap(r, tag):
    torch.cuda.synchronize()
    d = {}
    for nm in ("X", "AX", "P", "AP", "X2", "AX2", "P2", "AP2", "AWbuf", "red", "g2"):
        d[nm] = getattr(r, nm).detach().cpu().numpy().copy()
    d["W0"] = r.Wbufs[0].cpu().numpy().copy()
    d["W1"] = r.Wbufs[1].cpu().numpy().copy()
    d["h_red"] = r.h_red.numpy().copy()
    d["h_g2"] = r.h_g2.numpy().copy()
    d["lam"] = np.array(r.lam, dtype=float).copy()
    return d


runs = []
for k in range(2):
    r = lb.LOBPCGRun(a, t=T, config=cfg)
    snaps = [snap(r, "init")]
    for i in range(3):
        r.step()
        snaps.append(snap(r, f"step{i}"))
    runs.append(snaps)
    del r
for i, (s0, s1) in enumerate(zip(*runs)):
    diffs = [k for k in s0 if not np.array_equal(s0[k], s1[k], equal_nan=True)]
    print(f"after {'init' if i == 0 else 'step' + str(i - 1)}: differing {diffs}", flush=True)
    for k in diffs[:6]:
        a0, a1 = s0[k].ravel(), s1[k].ravel()
        idx = np.flatnonzero(~((a0 == a1) | (np.isnan(a0) & np.isnan(a1))))
        print(f"   {k}: {idx.size} entries differ, first at {idx[:5]}, vals {a0[idx[:3]]} vs {a1[idx[:3]]}")
