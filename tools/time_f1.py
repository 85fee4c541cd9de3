"""CUDA-event timing of F1 (b2l_lobpcg_step) alone on random full blocks:
N^3 rows, block m, 30 launches after 5 warm-ups, ping-ponged outputs (inputs
far exceed L2).  Prints ms per launch and the algorithmic GB/s 8n(6m+5k).
Diagnostic only:  python tools/time_f1.py [N m]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0705_2626_b200 import device as dv  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = N ** 3
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
ld = m + (m & 1)
blk = lambda: torch.randn((n, ld), dtype=torch.float64, device=dev, generator=g)  # noqa: E731
X, AX, P, AP, W, AW = (blk() for _ in range(6))
outs = [torch.empty((n, ld), dtype=torch.float64, device=dev) for _ in range(5)]
r = np.random.default_rng(0)
coef = torch.from_numpy(r.standard_normal(3 * m * m) * 0.3).to(dev)
lam = torch.from_numpy(r.uniform(1, 5, m)).to(dev)
pcols = torch.arange(m, dtype=torch.int32, device=dev)
wpos = torch.arange(m, dtype=torch.int32, device=dev)
red = torch.empty(2 * m + 3 * m * 4 * m, dtype=torch.float64, device=dev)


def launch():
    dv.lobpcg_step(n, m, X, AX, W, AW, m, P, AP, m, pcols, coef, outs[0], outs[1], outs[2],
                   outs[3], lam, None, 1, 0.25, None, wpos, m, outs[4], True, red)


for _ in range(5):
    launch()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
by = 8.0 * n * 11 * m
print(f"F1 N={N} m={m}: median {np.median(ts):.4f} ms  min {ts.min():.4f}  "
      f"{by / np.median(ts) / 1e6:.0f} GB/s")
