"""Time the fused stencil + Gram pass (K1+K5b) at C2 shape over z-chunk
lengths (B2L_SGRAM_ZCHUNK).  Diagnostic only."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0705_2626_b200 import device as dv  # noqa: E402

N, M = 128, 10
n = N ** 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
w = torch.rand((n, M), dtype=torch.float64, device=dev, generator=g)
x = torch.rand((n, M), dtype=torch.float64, device=dev, generator=g)
aw = torch.empty_like(w)
gout = torch.empty((2 * M) * M, dtype=torch.float64, device=dev)
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device=dev)
for zc in [int(a) for a in sys.argv[1:]] or [0]:
    if zc:
        os.environ["B2L_SGRAM_ZCHUNK"] = str(zc)
    else:
        os.environ.pop("B2L_SGRAM_ZCHUNK", None)
    ts = []
    for r in range(25):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dv.stencil7_gram(w, aw, N, N, N, float((N + 1) ** 2), x, M, M, gout)
        b.record()
        torch.cuda.synchronize()
        if r >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"zchunk {zc or 'model'}: median {1e3 * ts[len(ts) // 2]:.1f} us  min {1e3 * ts[0]:.1f} us")
