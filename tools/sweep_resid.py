"""Residual kernel over every m = 1..64, T mode and B mode; plain stencil up
to 64 columns.  Diagnostic."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests import test_gpu_kernels as tk  # noqa: E402

dev = torch.device("cuda")
bad = total = 0
for m in range(1, 65):
    for tmode in (0, 1, 2):
        for useb in (False, True):
            total += 1
            try:
                tk.test_residual_kernel(dev, m, tmode, useb)
            except Exception as e:  # noqa: BLE001
                bad += 1
                print("FAIL resid", (m, tmode, useb), type(e).__name__, str(e)[:100], flush=True)
for k in range(1, 65):
    total += 1
    try:
        tk.test_stencil_bitwise_vs_oracle(dev, (11 + k % 5, 9, 13), k)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL stencil", k, type(e).__name__, str(e)[:100], flush=True)
print(f"{total - bad} / {total} pass")
