"""Random (m, kw, kp, kw_next, B, T) shapes through the F1 unit check of
tests/test_gpu_kernels.py (kw_next <= kw <= m, kp <= m).  Diagnostic:
python tools/fuzz_f1.py [count] [seed]"""
import sys
import traceback
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_gpu_kernels import test_lobpcg_step_kernel as check  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dev = torch.device("cuda")
bad = []
for i in range(count):
    m = int(r.integers(1, 17))
    kw = int(r.integers(1, m + 1))
    kp = int(r.integers(0, m + 1))
    kwn = int(r.integers(1, kw + 1))
    n = int(r.choice([257, 3001, 20011, 70001]))
    useb = bool(r.integers(0, 2))
    tmode = int(r.integers(0, 3))
    try:
        check.__wrapped__(dev, n, m, kw, kp, kwn, useb, tmode) if hasattr(check, "__wrapped__") \
            else check(dev, n, m, kw, kp, kwn, useb, tmode)
    except Exception as e:  # noqa: BLE001
        bad.append((n, m, kw, kp, kwn, useb, tmode, type(e).__name__, str(e)[:80]))
        print("FAIL", bad[-1], flush=True)
print(f"{count - len(bad)} / {count} shapes pass")
