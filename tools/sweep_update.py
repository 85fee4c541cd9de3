"""K6 update over (m, kw, kp) corners incl. W blocks wider than m (constraint
projections: kw = number of constraints).  Diagnostic."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_gpu_kernels import test_update_kernel as check  # noqa: E402

dev = torch.device("cuda")
bad = total = 0
for m in (1, 2, 3, 5, 8, 9, 10, 13, 16, 17, 24, 33, 40, 64):
    for kw in sorted({1, max(1, m // 2), m, m + 3, 2 * m + 1, 70, 100}):
        for kp in sorted({0, 1, m // 2, m}):
            total += 1
            try:
                check(dev, m, kw, kp)
            except Exception as e:  # noqa: BLE001
                bad += 1
                print("FAIL", (m, kw, kp), type(e).__name__, str(e)[:100], flush=True)
print(f"{total - bad} / {total} shapes pass")
