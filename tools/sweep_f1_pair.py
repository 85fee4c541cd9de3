"""Every (m, kw, kp, kw_next) of the F1 pair kernel (m = 9, 10; kw_next <= kw)
through the unit check.  Diagnostic."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_gpu_kernels import test_lobpcg_step_kernel as check  # noqa: E402

dev = torch.device("cuda")
bad = total = 0
for m in (9, 10):
    for kw in range(1, m + 1):
        for kp in range(0, m + 1):
            for kwn in sorted({1, kw // 2 or 1, kw}):
                total += 1
                try:
                    check(dev, 2003 + 7 * kw + kp, m, kw, kp, kwn, (kw + kp) % 2 == 0, (kw + kp) % 3)
                except Exception as e:  # noqa: BLE001
                    bad += 1
                    print("FAIL", (m, kw, kp, kwn), type(e).__name__, str(e)[:100], flush=True)
print(f"{total - bad} / {total} shapes pass")
