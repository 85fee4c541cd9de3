"""Corner (kw, kp, kw_next) shapes of every F1 kernel variant, m = 1..16."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_gpu_kernels import test_lobpcg_step_kernel as check  # noqa: E402

dev = torch.device("cuda")
bad = total = 0
for m in range(1, 17):
    for kw in sorted({1, 2, max(1, m // 2), m} & set(range(1, m + 1))):
        for kp in sorted({0, 1, m // 2, m} & set(range(0, m + 1))):
            for kwn in sorted({1, kw}):
                for n in (61, 4099):
                    total += 1
                    try:
                        check(dev, n, m, kw, kp, kwn, (m + kw) % 2 == 0, (m + kp) % 3)
                    except Exception as e:  # noqa: BLE001
                        bad += 1
                        print("FAIL", (n, m, kw, kp, kwn), type(e).__name__, str(e)[:100], flush=True)
print(f"{total - bad} / {total} shapes pass")
