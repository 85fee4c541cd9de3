"""Random shapes through the unit checks of the stencil + Gram, residual and
update kernels (tests/test_gpu_kernels.py).  Diagnostic:
python tools/fuzz_kernels.py [count] [seed]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests import test_gpu_kernels as tk  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dev = torch.device("cuda")
bad = 0
for i in range(count):
    m = int(r.integers(1, 17))
    kw = int(r.integers(1, m + 1))
    kp = int(r.integers(0, m + 1))
    dims = tuple(int(v) for v in r.integers(1, 40, 3))
    cases = [("stencil7_gram", tk.test_stencil7_gram, (dev, dims, m, kw)),
             ("update", tk.test_update_kernel, (dev, m, kw, min(kp, kw))),
             ("residual", tk.test_residual_kernel, (dev, m, int(r.integers(0, 3)), bool(r.integers(0, 2))))]
    for name, fn, args in cases:
        try:
            fn(*args)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", name, args[1:], type(e).__name__, str(e)[:100], flush=True)
print(f"{3 * count - bad} / {3 * count} checks pass")
