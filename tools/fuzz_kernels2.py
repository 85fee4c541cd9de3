"""Random shapes through the unit checks of the Gram kernels, the plain
stencil, the seeded fill and the split (z-slab) stencil + Gram.  Diagnostic."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests import test_gpu_kernels as tk  # noqa: E402
from tests import test_gpu_slab as ts  # noqa: E402
from paper_0705_2626_b200 import _lib  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dev = torch.device("cuda")
lib = _lib.load()
bad = total = 0
for i in range(count):
    n = int(r.choice([1, 7, 300, 4099, 65537, 120001]))
    cols = tuple(int(v) for v in r.integers(1, 65, 3))
    dims = tuple(int(v) for v in r.integers(1, 45, 3))
    k = int(r.integers(1, 33))
    m = int(r.integers(1, 17))
    kw = int(r.integers(1, m + 1))
    world = int(r.integers(2, 6))
    sdims = (int(r.integers(4, 40)), int(r.integers(4, 40)), int(r.integers(world, 40)))
    cases = [("gram", tk.test_gram_multiblock, (dev, n, cols)),
             ("stencil", tk.test_stencil_bitwise_vs_oracle, (dev, dims, k)),
             ("fill", tk.test_seeded_fill_bitwise,
              (dev, int(r.integers(1, 50000)), m, m + (m & 1), int(r.integers(0, 10 ** 6)),
               int(r.integers(0, 1000)))),
             ("split", ts.test_split_stencil_gram_matches_global,
              (lib, sdims, m + (m & 1), m, kw, world))]
    for name, fn, args in cases:
        total += 1
        try:
            fn(*args)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", name, args[1:], type(e).__name__, str(e)[:120], flush=True)
print(f"{total - bad} / {total} checks pass")
