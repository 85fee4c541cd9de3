import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(GOLDEN / name, allow_pickle=False))

    return load


def trajectory_band_ok(ritz, g, floor=1e-8, factor=10.0, window=5):
    """Per-iteration Ritz parity against the golden trajectory.

    The reference's own trajectory is chaotic inside degenerate clusters: the
    golden fixture holds the reference re-run with the operator perturbed by
    1-2 ulp (``pert_ritz``, several runs).  The allowed relative deviation at
    iteration i is max(floor, factor * band_i), band_i being the largest
    perturbation-induced deviation within +-window iterations.
    Returns (ok, worst ratio of deviation to allowance)."""
    import numpy as np

    ref = g["csv_ritz"]
    pert = g["pert_ritz"]
    nit = min(len(ritz), len(ref), pert.shape[1])
    dev = np.abs(ritz[:nit] - ref[:nit]) / np.abs(ref[:nit])
    band = (np.abs(pert[:, :nit] - ref[None, :nit]) / np.abs(ref[None, :nit])).max(axis=(0, 2))
    env = np.array([band[max(0, i - window):i + window + 1].max() for i in range(nit)])
    allowed = np.maximum(floor, factor * env)[:, None]
    return bool(np.all(dev <= allowed)), float((dev / allowed).max())
