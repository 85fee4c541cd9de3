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


def golden20_band(golden):
    """The 20^3 golden case with its full reference band: the CSV run, the
    coherent-scaling runs (golden_20cubed_m10_jacobi_seed2.npz) and the
    rounding-noise runs (golden_20cubed_band.npz: operator outputs and Ritz
    coefficients perturbed by +-1 ulp; make_golden.py --band20)."""
    import numpy as np

    g = golden("golden_20cubed_m10_jacobi_seed2.npz")
    b = golden("golden_20cubed_band.npz")
    n = min(g["pert_ritz"].shape[1], b["pert_ritz"].shape[1])
    out = dict(g)
    out["pert_ritz"] = np.concatenate([g["pert_ritz"][:, :n], b["pert_ritz"][:, :n]])
    out["all_iterations"] = np.concatenate([[int(g["iterations_used"])], g["pert_iterations"],
                                            b["pert_iterations"]])
    out["all_locks"] = np.vstack([g["lock_iterations"], g["pert_locks"], b["pert_locks"]])
    return out


def locks_in_band(locks, all_locks, slack=0.1):
    """Lock iterations of degenerate clusters are not a stable observable
    (two basins, long tails under rounding noise): each column's lock
    iteration must lie within the reference band widened by `slack`
    (relative) + 1."""
    import numpy as np

    lo = np.floor(all_locks.min(0) * (1.0 - slack)) - 1
    hi = np.ceil(all_locks.max(0) * (1.0 + slack)) + 1
    return bool(np.all((locks >= lo) & (locks <= hi))), lo, hi
