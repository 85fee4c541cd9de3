"""Host logic of the GPU solver on CPU stand-ins of the kernels
(tests/emulation.py): proves the Gram bookkeeping, the folded Cholesky-QR
and the repair ladder reproduce the reference before any GPU is involved."""

import numpy as np

from tests.conftest import golden20_band, locks_in_band, trajectory_band_ok
import pytest

from tests.emulation import emulate


@pytest.fixture
def pk(monkeypatch):
    import paper_0705_2626_b200 as pk

    with emulate(monkeypatch):
        yield pk


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))


def test_golden_trajectory_emulated(pk, golden):
    g = golden20_band(golden)
    a = pk.laplacian3d((20, 20, 20))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=10, tol=1e-6, max_iter=200, seed=2))
    ritz = np.array([h.ritz for h in rep.history])
    ok, worst = trajectory_band_ok(ritz, g)
    assert ok, worst
    assert rep.status == "Converged"
    its = g["all_iterations"]
    assert its.min() - 1 <= rep.iterations_used <= its.max() + 1
    ok, lo, hi = locks_in_band(rep.lock_iterations, g["all_locks"])
    assert ok, (rep.lock_iterations, lo, hi)


def test_diag_pencil_emulated(pk, golden):
    g = golden("diag_pencil_n30_m4.npz")
    a = pk.DiagonalOperator(np.arange(1.0, 31.0))
    rep = pk.solve(a, b=pk.DiagonalOperator(g["bdiag"]),
                   config=pk.SolverConfig(block_size=4, tol=1e-10, max_iter=300))
    assert rep.all_converged
    np.testing.assert_allclose(rep.eigenvalues, g["dense_vals"], rtol=1e-10)


def test_diag_b_laplacian_emulated(pk, golden):
    g = golden("lap12_m6_diagB.npz")
    s = float(13 ** 2)
    a = pk.Laplacian3D((12, 12, 12), scale=s)
    rep = pk.solve(a, b=pk.DiagonalOperator(g["bdiag"]), t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=6, tol=1e-6, max_iter=150, seed=0))
    assert rep.status == str(g["status"])
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= 1e-8
