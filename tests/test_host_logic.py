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


def test_staged_walk_emulated(pk, golden):
    """solve_staged + constraint projection host logic on CPU stand-ins."""
    g = golden("staged_walk.npz")
    rep = pk.solve_staged(pk.DiagonalOperator(np.arange(1.0, 11.0)), total_wanted=6, stage_block=2,
                          config=pk.SolverConfig(tol=1e-10, max_iter=100))
    assert rep.ok and rep.all_converged and rep.status == str(g["status"])
    np.testing.assert_allclose(rep.eigenvalues, np.arange(1.0, 7.0), rtol=0.0, atol=1e-8)
    its = np.array([r.iterations_used for r in rep.stages])
    assert np.all(np.abs(its - g["stage_iterations"]) <= 2), its
    assert sorted({h.stage for h in rep.history}) == [0, 1, 2]


def test_constrained_pencil_emulated(pk, golden):
    g = golden("staged_pencil.npz")
    b = pk.DiagonalOperator(g["bdiag"])
    cons = pk.Constraints.from_basis(g["ybasis"], b)
    rep = pk.solve(pk.DiagonalOperator(np.arange(1.0, 31.0)), b=b, y=cons,
                   config=pk.SolverConfig(block_size=2, tol=1e-10, max_iter=300))
    assert rep.all_converged
    np.testing.assert_allclose(rep.eigenvalues, g["dense_vals"][2:4], rtol=1e-9)
    assert max(h.constraint_violation for h in rep.history) <= 1e-8


def test_pcg_emulated(pk, golden):
    """Host control of the column-batched PCG (device scalars, stop flags)
    on CPU stand-ins, against the reference's pcg_solve vectors."""
    g = golden("pcg_cases.npz")
    L = pk.laplacian3d((8, 9, 7))
    for name, m in (("none", None), ("jacobi", pk.jacobi_preconditioner(L))):
        for it in (1, 5, 30):
            x = pk.pcg_solve(L, m, g["b"], it, 0.0)
            ref = g[f"x_{name}_{it}"]
            np.testing.assert_allclose(x, ref, rtol=0, atol=1e-10 * np.abs(ref).max())
        x = pk.pcg_solve(L, m, g["b"], 200, 1e-6)
        np.testing.assert_allclose(x, g[f"x_{name}_rtol"], rtol=0,
                                   atol=1e-10 * np.abs(g[f"x_{name}_rtol"]).max())


def _tb_tridiag(v):
    y = 3.0 * v
    y[1:] -= v[:-1]
    y[:-1] -= v[1:]
    return y


def test_generic_b_emulated(pk, golden):
    """A non-diagonal B callback: BX / BW / BP carried by recurrence through
    the standalone kernels (host bookkeeping on the CPU stand-ins)."""
    g = golden("genb_tri8.npz")
    N = 8
    a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
    calls = []

    def b(v):
        calls.append(tuple(v.shape))
        return _tb_tridiag(v.clone())

    rep = pk.solve(a, b=b, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=4, tol=1e-8, max_iter=300, seed=0))
    assert rep.status == str(g["status"])
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 1
    np.testing.assert_allclose(rep.eigenvalues, g["dense_vals"], rtol=1e-10)
    # b sees (n, |J|) blocks only, like the reference (lobpcg.py:396, :476)
    assert all(s[0] == N ** 3 and 1 <= s[1] <= 4 for s in calls)
    actives = [int(h.active.sum()) for h in rep.history[:-1]]
    assert [c[1] for c in calls[1:]] == actives[:len(calls) - 1]
