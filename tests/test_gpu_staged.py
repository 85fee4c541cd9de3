"""Hard locking on the GPU: Constraints, apply_constraints
and solve_staged against the reference's own tests (test_lobpcg.py:385-471,
test_acceptance.py:160-178) and the golden fixtures the real reference
produced for them (tests/golden/staged_*.npz, make_golden.py --staged)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_0705_2626_b200 as pk

    return pk


def diag_range(pk, n):
    return pk.DiagonalOperator(np.arange(1.0, n + 1.0))


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))


def test_apply_constraints_projects(pk):
    r = np.random.default_rng(3)
    n = 5000
    d = r.uniform(0.5, 2.0, n)
    b = pk.DiagonalOperator(d)
    y = r.standard_normal((n, 7))
    x = r.standard_normal((n, 5))
    cons = pk.Constraints.from_basis(y, b)
    assert cons.count == 7
    got = pk.apply_constraints(x, cons)
    by = d[:, None] * y
    ref = x - y @ np.linalg.solve(y.T @ by, by.T @ x)
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    assert np.abs(by.T @ got).max() <= 1e-9 * np.abs(x).max() * n ** 0.5
    # degenerate basis: NotSPD, as the reference
    with pytest.raises(pk.NotSPD):
        pk.Constraints.from_basis(np.hstack([y, y[:, :1]]), b)


def test_constrained_generalized_pencil(pk, golden):
    g = golden("staged_pencil.npz")
    a = diag_range(pk, 30)
    b = pk.DiagonalOperator(g["bdiag"])
    cons = pk.Constraints.from_basis(g["ybasis"], b)
    rep = pk.solve(a, b=b, y=cons, config=pk.SolverConfig(block_size=2, tol=1e-10, max_iter=300))
    assert rep.all_converged and rep.status == str(g["status"])
    np.testing.assert_allclose(rep.eigenvalues, g["dense_vals"][2:4], rtol=1e-9, atol=0.0)
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 2
    for h in rep.history:
        assert h.constraint_violation is not None and h.constraint_violation <= 1e-8


def test_exact_constraints_shift_the_floor(pk, golden):
    g = golden("staged_floor.npz")
    cons = pk.Constraints.from_basis(np.eye(10)[:, :3])
    rep = pk.solve(diag_range(pk, 10), y=cons,
                   config=pk.SolverConfig(block_size=2, tol=1e-10, max_iter=100))
    assert rep.all_converged
    assert rep.status.startswith("BasisFallback") == str(g["status"]).startswith("BasisFallback")
    np.testing.assert_allclose(rep.eigenvalues, [4.0, 5.0], rtol=0.0, atol=1e-9)
    for h in rep.history:
        assert h.ritz.min() >= 4.0 - 1e-8


def test_staged_walks_the_spectrum(pk, golden):
    g = golden("staged_walk.npz")
    rep = pk.solve_staged(diag_range(pk, 10), total_wanted=6, stage_block=2,
                          config=pk.SolverConfig(tol=1e-10, max_iter=100))
    assert rep.ok and rep.all_converged and rep.status == str(g["status"])
    np.testing.assert_allclose(rep.eigenvalues, np.arange(1.0, 7.0), rtol=0.0, atol=1e-8)
    assert len(rep.stages) == 3
    assert rep.iterations_used == sum(r.iterations_used for r in rep.stages)
    assert sorted({h.stage for h in rep.history}) == [0, 1, 2]
    its = np.array([r.iterations_used for r in rep.stages])
    assert np.all(np.abs(its - g["stage_iterations"]) <= 2), its


def test_staged_validation(pk):
    a = diag_range(pk, 6)
    with pytest.raises(ValueError):
        pk.solve_staged(a, total_wanted=4, stage_block=0)
    with pytest.raises(ValueError):
        pk.solve_staged(a, total_wanted=1, stage_block=2)
    with pytest.raises(ValueError):   # m > n - ncons (lobpcg.py:377-381)
        pk.solve(a, y=pk.Constraints.from_basis(np.eye(6)[:, :5]),
                 config=pk.SolverConfig(block_size=2))


def test_staged_union_is_b_orthonormal(pk, golden):
    g = golden("staged_union.npz")
    b = pk.DiagonalOperator(g["bdiag"])
    rep = pk.solve_staged(diag_range(pk, 20), b=b, total_wanted=6, stage_block=3,
                          config=pk.SolverConfig(tol=1e-10, max_iter=200))
    assert rep.all_converged
    v = rep.eigenvectors
    gm = v.T @ (g["bdiag"][:, None] * v)
    assert np.abs(gm - np.eye(6)).max() <= 1e-8
    np.testing.assert_allclose(rep.eigenvalues, g["eigenvalues"], rtol=1e-9)


def test_staged_stall_propagates_status(pk, golden):
    g = golden("staged_stall.npz")
    rep = pk.solve_staged(pk.laplacian3d((6, 6, 6)), total_wanted=4, stage_block=2,
                          config=pk.SolverConfig(tol=1e-12, max_iter=2))
    assert rep.status == str(g["status"]) == "MaxIterReached"
    assert not rep.all_converged
    assert len(rep.stages) == 1


def test_criterion_5_staged_hard_locking(pk, golden):
    """10^3, 10 eigenpairs in two stages of 5 (test_acceptance.py:160-178)."""
    g = golden("staged_crit5.npz")
    L = pk.laplacian3d((10, 10, 10))
    rep = pk.solve_staged(L, t=pk.jacobi_preconditioner(L), total_wanted=10, stage_block=5,
                          config=pk.SolverConfig(tol=1e-6, max_iter=300))
    assert rep.ok and rep.all_converged
    exact = pk.exact_eigenvalues((10, 10, 10), 10)
    assert rel(rep.eigenvalues, exact).max() <= 1e-6
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= 1e-8
    second = [h for h in rep.history if h.stage == 1]
    assert second
    for h in second:
        assert h.constraint_violation is not None and h.constraint_violation <= 1e-8
    its = np.array([r.iterations_used for r in rep.stages])
    assert np.all(np.abs(its - g["stage_iterations"]) <= np.maximum(2, 0.1 * g["stage_iterations"]))


def test_staged_scaled_laplacian(pk, golden):
    g = golden("staged_lap16.npz")
    s = float(17 ** 2)
    A = pk.Laplacian3D((16, 16, 16), scale=s)
    rep = pk.solve_staged(A, t=pk.jacobi_preconditioner(A), total_wanted=8, stage_block=4,
                          config=pk.SolverConfig(tol=1e-6, max_iter=300, seed=5))
    assert rep.status == str(g["status"])
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= 1e-8
    exact = pk.exact_eigenvalues((16, 16, 16), 8, scale=s)
    assert rel(rep.eigenvalues, exact).max() <= 1e-8
    its = np.array([r.iterations_used for r in rep.stages])
    assert np.all(np.abs(its - g["stage_iterations"]) <= np.maximum(2, 0.1 * g["stage_iterations"]))
