"""Solver behaviours the reference's own suite pins (pkg/tests/test_lobpcg.py)
that the trajectory tests do not touch: report / status bookkeeping, the
printed summary, honest failure, history switches, constraint validation.
Each case names the reference test it restates."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    assert torch.cuda.is_available()
    import paper_0705_2626_b200 as pk

    return pk


def ramp(pk, n):
    """diag(1..n): eigenpairs known exactly."""
    return pk.DiagonalOperator(np.arange(1.0, n + 1.0))


def test_status_string_follows_fallback_count(pk):
    # test_solve_status_string_matches_fallback_count (test_lobpcg.py)
    rep = pk.solve(ramp(pk, 10), config=pk.SolverConfig(block_size=3, tol=1e-10, max_iter=100))
    want = f"BasisFallback({rep.basis_fallbacks})" if rep.basis_fallbacks else "Converged"
    assert rep.status == want
    np.testing.assert_allclose(rep.eigenvalues, [1.0, 2.0, 3.0], rtol=1e-9)


def test_block_larger_than_free_dimension(pk):
    # test_solve_block_size_exceeding_free_dimension: n = 4, two constraints
    cons = pk.Constraints.from_basis(np.eye(4)[:, :2])
    with pytest.raises(ValueError):
        pk.solve(ramp(pk, 4), y=cons, config=pk.SolverConfig(block_size=3))


def test_printed_summary(pk, capsys):
    # test_verbosity_zero_is_silent / test_verbosity_one_prints_summary
    pk.solve(ramp(pk, 6), config=pk.SolverConfig(block_size=2, tol=1e-8))
    assert capsys.readouterr().out == ""
    pk.solve(ramp(pk, 6), config=pk.SolverConfig(block_size=2, tol=1e-8, verbosity=1))
    out = capsys.readouterr().out
    assert "[blockeig]" in out and "converged" in out


def test_unreachable_tolerance_is_reported_as_failure(pk):
    # test_unreachable_tolerance_fails_honestly: m = n makes the first
    # Rayleigh-Ritz step exact, the residual block is roundoff, 1e-30 is never
    # met and the basis degenerates
    rep = pk.solve(ramp(pk, 3), config=pk.SolverConfig(block_size=3, tol=1e-30, max_iter=50))
    assert rep.status == "Failed(BasisDegeneracy)"
    assert not rep.ok and not rep.converged.any()


def test_max_iterations_reported(pk):
    # test_max_iterations_reported
    a = pk.laplacian3d((6, 6, 6))
    rep = pk.solve(a, config=pk.SolverConfig(block_size=3, tol=1e-12, max_iter=4))
    assert rep.status == "MaxIterReached"
    assert rep.iterations_used == 4 and len(rep.history) == 5
    assert not rep.all_converged


def test_history_and_lock_bookkeeping(pk):
    # test_history_indexing_and_lock_consistency / test_history_disabled_omits_trajectories
    a = pk.laplacian3d((6, 6, 6))
    cfg = pk.SolverConfig(block_size=4, tol=1e-7, max_iter=400)
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a), config=cfg)
    assert rep.all_converged
    assert [h.iteration for h in rep.history] == list(range(rep.iterations_used + 1))
    for j, it in enumerate(rep.lock_iterations):
        h = rep.history[int(it)]
        assert j in h.locked_now and h.residual_norms[j] < cfg.tol
        assert all(not e.active[j] for e in rep.history[int(it):])
    locked = [j for h in rep.history for j in h.locked_now]
    assert sorted(locked) == list(range(4))             # each column locks once
    quiet = pk.solve(a, t=pk.jacobi_preconditioner(a),
                     config=pk.SolverConfig(block_size=4, tol=1e-7, max_iter=400,
                                            lock_history=False))
    assert all(h.ritz is None and h.residual_norms is None for h in quiet.history)
    np.testing.assert_array_equal(quiet.eigenvalues, rep.eigenvalues)
    np.testing.assert_array_equal(quiet.lock_iterations, rep.lock_iterations)


def test_constraint_basis_validation(pk):
    # test_constraints_from_basis_count / _require_2d_basis / _reject_dependent_basis
    cons = pk.Constraints.from_basis(np.eye(5)[:, :3])
    assert cons.count == 3
    with pytest.raises(ValueError):
        pk.Constraints.from_basis(np.ones(5))
    dep = np.ones((5, 2))
    with pytest.raises((ValueError, pk.NotSPD)):
        pk.Constraints.from_basis(dep)
    x = np.random.default_rng(3).standard_normal((5, 2))
    assert pk.apply_constraints(x, None) is x
    px = pk.apply_constraints(x, cons)
    np.testing.assert_allclose(px[:3], 0.0, atol=1e-14)     # projected out of span(e1..e3)
    np.testing.assert_allclose(px[3:], x[3:], atol=1e-14)
    np.testing.assert_allclose(pk.apply_constraints(px, cons), px, atol=1e-14)  # idempotent


def test_invariant_checker_and_relative_tolerance(pk):
    # test_internal_invariant_checks_pass / test_relative_tolerance_mode
    a = pk.laplacian3d((5, 5, 5))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=3, tol=1e-7, max_iter=300,
                                          check_invariants=True))
    assert rep.all_converged
    rel = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=3, tol=1e-7, max_iter=300,
                                          relative_tol=True))
    assert rel.all_converged
    exact = pk.exact_eigenvalues((5, 5, 5), 3)
    np.testing.assert_allclose(rel.eigenvalues, exact, rtol=1e-8)
    # relative mode: residual below tol * |A x_j| ~ tol * lambda_j
    assert np.all(rel.residual_norms <= 1.01e-7 * rel.eigenvalues * 1.0 + 1e-12)
