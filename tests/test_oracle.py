"""Pin the CPU oracle against the reference's own golden outputs.

The fixtures under tests/golden/ were produced by tests/golden/make_golden.py
from the real reference package (blockeig 0.1.0).  The oracle must reproduce
the golden trajectory pkg/demos/convergence_history.csv bit for bit.
"""

import numpy as np
import pytest

from oracle import lobpcg_oracle as orc


def test_golden_trajectory_bitwise(golden):
    g = golden("golden_20cubed_m10_jacobi_seed2.npz")
    r = orc.laplacian_case(20, 10, scaled=False, tol=1e-6, max_iter=200, seed=2)
    assert r.status == "Converged"
    assert r.iterations_used == 180
    ritz = np.array(r.hist_ritz)
    resid = np.array(r.hist_resid)
    assert ritz.shape == g["csv_ritz"].shape
    assert np.array_equal(ritz, g["csv_ritz"])
    assert np.array_equal(resid, g["csv_resid"])
    assert np.array_equal(np.array(r.hist_active), g["csv_active"])
    assert list(r.lock_iterations) == [66, 67, 71, 74, 84, 92, 98, 103, 136, 180]
    assert np.array_equal(r.eigenvalues, g["eigenvalues"])


def test_stencil_known_answers_bitwise(golden):
    g = golden("stencil_known_answers.npz")
    for case in range(5):
        nx, ny, nz = (int(v) for v in g[f"dims{case}"])
        x = g[f"x{case}"]
        assert np.array_equal(orc.stencil7(x, nx, ny, nz), g[f"y{case}"])
        s = float((nx + 1) ** 2)
        assert np.array_equal(orc.stencil7(x, nx, ny, nz, s), g[f"ys{case}"])


def test_stencil_ones_counts_neighbours():
    # test_operators.py:155-172 restated
    nx, ny, nz = 3, 2, 4
    out = orc.stencil7(np.ones((nx * ny * nz, 1)), nx, ny, nz)[:, 0]
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                nb = sum(0 <= c < n for c, n in ((i - 1, nx), (i + 1, nx), (j - 1, ny),
                                                 (j + 1, ny), (k - 1, nz), (k + 1, nz)))
                assert out[i + nx * (j + ny * k)] == 6.0 - nb


def test_small_laplacian_matches_reference(golden):
    g = golden("lap5_m4_jacobi.npz")
    n = 125
    r = orc.run_lobpcg(lambda v: orc.stencil7(v, 5, 5, 5), n, 4, tinv=1.0 / np.full(n, 6.0),
                       tol=1e-8, max_iter=300)
    assert r.status == str(g["status"])
    assert r.iterations_used == int(g["iterations_used"])
    np.testing.assert_allclose(r.eigenvalues, g["eigenvalues"], rtol=1e-13)
    np.testing.assert_allclose(r.eigenvalues, orc.closed_form_smallest(5, 5, 5, 4), rtol=1e-8)


def test_diag_pencil_matches_reference(golden):
    g = golden("diag_pencil_n30_m4.npz")
    a = np.arange(1.0, 31.0)
    r = orc.run_lobpcg(lambda v: a[:, None] * v, 30, 4, bdiag=g["bdiag"], tol=1e-10, max_iter=300)
    assert r.status == str(g["status"])
    assert r.iterations_used == int(g["iterations_used"])
    np.testing.assert_allclose(r.eigenvalues, g["dense_vals"], rtol=1e-10)
    np.testing.assert_allclose(r.eigenvalues, g["eigenvalues"], rtol=1e-13)


def test_diag_b_laplacian_matches_reference(golden):
    g = golden("lap12_m6_diagB.npz")
    r = orc.laplacian_case(12, 6, bseed=1000, tol=1e-6, max_iter=150)
    assert r.status == str(g["status"])
    assert r.iterations_used == int(g["iterations_used"])
    np.testing.assert_allclose(r.eigenvalues, g["eigenvalues"], rtol=1e-12)
    assert np.array_equal(r.lock_iterations, g["lock_iterations"])


def test_c1_200_matches_reference(golden):
    g = golden("c1_32cubed_m4_200it.npz")
    r = orc.laplacian_case(32, 4, precond=None, tol=1e-6, max_iter=200, seed=0)
    assert r.status == str(g["status"]) == "MaxIterReached"
    assert r.iterations_used == 200
    np.testing.assert_allclose(r.eigenvalues, g["eigenvalues"], rtol=1e-12)
    np.testing.assert_allclose(np.array(r.hist_ritz), g["hist_ritz"], rtol=1e-10)


def test_closed_form_shortcut_matches_full_formula():
    # problems.py:44-92 on small grids vs the m-smallest shortcut
    for dims, m in [((6, 6, 6), 20), ((8, 9, 10), 10), ((5, 3, 7), 12)]:
        nx, ny, nz = dims
        t = [4.0 * np.sin(np.arange(1, c + 1) * np.pi / (2.0 * (c + 1))) ** 2 for c in dims]
        full = np.sort((t[0][:, None, None] + t[1][None, :, None] + t[2][None, None, :]).ravel())
        np.testing.assert_allclose(orc.closed_form_smallest(nx, ny, nz, m), full[:m], rtol=1e-15)


def _b_tridiag(v):
    y = 3.0 * v
    y[1:] -= v[:-1]
    y[:-1] -= v[1:]
    return y


def _b_zcouple(v, plane=144):
    y = 2.5 * v
    y[plane:] -= 0.5 * v[:-plane]
    y[:-plane] -= 0.5 * v[plane:]
    return y


@pytest.mark.parametrize("name,N,m,tol,jac,bfun", [
    ("tri8", 8, 4, 1e-8, True, _b_tridiag),
    ("zc12", 12, 6, 1e-7, False, _b_zcouple)])
def test_generic_b_matches_reference(golden, name, N, m, tol, jac, bfun):
    """Non-diagonal B (BX, BW, BP by recurrence, lobpcg.py:396, :476,
    :533-538): the oracle reproduces the reference's trajectory."""
    g = golden(f"genb_{name}.npz")
    n = N ** 3
    s = float((N + 1) ** 2)
    r = orc.run_lobpcg(lambda v: orc.stencil7(v, N, N, N, s), n, m, apply_b=bfun,
                       tinv=(1.0 / np.full(n, 6.0 * s)) if jac else None, tol=tol,
                       max_iter=300, seed=0)
    assert r.status == str(g["status"])
    assert r.iterations_used == int(g["iterations_used"])
    np.testing.assert_allclose(np.array(r.hist_ritz), g["hist_ritz"], rtol=1e-12)
    np.testing.assert_allclose(r.eigenvalues, g["dense_vals"], rtol=1e-10)


@pytest.mark.parametrize("name,seed", [("c1", 1), ("c1", 2), ("c5", 1), ("c5", 2)])
def test_seeds_1_2_bitwise(golden, name, seed):
    """Seeds 1 and 2 of the BASELINE shapes (SURVEY 8c harness rules), from the
    real reference (tests/golden/make_seeds.py): the oracle reproduces the
    reference's per-iteration Ritz values and residual norms bit for bit
    (one BLAS thread on both sides)."""
    from threadpoolctl import threadpool_limits

    N, m, precond, diag_b, tol, max_iter = {
        "c1": (32, 4, None, False, 1e-6, 120), "c5": (24, 32, "jacobi", True, 1e-6, 40)}[name]
    g = golden("seeds12.npz")
    k = f"{name}_s{seed}_"
    with threadpool_limits(limits=1, user_api="blas"):
        r = orc.laplacian_case(N, m, precond=precond, bseed=1000 + seed if diag_b else None,
                               tol=tol, max_iter=max_iter, seed=seed)
    assert r.status == str(g[k + "status"]) == "MaxIterReached"
    assert r.iterations_used == int(g[k + "iterations_used"])
    assert np.array_equal(np.array(r.hist_ritz), g[k + "hist_ritz"])
    assert np.array_equal(np.array(r.hist_resid), g[k + "hist_resid"])
    assert np.array_equal(r.eigenvalues, g[k + "eigenvalues"])
