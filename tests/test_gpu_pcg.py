"""Inner-PCG preconditioner on the GPU: the column-batched
PCG (csrc/pcg.cu) against the reference's pcg_solve vectors, its breakdown
behaviour, and the reference demo's outer-iteration table
(pkg/demos/preconditioner_quality.csv) -- fixtures from the real reference
(tests/golden/pcg_cases.npz, make_golden.py --pcg)."""

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


@pytest.mark.parametrize("name", ["none", "jacobi"])
@pytest.mark.parametrize("it", [1, 5, 30, "rtol"])
def test_pcg_solve_matches_reference(pk, golden, name, it):
    g = golden("pcg_cases.npz")
    L = pk.laplacian3d((8, 9, 7))
    m = pk.jacobi_preconditioner(L) if name == "jacobi" else None
    if it == "rtol":
        x = pk.pcg_solve(L, m, g["b"], 200, 1e-6)
    else:
        x = pk.pcg_solve(L, m, g["b"], it, 0.0)
    ref = g[f"x_{name}_{it}"]
    assert isinstance(x, np.ndarray) and x.shape == ref.shape
    # elementwise rounding as numpy; only the dot products sum in another order
    np.testing.assert_allclose(x, ref, rtol=0, atol=1e-10 * np.abs(ref).max())


def test_pcg_block_columns_independent(pk, golden):
    """k columns side by side == k single-column solves (each column keeps
    its own scalars and stop flag)."""
    from paper_0705_2626_b200.pcg import pcg_block

    g = golden("pcg_cases.npz")
    L = pk.laplacian3d((8, 9, 7))
    m = pk.jacobi_preconditioner(L)
    r = np.random.default_rng(5)
    B = np.stack([g["b"], r.standard_normal(L.dim), np.zeros(L.dim), 1e-3 * g["b"]], axis=1)
    Bt = torch.as_tensor(B, device="cuda")
    X = pcg_block(L, m, Bt, 12, 1e-4).cpu().numpy()
    for j in range(4):
        xj = pk.pcg_solve(L, m, B[:, j], 12, 1e-4)
        np.testing.assert_allclose(X[:, j], xj, rtol=0, atol=1e-12 * max(1.0, np.abs(xj).max()))
    assert np.all(X[:, 2] == 0.0)


def test_pcg_breakdown(pk, golden):
    g = golden("pcg_cases.npz")
    assert int(g["breakdown"]) == 1
    d = pk.DiagonalOperator(np.linspace(-1.0, 3.0, 50))
    with pytest.raises(pk.PCGBreakdown):
        pk.pcg_solve(d, None, np.ones(50), 10)


def test_pcg_validation(pk):
    L = pk.laplacian3d((4, 4, 4))
    with pytest.raises(ValueError):
        pk.pcg_solve(L, None, np.ones(10), 5)
    with pytest.raises(ValueError):
        pk.pcg_solve(L, None, np.ones(64), 0)
    with pytest.raises(ValueError):
        pk.inner_pcg_preconditioner(L, None, 0)
    with pytest.raises(ValueError):
        pk.inner_pcg_preconditioner(L, pk.jacobi_preconditioner(pk.laplacian3d((3, 3, 3))), 2)


def test_generic_operator_and_inner(pk, golden):
    """Callback A and a callback inner preconditioner take the generic path
    (A p by the callback + b2l_gram; z = M r by the callback + b2l_pcg_dot)."""
    g = golden("pcg_cases.npz")
    L = pk.laplacian3d((8, 9, 7))
    Lcb = pk.MatrixFreeOperator(L.dim, lambda v: L(v), spd=True)
    jac = pk.jacobi_preconditioner(L)

    class CB(pk.Preconditioner):
        def _apply(self, x):
            return jac(x)

    x = pk.pcg_solve(Lcb, CB(L.dim), g["b"], 30, 0.0)
    ref = g["x_jacobi_30"]
    np.testing.assert_allclose(x, ref, rtol=0, atol=1e-10 * np.abs(ref).max())


@pytest.mark.parametrize("k", [0, 1, 2, 5, 10, 15, 20])
def test_demo_outer_iterations(pk, golden, k):
    """pkg/demos/preconditioner_quality.csv: 20^3, m = 1, tol 1e-6, seed 2."""
    g = golden("pcg_cases.npz")
    want = int(g["demo_outer"][list(g["demo_steps"]).index(k)])
    a = pk.laplacian3d((20, 20, 20))
    jacobi = pk.jacobi_preconditioner(a)
    t = jacobi if k == 0 else pk.inner_pcg_preconditioner(a, jacobi, k)
    rep = pk.solve(a, t=t, config=pk.SolverConfig(block_size=1, tol=1e-6, max_iter=600, seed=2,
                                                  lock_history=False))
    assert rep.status == "Converged"
    assert abs(rep.iterations_used - want) <= 1, (rep.iterations_used, want)


def test_inner_pcg_block_solve(pk, golden):
    g = golden("pcg_cases.npz")
    s = float(25 ** 2)
    A = pk.Laplacian3D((24, 24, 24), scale=s)
    t = pk.inner_pcg_preconditioner(A, pk.jacobi_preconditioner(A), 5)
    rep = pk.solve(A, t=t, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=200, seed=1))
    assert rep.status == str(g["block_status"])
    assert abs(rep.iterations_used - int(g["block_iterations_used"])) <= 2
    exact = pk.exact_eigenvalues((24, 24, 24), 4, scale=s)
    assert np.max(np.abs(rep.eigenvalues - exact) / exact) <= 1e-8
