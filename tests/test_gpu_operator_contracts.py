"""Operator / preconditioner / problem-helper contracts as the reference's
suite pins them (pkg/tests/test_operators.py, test_problems.py), on the CUDA
classes of the same names: numpy in gives numpy out, CUDA in gives CUDA out."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    assert torch.cuda.is_available()
    import paper_0705_2626_b200 as pk

    return pk


def dense_matrix(op):
    from paper_0705_2626_b200.problems import dense_matrix as f

    return f(op)


def probe_diagonal(op, chunk=256):
    from paper_0705_2626_b200.operators import probe_diagonal as f

    return f(op, chunk=chunk)


def host(v):
    return v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v)


def block(n, k, seed):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((n, k))


def test_grid(pk):
    # test_grid_index_map / _covers_all_points_once / _out_of_range / test_grid_validation
    g = pk.Grid3D(3, 4, 5)
    assert g.n == 60
    assert [g.index(*p) for p in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (2, 3, 4)]] == \
        [0, 1, 3, 12, 59]
    g2 = pk.Grid3D(2, 3, 2)
    assert sorted(g2.index(i, j, k) for k in range(2) for j in range(3) for i in range(2)) == \
        list(range(12))
    for bad in [(2, 0, 0), (0, -1, 0)]:
        with pytest.raises(IndexError):
            pk.Grid3D(2, 2, 2).index(*bad)
    for dims in [(0, 1, 1), (2, 2.5, 2)]:
        with pytest.raises(ValueError):
            pk.Grid3D(*dims)


def test_wrappers(pk):
    # dense / diagonal / identity / matrix-free wrappers
    with pytest.raises(ValueError):
        pk.DenseOperator(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        pk.DenseOperator(np.ones((2, 3)))
    a = np.array([[2.0, 1.0], [1.0, 4.0]])
    op = pk.DenseOperator(a)
    np.testing.assert_array_equal(dense_matrix(op), a)
    np.testing.assert_array_equal(host(op.diagonal()), [2.0, 4.0])

    d = pk.DiagonalOperator([2.0, 3.0, 5.0])
    assert d.spd and not pk.DiagonalOperator([1.0, -1.0]).spd
    y = d(np.ones(3))
    assert isinstance(y, np.ndarray) and y.shape == (3,)           # 1-D passes through
    np.testing.assert_array_equal(y, [2.0, 3.0, 5.0])
    np.testing.assert_array_equal(host(d.diagonal()), [2.0, 3.0, 5.0])
    yc = d(torch.ones(3, 2, dtype=torch.float64, device="cuda"))
    assert isinstance(yc, torch.Tensor) and yc.is_cuda and yc.shape == (3, 2)

    eye = pk.IdentityOperator(4)
    x = block(4, 2, 0)
    np.testing.assert_array_equal(eye(x), x)
    np.testing.assert_array_equal(host(eye.diagonal()), np.ones(4))
    with pytest.raises(ValueError):
        eye(np.ones((3, 2)))

    with pytest.raises(ValueError):
        pk.MatrixFreeOperator(3, lambda v: v[:2])(np.ones((3, 1)))
    mf = pk.MatrixFreeOperator(2, lambda v: v.clone(), diag=[1.0, 1.0])
    np.testing.assert_array_equal(host(mf.diagonal()), [1.0, 1.0])
    assert pk.MatrixFreeOperator(2, lambda v: v).diagonal() is None


def test_laplacian_structure(pk):
    # test_laplacian_dense_structure / _symmetric / _linearity / _diagonal_is_six
    a = dense_matrix(pk.laplacian3d(pk.Grid3D(4, 4, 4)))
    np.testing.assert_array_equal(a, a.T)
    np.testing.assert_array_equal(np.diag(a), np.full(64, 6.0))
    off = a - np.diag(np.diag(a))
    assert set(np.unique(off)) <= {-1.0, 0.0}
    assert np.all(a.sum(axis=1) >= 0.0)
    op = pk.laplacian3d((5, 4, 3))
    for seed in range(6):
        x, y = block(op.dim, 2, 2 * seed), block(op.dim, 2, 2 * seed + 1)
        np.testing.assert_allclose(x.T @ op(y), (y.T @ op(x)).T, rtol=0.0, atol=1e-13)
    lin = pk.laplacian3d((4, 3, 2))
    x, y = block(lin.dim, 3, 5), block(lin.dim, 3, 6)
    np.testing.assert_allclose(lin(2.0 * x - 3.0 * y), 2.0 * lin(x) - 3.0 * lin(y),
                               rtol=0.0, atol=1e-12)
    small = pk.laplacian3d((3, 3, 3))
    np.testing.assert_array_equal(host(small.diagonal()), np.full(27, 6.0))
    np.testing.assert_allclose(host(probe_diagonal(small, chunk=7)), np.full(27, 6.0))


def test_shift(pk):
    # test_shift_zero_is_identity_on_results / _moves_diagonal_pencil /
    # _with_general_b / _dimension_mismatch
    op = pk.laplacian3d((3, 3, 3))
    x = block(op.dim, 2, 9)
    np.testing.assert_array_equal(pk.shift_operator(op, None, 0.0)(x), op(x))
    a = pk.DiagonalOperator([1.0, 2.0])
    s = pk.shift_operator(a, None, 3.0)
    np.testing.assert_array_equal(dense_matrix(s), np.diag([4.0, 5.0]))
    np.testing.assert_array_equal(host(s.diagonal()), [4.0, 5.0])
    sb = pk.shift_operator(a, pk.DiagonalOperator([2.0, 4.0]), 0.5)
    np.testing.assert_array_equal(dense_matrix(sb), np.diag([2.0, 4.0]))
    np.testing.assert_array_equal(host(sb.diagonal()), [2.0, 4.0])
    with pytest.raises(ValueError):
        pk.shift_operator(pk.IdentityOperator(3), pk.IdentityOperator(4), 1.0)


def test_jacobi_and_identity_preconditioners(pk):
    op = pk.laplacian3d((3, 3, 3))
    x = block(op.dim, 2, 20)
    np.testing.assert_array_equal(pk.jacobi_preconditioner(op)(x), x * (1.0 / 6.0))
    t = pk.jacobi_preconditioner(pk.DiagonalOperator([2.0, 4.0]))
    np.testing.assert_array_equal(t(np.array([2.0, 4.0])), [1.0, 1.0])
    t = pk.jacobi_preconditioner(pk.laplacian3d((4, 2, 3)))
    u, v = block(t.dim, 1, 21)[:, 0], block(t.dim, 1, 22)[:, 0]
    assert u @ t(u) > 0.0
    np.testing.assert_allclose(u @ t(v), v @ t(u), rtol=0.0, atol=1e-14)
    hidden = pk.MatrixFreeOperator(3, pk.DiagonalOperator([1.0, 2.0, 3.0]))
    with pytest.raises(ValueError):
        pk.jacobi_preconditioner(hidden)
    np.testing.assert_allclose(pk.jacobi_preconditioner(hidden, probe=True)(np.ones(3)),
                               [1.0, 0.5, 1.0 / 3.0])
    for bad in ([1.0, 0.0], [1.0, -2.0]):
        with pytest.raises(ValueError):
            pk.jacobi_preconditioner(pk.DiagonalOperator(bad))
    x3 = block(3, 2, 23)
    np.testing.assert_array_equal(pk.IdentityPreconditioner(3)(x3), x3)
    a = block(10, 10, 24)
    dop = pk.DenseOperator(0.5 * (a + a.T))
    np.testing.assert_array_equal(host(probe_diagonal(dop, chunk=3)),
                                  np.diag(0.5 * (a + a.T)))


def test_closed_form_spectrum(pk):
    # test_problems.py: single point, 2^3, line grid, ordering / ties,
    # multiplicities, axis permutations, validation, oracle agreement
    np.testing.assert_allclose(pk.exact_eigenvalues((1, 1, 1), 1), [6.0], rtol=1e-15)
    lam2 = 4.0 * np.sin(np.pi / 6.0) ** 2
    np.testing.assert_allclose(pk.exact_eigenvalues((2, 2, 2), 1), [3 * lam2], rtol=1e-14)
    line = pk.exact_eigenvalues((7, 1, 1), 7)
    want = 4.0 * np.sin(np.arange(1, 8) * np.pi / 16.0) ** 2 + 2 * 4.0 * np.sin(np.pi / 4.0) ** 2
    np.testing.assert_allclose(line, np.sort(want), rtol=1e-14)
    cube = pk.exact_eigenvalues((6, 6, 6), 7)
    assert np.all(np.diff(cube) >= 0.0)
    np.testing.assert_allclose(cube[1:4], cube[1], rtol=1e-14)        # the (1,1,2) triple
    for perm in [(3, 4, 5), (5, 3, 4), (4, 5, 3)]:
        np.testing.assert_allclose(pk.exact_eigenvalues(perm, 10),
                                   pk.exact_eigenvalues((3, 4, 5), 10), rtol=1e-14)
    for m in (0, 65):
        with pytest.raises(ValueError):
            pk.exact_eigenvalues((4, 4, 4), m)
    for dims in [(4, 4, 4), (3, 4, 2)]:
        n = int(np.prod(dims))
        vals = pk.dense_oracle_spectrum(pk.laplacian3d(dims))
        np.testing.assert_allclose(vals, pk.exact_eigenvalues(dims, n), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(pk.dense_oracle_spectrum(pk.DiagonalOperator([3.0, 1.0, 2.0])),
                               [1.0, 2.0, 3.0], rtol=1e-14)
    from paper_0705_2626_b200.problems import DENSE_ORACLE_LIMIT

    big = pk.IdentityOperator(DENSE_ORACLE_LIMIT + 1)
    with pytest.raises(ValueError):
        pk.dense_oracle_spectrum(big)


def test_pcg_names_live_in_operators_too(pk):
    # the reference keeps pcg_solve / InnerPCGPreconditioner in operators.py
    from paper_0705_2626_b200 import operators, pcg

    for name in ("PCGBreakdown", "pcg_solve", "InnerPCGPreconditioner",
                 "inner_pcg_preconditioner"):
        assert getattr(operators, name) is getattr(pcg, name)
        assert name in operators.__all__
