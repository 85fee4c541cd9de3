"""The reference's multivec / b_orthonormalize / dense-oracle API on the B200
path (multivec.py:1-229, lobpcg.py:147-179, problems.py:95-113), checked the
way the reference's test_multivec.py / test_lobpcg.py check them."""

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


@pytest.fixture(scope="module")
def mv(pk):
    from paper_0705_2626_b200 import multivec

    return multivec


def blk(n, k, seed):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((n, k))


def test_gram_and_multiply_match_numpy(mv):
    for n, kx, ky, seed in [(1, 1, 1, 0), (37, 3, 5, 1), (5000, 7, 2, 2), (20001, 16, 16, 3)]:
        x, y = blk(n, kx, seed), blk(n, ky, seed + 10)
        np.testing.assert_allclose(mv.gram(x, y), x.T @ y, rtol=1e-12, atol=1e-12 * n)
        c = blk(kx, ky, seed + 20)
        np.testing.assert_allclose(mv.multiply(x, c), x @ c, rtol=1e-12, atol=1e-12 * kx)
    with pytest.raises(ValueError):
        mv.gram(blk(5, 2, 0), blk(6, 2, 0))
    with pytest.raises(ValueError):
        mv.multiply(blk(5, 2, 0), blk(3, 2, 0))
    # permutation swaps columns exactly
    x = blk(100, 2, 4)
    np.testing.assert_array_equal(mv.multiply(x, np.array([[0.0, 1.0], [1.0, 0.0]])), x[:, ::-1])


def test_device_blocks_stay_on_device(mv):
    x = torch.as_tensor(blk(1000, 3, 5), device="cuda")
    c = blk(3, 4, 6)
    y = mv.multiply(x, c)
    assert isinstance(y, torch.Tensor) and y.is_cuda and tuple(y.shape) == (1000, 4)
    np.testing.assert_allclose(y.cpu().numpy(), x.cpu().numpy() @ c, rtol=1e-12, atol=1e-12)


def test_tri_solve_right(mv):
    x = blk(3000, 4, 7)
    r = np.triu(blk(4, 4, 8)) + 4.0 * np.eye(4)
    z = mv.tri_solve_right(x, r)
    np.testing.assert_allclose(z @ r, x, rtol=0, atol=1e-12 * np.abs(x).max())
    d = np.diag([2.0, 4.0, 0.5, 1.0])
    np.testing.assert_allclose(mv.tri_solve_right(x, d), x / np.diag(d), rtol=1e-15)
    with pytest.raises(ValueError):
        mv.tri_solve_right(x, np.diag([1.0, 0.0, 1.0, 1.0]))
    empty = np.zeros((10, 0))
    assert mv.tri_solve_right(empty, np.zeros((0, 0))).shape == (10, 0)


def test_small_dense(mv, pk):
    g = np.array([[4.0, 2.0], [2.0, 3.0]])
    r = mv.cholesky(g)
    np.testing.assert_allclose(r.T @ r, g, rtol=1e-15)
    with pytest.raises(pk.NotSPD) as exc:
        mv.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert exc.value.pivot == 1
    a = np.diag([3.0, 1.0, 2.0])
    vals, vecs = mv.sym_eig(a)
    np.testing.assert_array_equal(vals, [1.0, 2.0, 3.0])
    vals, c = mv.gen_sym_eig(np.diag([2.0, 6.0]), np.diag([1.0, 2.0]), want=1)
    np.testing.assert_allclose(vals, [2.0])
    with pytest.raises(ValueError):
        mv.gen_sym_eig(np.eye(2), np.eye(2), want=3)
    rhs = blk(3, 2, 9)
    spd = np.array([[4.0, 1.0, 0.0], [1.0, 3.0, 1.0], [0.0, 1.0, 2.0]])
    np.testing.assert_allclose(mv.chol_solve(mv.cholesky(spd), rhs), np.linalg.solve(spd, rhs),
                               rtol=1e-13)


def test_column_norms(mv):
    x = blk(4096, 5, 11)
    np.testing.assert_allclose(mv.column_norms(x), np.linalg.norm(x, axis=0), rtol=1e-13)
    np.testing.assert_allclose(mv.column_norms(np.array([[3.0], [4.0]])), [5.0], rtol=1e-15)


def test_seeded_random_fill_is_numpy_pcg64(mv):
    for n, k, seed in [(1, 1, 0), (999, 3, 7), (100000, 10, 12345)]:
        ref = np.random.Generator(np.random.PCG64(seed)).uniform(-1.0, 1.0, size=(n, k))
        np.testing.assert_array_equal(mv.seeded_random_fill(n, k, seed), ref)
    with pytest.raises(ValueError):
        mv.seeded_random_fill(0, 2, 0)


def test_b_orthonormalize(pk, mv):
    x = np.zeros((4, 1))
    x[0, 0] = 2.0
    xo, bxo, r = pk.b_orthonormalize(x, x)
    np.testing.assert_array_equal(xo, np.eye(4)[:, :1])
    assert bxo is xo
    np.testing.assert_array_equal(r, [[2.0]])
    b = pk.DiagonalOperator(np.arange(1.0, 31.0))
    d = np.arange(1.0, 31.0)
    for seed in range(5):
        x = blk(30, 4, seed)
        xo, bxo, r = pk.b_orthonormalize(x, d[:, None] * x)
        np.testing.assert_allclose(xo.T @ bxo, np.eye(4), rtol=0.0, atol=1e-11)
        np.testing.assert_allclose(bxo, b(xo), rtol=0.0, atol=1e-11)
        np.testing.assert_allclose(xo @ r, x, rtol=0.0, atol=1e-11 * np.abs(x).max())
        np.testing.assert_array_equal(np.tril(r, -1), np.zeros((4, 4)))
    with pytest.raises(pk.NotSPD):
        pk.b_orthonormalize(np.ones((6, 2)), np.ones((6, 2)))
    z = np.eye(5)[:, :3].copy()
    z[:, 1] = 0.0
    with pytest.raises(pk.NotSPD) as exc:
        pk.b_orthonormalize(z, z)
    assert exc.value.pivot == 1


def test_dense_oracle_spectrum(pk):
    vals = pk.dense_oracle_spectrum(pk.laplacian3d((4, 5, 3)))
    np.testing.assert_allclose(vals, pk.exact_eigenvalues((4, 5, 3), 60), rtol=1e-12)
    with pytest.raises(ValueError):
        pk.dense_oracle_spectrum(pk.laplacian3d((10, 10, 10)))


def test_project_pencil_matches_reference(pk, golden):
    """project_pencil against the reference's private _project_pencil
    (lobpcg.py:299-340) on the same blocks, with and without exact_diagonal
    (SURVEY 8 f-4), host arrays and CUDA tensors."""
    g = golden("project_pencil.npz")
    names = ("x", "ax", "w", "aw", "bw", "pj", "apj", "bpj", "bx")
    host = {k: g[k] for k in names}
    dev = {k: torch.from_numpy(g[k]).cuda() for k in names}
    for blocks in (host, dev):
        args = [blocks[k] for k in names]
        for exact in (False, True):
            ga, gb = pk.project_pencil(g["lam"], *args, exact_diagonal=exact)
            np.testing.assert_allclose(ga, g[f"ga_{int(exact)}"], rtol=1e-12, atol=1e-11)
            np.testing.assert_allclose(gb, g[f"gb_{int(exact)}"], rtol=1e-12, atol=1e-11)
        a2 = args[:5] + [None, None, None, args[8]]
        ga, gb = pk.project_pencil(g["lam"], *a2)
        np.testing.assert_allclose(ga, g["ga_nop"], rtol=1e-12, atol=1e-11)
        np.testing.assert_allclose(gb, g["gb_nop"], rtol=1e-12, atol=1e-11)
        # the lower-triangular blocks stay empty, as in the reference
        assert np.all(ga[4:, :4] == 0.0) and np.all(gb[4:, :4] == 0.0)
