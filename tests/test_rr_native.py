"""b2l_rayleigh_ritz (host, native) against the numpy checker
tests/rr_reference.py on Gram blocks of random tall blocks, including every
rung of the repair ladders (lobpcg.py:475-519).  CPU only: the routine is host
code, no GPU is needed."""

import numpy as np
import pytest

from paper_0705_2626_b200.small import NativeRitz, RitzFailure
from tests.rr_reference import Degenerate, rayleigh_ritz_ref

FLOOR = 1e-8


def _case(n, m, kst, have_p, seed, bdiag=False, dup_w=None, dup_p=None, zero_w=None):
    r = np.random.default_rng(seed)
    a = r.standard_normal((n, n))
    A = a @ a.T / n + np.diag(np.linspace(1.0, 3.0, n))
    d = r.uniform(0.5, 2.0, n) if bdiag else np.ones(n)
    X = r.standard_normal((n, m))
    # B-orthonormal X of Ritz vectors of the subspace (what the solver keeps)
    g = X.T @ (d[:, None] * X)
    L = np.linalg.cholesky(g)
    X = X @ np.linalg.inv(L).T
    ev, V = np.linalg.eigh(X.T @ A @ X)
    X = X @ V
    lam = ev
    W = r.standard_normal((n, kst))
    P = r.standard_normal((n, m))
    if dup_w is not None:
        W[:, dup_w[1]] = W[:, dup_w[0]] * (1.0 + 1e-14)
    if zero_w is not None:
        W[:, zero_w] = 0.0
    if dup_p is not None:
        P[:, dup_p[1]] = P[:, dup_p[0]]
    BX, BW, BP = d[:, None] * X, d[:, None] * W, d[:, None] * P
    AW, AP = A @ W, A @ P
    if have_p:
        G1 = np.hstack([X, W, P]).T @ np.hstack([BX, BW, BP, AP])
    else:
        G1 = np.hstack([X, W]).T @ np.hstack([BX, BW])
    G2 = np.hstack([X, W]).T @ AW
    return G1, G2, lam


def _both(m, kst, have_p, G1, G2, lam, J, sel):
    nat = NativeRitz(m)
    try:
        got = nat(m, kst, have_p, G1, G2, lam, J, sel, FLOOR)
        gerr = None
    except RitzFailure as f:
        got, gerr = None, f.fallbacks
    try:
        ref = rayleigh_ritz_ref(m, kst, have_p, G1, G2, lam, J, sel, FLOOR)
        rerr = None
    except Degenerate as f:
        ref, rerr = None, f.fallbacks
    return got, gerr, ref, rerr


def _compare(got, ref, m, kst):
    lam_g, coef_g, pc_g, fb_g = got
    lam_r, coef_r, pc_r, fb_r = ref
    assert fb_g == fb_r
    assert np.array_equal(pc_g, pc_r)
    np.testing.assert_allclose(lam_g, lam_r, rtol=1e-10, atol=1e-12)
    assert coef_g.shape == coef_r.shape
    # eigenvectors are defined up to sign: compare column by column
    kp = pc_g.size
    rows = m + kst + kp

    def cols(c):
        return np.vstack([c[:m * m].reshape(m, m), c[m * m:m * m + kst * m].reshape(kst, m),
                          c[m * m + kst * m:].reshape(kp, m)])

    cg, cr = cols(coef_g), cols(coef_r)
    assert cg.shape == (rows, m)
    for j in range(m):
        s = np.sign(cg[:, j] @ cr[:, j])
        np.testing.assert_allclose(s * cg[:, j], cr[:, j], rtol=1e-7,
                                   atol=1e-9 * np.abs(cr[:, j]).max())


@pytest.mark.parametrize("m,kst,have_p,bdiag", [(4, 4, False, False), (4, 4, True, False),
                                                (10, 10, True, False), (6, 6, True, True),
                                                (1, 1, True, False)])
def test_native_rr_matches_numpy(m, kst, have_p, bdiag):
    G1, G2, lam = _case(300, m, kst, have_p, seed=m * 7 + kst, bdiag=bdiag)
    J = np.arange(m)
    got, gerr, ref, rerr = _both(m, kst, have_p, G1, G2, lam, J, J.copy())
    assert gerr is None and rerr is None
    _compare(got, ref, m, kst)


def test_native_rr_locked_subset():
    # 3 of 8 columns locked: W holds the 6 previous-active columns, J is 5 of them
    m, kst = 8, 6
    G1, G2, lam = _case(250, m, kst, True, seed=11)
    jprev = np.array([0, 2, 3, 5, 6, 7])
    J = np.array([0, 3, 5, 6, 7])
    sel = np.searchsorted(jprev, J)
    got, gerr, ref, rerr = _both(m, kst, True, G1, G2, lam, J, sel)
    assert gerr is None and rerr is None
    _compare(got, ref, m, kst)
    # unused W column (stored position 1) gets zero coefficients
    coef = got[1]
    assert np.all(coef[m * m + 1 * m:m * m + 2 * m] == 0.0)


def test_native_rr_drops_dependent_w_column():
    m = 5
    G1, G2, lam = _case(200, m, m, True, seed=3, dup_w=(1, 3))
    J = np.arange(m)
    got, gerr, ref, rerr = _both(m, m, True, G1, G2, lam, J, J.copy())
    assert gerr is None and rerr is None
    assert got[3] >= 1 and got[3] == ref[3]
    _compare(got, ref, m, m)


def test_native_rr_drops_degenerate_p():
    m = 5
    G1, G2, lam = _case(200, m, m, True, seed=4, dup_p=(0, 2))
    J = np.arange(m)
    got, gerr, ref, rerr = _both(m, m, True, G1, G2, lam, J, J.copy())
    assert gerr is None and rerr is None
    assert got[2].size == 0 and ref[2].size == 0   # P dropped
    _compare(got, ref, m, m)


def test_native_rr_all_w_zero_is_degenerate():
    m = 3
    G1, G2, lam = _case(100, m, m, True, seed=5)
    z = np.zeros_like(G1)
    z[:m, :m] = G1[:m, :m]
    J = np.arange(m)
    got, gerr, ref, rerr = _both(m, m, True, z, G2, lam, J, J.copy())
    assert got is None and ref is None
    assert gerr == rerr == m


def _split(m, kst, have_p, G1, G2, lam, J, sel):
    nat = NativeRitz(m)
    try:
        nat.begin(m, kst, have_p, G1, J, sel, FLOOR)
        return nat.finish(m, G2, lam), None
    except RitzFailure as f:
        return None, f.fallbacks


@pytest.mark.parametrize("m,kst,have_p,bdiag,kw", [
    (10, 10, True, False, {}), (6, 6, True, True, {}), (4, 4, False, False, {}),
    (5, 5, True, False, {"dup_w": (1, 3)}), (5, 5, True, False, {"dup_p": (0, 2)}),
    (24, 24, True, True, {})])   # 72 x 72 pencil: the LAPACK branch
def test_split_rr_equals_one_call(m, kst, have_p, bdiag, kw):
    """b2l_rayleigh_ritz_begin + _finish (the overlapped form of the unfused
    path) give exactly what b2l_rayleigh_ritz gives."""
    G1, G2, lam = _case(max(300, 4 * m), m, kst, have_p, seed=m + 17, bdiag=bdiag, **kw)
    J = np.arange(m)
    one = NativeRitz(m)(m, kst, have_p, G1, G2, lam, J, J.copy(), FLOOR)
    two, err = _split(m, kst, have_p, G1, G2, lam, J, J.copy())
    assert err is None
    assert two[3] == one[3]
    assert np.array_equal(two[0], one[0])
    assert np.array_equal(two[1], one[1])
    assert np.array_equal(two[2], one[2])


def test_split_rr_degenerate_raises_at_finish():
    m = 3
    G1, G2, lam = _case(100, m, m, True, seed=5)
    z = np.zeros_like(G1)
    z[:m, :m] = G1[:m, :m]
    J = np.arange(m)
    got, fb = _split(m, m, True, z, G2, lam, J, J.copy())
    assert got is None and fb == m


def _large_rr(threads, case=None):
    m = 24
    G1, G2, lam = case if case is not None else _case(400, m, m, True, seed=29)
    J = np.arange(m)
    from threadpoolctl import ThreadpoolController

    with ThreadpoolController().limit(limits=threads, user_api="blas"):
        return NativeRitz(m)(m, m, True, G1, G2, lam, J, J.copy(), FLOOR)


def _large_rr_file(threads, path, out):
    d = np.load(path)
    r = _large_rr(threads, (d["G1"], d["G2"], d["lam"]))
    np.savez(out, lam=r[0], coef=r[1], pcols=r[2])


def test_large_pencil_rr_is_host_thread_independent(tmp_path):
    """m >= 22 (LAPACK/BLAS branch): the result computed under a 4-thread
    BLAS caller equals, bit for bit, the one of a separate process whose
    OpenBLAS only ever had one thread (OPENBLAS_NUM_THREADS=1) on the same
    input Grams, and the caller's setting is restored afterwards."""
    import os
    import subprocess
    import sys

    pytest.importorskip("threadpoolctl")
    from threadpoolctl import ThreadpoolController

    case = _case(400, 24, 24, True, seed=29)
    inp = tmp_path / "in.npz"
    np.savez(inp, G1=case[0], G2=case[1], lam=case[2])
    got = _large_rr(4, case)
    ctl = ThreadpoolController()
    with ctl.limit(limits=4, user_api="blas"):
        _large_rr(4, case)
        assert {i["num_threads"] for i in ctl.select(user_api="blas").info()} == {4}
    out = tmp_path / "one.npz"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); "
            "from tests.test_rr_native import _large_rr_file; _large_rr_file(1, %r, %r)"
            ) % (root, str(inp), str(out))
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root)
    ref = np.load(out)
    for a, b in zip(got[:3], (ref["lam"], ref["coef"], ref["pcols"])):
        assert np.array_equal(a, b)


def test_cluster_alignment_picks_the_basis_closest_to_x():
    """A wanted triple eigenvalue: with a cluster gap set (b2l_set_rr_align,
    what the solver does every step) the eigensolve returns the cluster's
    basis closest to the current Ritz vectors -- the X block of the cluster's
    coefficients is symmetric positive definite -- and it is the same
    invariant subspace, the same Ritz values and as B-orthonormal as the
    unaligned answer (any basis of the cluster is a valid eigensolver
    output)."""
    n, m = 80, 5
    r = np.random.default_rng(11)
    ev = np.concatenate([[1.0, 2.0, 2.0, 2.0, 3.0], np.linspace(4.0, 9.0, n - 5)])
    A = np.diag(ev)
    # Ritz vectors close to e_1..e_5 with the triple rotated inside its span
    q, _ = np.linalg.qr(r.standard_normal((3, 3)))
    X = np.eye(n)[:, :m].copy()
    X[:, 1:4] = X[:, 1:4] @ q
    X += 1e-6 * r.standard_normal((n, m))
    X, _ = np.linalg.qr(X)
    th, V = np.linalg.eigh(X.T @ A @ X)
    X, lam = X @ V, th
    W = (A @ X - X * lam)                       # residuals
    P = 1e-3 * r.standard_normal((n, m))
    G1 = np.hstack([X, W, P]).T @ np.hstack([X, W, P, A @ P])
    G2 = np.hstack([X, W]).T @ (A @ W)
    J = np.arange(m)
    out = {}
    for gap in (0.0, 1e-5):
        nat = NativeRitz(m)
        nat.align = gap
        lam_n, coef, pcols, fb = nat(m, m, True, G1, G2, lam, J, J.copy(), FLOOR)
        kp = pcols.size
        cx = coef[:m * m].reshape(m, m)
        cw = coef[m * m:2 * m * m].reshape(m, m)
        cp = coef[2 * m * m:].reshape(kp, m)
        Xn = X @ cx + W @ cw + P[:, pcols] @ cp
        np.testing.assert_allclose(Xn.T @ Xn, np.eye(m), atol=1e-10)
        out[gap] = (lam_n, cx, Xn)
    (l0, c0, x0), (l1, c1, x1) = out[0.0], out[1e-5]
    np.testing.assert_allclose(l0, l1, rtol=1e-13)
    assert l1[3] - l1[1] < 1e-9                       # inside the gap and the 1e-8 relative cap
    s = slice(1, 4)
    # same invariant subspace of the cluster, same vectors outside it
    np.testing.assert_allclose(x0[:, s] @ x0[:, s].T, x1[:, s] @ x1[:, s].T, atol=1e-9)
    for j in (0, 4):
        np.testing.assert_allclose(np.abs(x0[:, j] @ x1[:, j]), 1.0, atol=1e-12)
    g = c1[s, s]
    # aligned: symmetric (in the orthonormalised basis exactly; the folded
    # coefficients of the raw blocks carry the W / P couplings, ~1e-7 here) ...
    np.testing.assert_allclose(g, g.T, atol=1e-6)
    assert np.linalg.eigvalsh(0.5 * (g + g.T)).min() > 0.5   # ... positive definite, near I
    # and it is the closest basis: no rotation of the cluster brings the X block nearer to I
    u, _, vt = np.linalg.svd(c0[s, s])
    best = c0[:, s] @ (vt.T @ u.T)                   # polar alignment of the unaligned answer
    np.testing.assert_allclose(best[s], g, atol=1e-6)
