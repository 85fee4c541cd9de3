"""Host fp64 algebra on the small projected matrices (<= 3m x 3m).

The reference does this on the host too (multivec.py:89-211, scipy LAPACK):
the k x k Cholesky is written out so a failure names its pivot (the first
numerically dependent column), which drives the basis-repair ladder of
lobpcg.py:182-200 and :501-519.  Sizes here are at most 192 x 192.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import eigh, solve_triangular


class NotSPD(Exception):
    """A Cholesky pivot failed; ``pivot`` is its zero-based index
    (reference multivec.py:34-48)."""

    def __init__(self, pivot):
        super().__init__(f"matrix is not positive definite (pivot {pivot})")
        self.pivot = int(pivot)


def cholesky(g: np.ndarray, pivot_floor: float = 0.0) -> np.ndarray:
    """Upper R with g = R^T R from g's upper triangle; a pivot <= floor*g_jj
    (or non-finite) raises NotSPD(j) (multivec.py:89-122)."""
    g = np.asarray(g, dtype=np.float64)
    k = g.shape[0]
    if g.ndim != 2 or g.shape[1] != k:
        raise ValueError(f"matrix must be square, got shape {g.shape}")
    r = np.zeros((k, k))
    for j in range(k):
        col = r[:j, j]
        piv = g[j, j] - col @ col
        if not (piv > pivot_floor * g[j, j]) or not np.isfinite(piv):
            raise NotSPD(j)
        rjj = np.sqrt(piv)
        r[j, j] = rjj
        if j + 1 < k:
            r[j, j + 1:] = (g[j, j + 1:] - col @ r[:j, j + 1:]) / rjj
    return r


def sym_eig(g: np.ndarray):
    """Ascending eigenpairs of a symmetric matrix, upper triangle read."""
    return eigh(np.asarray(g, dtype=np.float64), lower=False)


def gen_sym_eig(ga: np.ndarray, gb: np.ndarray, want: int, pivot_floor: float = 0.0):
    """Smallest ``want`` pairs of ga c = lam gb c via gb = R^T R
    (multivec.py:174-211); only upper triangles are read."""
    ga = np.triu(ga) + np.triu(ga, 1).T
    r = cholesky(gb, pivot_floor)
    t = solve_triangular(r, ga, trans="T", lower=False)
    t = solve_triangular(r, t.T, trans="T", lower=False)
    t = 0.5 * (t + t.T)
    vals, vecs = eigh(t, lower=False)
    c = solve_triangular(r, vecs[:, :want], trans="N", lower=False)
    return vals[:want], c


def upper_inverse(r: np.ndarray) -> np.ndarray:
    """R^{-1} for an upper-triangular R (used to fold Cholesky-QR factors
    into the Gram blocks and update coefficients instead of rewriting the
    tall block, which the reference does with tri_solve_right)."""
    k = r.shape[0]
    if k == 0:
        return np.zeros((0, 0))
    return solve_triangular(r, np.eye(k), lower=False)


def scaled_cholesky(g: np.ndarray, pivot_floor: float = 0.0):
    """Cholesky-QR factor of a block from its raw Gram g = X^T B X.

    Mirrors b_orthonormalize (lobpcg.py:147-179): columns are scaled to unit
    B-norm first (sq = diag(g)), the scaled Gram D^-1 g D^-1 is factored with
    the pivot floor, and the effective factor R_eff = R D is returned together
    with its inverse, so that X_orth = X @ inv(R_eff).  A column with
    non-positive or non-finite B-norm raises NotSPD(column).
    """
    sq = np.diag(g).copy()
    bad = ~(sq > 0.0) | ~np.isfinite(sq)
    if bad.any():
        raise NotSPD(int(np.flatnonzero(bad)[0]))
    s = np.sqrt(sq)
    gs = g / s[:, None] / s[None, :]
    r = cholesky(gs, pivot_floor)
    reff = r * s[None, :]
    return reff, upper_inverse(reff)
