"""Closed-form spectrum of the Dirichlet 7-point Laplacian (host, tiny).

Same formula as the reference oracles (problems.py:44-92):
lambda(i,j,k) = 4[sin^2(i pi/2(nx+1)) + sin^2(j pi/2(ny+1)) + sin^2(k pi/2(nz+1))].
``exact_eigenvalues`` only builds modes with every index <= m, which contain
the m smallest, so it is cheap at 464^3 (the reference materialises all n).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .operators import Grid3D

__all__ = ["AnalyticSpectrum", "analytic_spectrum", "exact_eigenvalues", "dense_matrix",
           "dense_oracle_spectrum", "DENSE_ORACLE_LIMIT"]

DENSE_ORACLE_LIMIT = 600   # problems.py:26


@dataclass(frozen=True)
class AnalyticSpectrum:
    grid: Grid3D
    values: np.ndarray
    indices: tuple


def _axis(count, upto):
    modes = np.arange(1, min(count, upto) + 1)
    return modes, 4.0 * np.sin(modes * np.pi / (2.0 * (count + 1))) ** 2


def analytic_spectrum(grid, limit=None):
    """Eigenvalues (ascending, ties lexicographic in (i, j, k)) of modes with
    indices <= limit (all modes when limit is None)."""
    if not isinstance(grid, Grid3D):
        grid = Grid3D(*grid)
    big = max(grid.nx, grid.ny, grid.nz)
    lim = big if limit is None else int(limit)
    mi, tx = _axis(grid.nx, lim)
    mj, ty = _axis(grid.ny, lim)
    mk, tz = _axis(grid.nz, lim)
    vals = (tx[:, None, None] + ty[None, :, None] + tz[None, None, :]).ravel()
    ii, jj, kk = (a.ravel() for a in np.meshgrid(mi, mj, mk, indexing="ij"))
    order = np.lexsort((kk, jj, ii, vals))
    return AnalyticSpectrum(grid, vals[order],
                            tuple(zip(ii[order].tolist(), jj[order].tolist(), kk[order].tolist())))


def exact_eigenvalues(grid, m, scale=1.0):
    """The m smallest eigenvalues of scale * L7 on ``grid``."""
    if not isinstance(grid, Grid3D):
        grid = Grid3D(*grid)
    if not 1 <= m <= grid.n:
        raise ValueError(f"m must be in 1..{grid.n}, got {m}")
    return analytic_spectrum(grid, limit=m).values[:m].copy() * scale


def dense_matrix(op):
    """Dense matrix of an operator: op applied to the identity's columns
    (problems.py:95-98).  Host numpy (n, n)."""
    y = op(np.eye(op.dim))
    return y.detach().cpu().numpy() if hasattr(y, "detach") else np.asarray(y, dtype=np.float64)


def dense_oracle_spectrum(op, n_limit=DENSE_ORACLE_LIMIT):
    """All eigenvalues ascending by brute force (problems.py:101-113); the
    dimension is capped (default 600), as in the reference."""
    if op.dim > n_limit:
        raise ValueError(f"operator dimension {op.dim} exceeds the dense oracle limit {n_limit}")
    from .small import sym_eig

    values, _ = sym_eig(dense_matrix(op))
    return values
