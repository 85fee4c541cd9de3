"""Block primitives of the reference's ``multivec`` module (multivec.py:1-229)
on the B200 path.

Same names and contracts.  The tall-block operations (``gram``, ``multiply``,
``tri_solve_right``, ``column_norms``, ``seeded_random_fill``) run in the
native kernels (K5 Gram, K6 update, K9 generator); the small dense ones
(``cholesky``, ``chol_solve``, ``sym_eig``, ``gen_sym_eig``) on the host with
LAPACK, as in the reference.  Blocks may be numpy arrays (answered in numpy,
as the reference does) or CUDA float64 tensors (answered on the device).
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as dv
from .small import NotSPD, chol_solve, gen_sym_eig as _gen_sym_eig, sym_eig as _sym_eig
from .small import cholesky as _cholesky

__all__ = ["NotSPD", "gram", "multiply", "cholesky", "tri_solve_right", "chol_solve",
           "sym_eig", "gen_sym_eig", "column_norms", "seeded_random_fill"]


def _device():
    from .operators import _default_device

    return _default_device()


def _tall(x, name):
    """(tensor (n, ld) padded block, k, host?) for a tall (n, k) block."""
    host = not isinstance(x, torch.Tensor)
    if host:
        a = np.asarray(x, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError(f"{name} must be 2-d, got shape {a.shape}")
        n, k = a.shape
        t = dv.new_block(n, dv.even(k), _device())
        t[:, :k] = torch.from_numpy(np.ascontiguousarray(a))
        return t, k, True
    if x.dim() != 2:
        raise ValueError(f"{name} must be 2-d, got shape {tuple(x.shape)}")
    n, k = x.shape
    if (x.is_cuda and x.dtype == torch.float64 and x.stride(1) == 1 and x.stride(0) % 2 == 0
            and x.stride(0) >= k and x.data_ptr() % 16 == 0):
        return x, k, False
    t = dv.new_block(n, dv.even(k), x.device if x.is_cuda else _device())
    t[:, :k] = x
    return t, k, False


def _small(a, name):
    a = np.asarray(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                   dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-d, got shape {a.shape}")
    return a


def gram(x, y):
    """x.T @ y of two tall blocks (multivec.py:58-71); a small host matrix."""
    X, kx, _ = _tall(x, "x")
    Y, ky, _ = _tall(y, "y")
    if X.shape[0] != Y.shape[0]:
        raise ValueError(f"row dimensions differ: x has {X.shape[0]}, y has {Y.shape[0]}")
    return dv.to_host(dv.gram(X.shape[0], [(X, kx)], [(Y, ky)])).copy()


def multiply(x, c):
    """x @ c (multivec.py:74-86): the K6 update with no X term."""
    X, k, host = _tall(x, "x")
    c = _small(c, "c")
    if c.shape[0] != k:
        raise ValueError(f"inner dimensions differ: x has {k} columns, c has {c.shape[0]} rows")
    n, r = X.shape[0], c.shape[1]
    out = dv.new_block(n, dv.even(r), X.device)
    if r:
        dv.update(n, r, None, None, None, out, None, w=X, kw=k, cw=dv.to_device(c, X.device),
                  x_plus_p=True)
    res = out[:, :r]
    return dv.to_host(res).copy() if host else res


def cholesky(g, pivot_floor=0.0):
    """Upper R with g = R^T R (multivec.py:89-122); NotSPD(pivot) on failure."""
    g = _small(g, "g")
    if g.shape[0] != g.shape[1]:
        raise ValueError(f"matrix must be square, got shape {g.shape}")
    return _cholesky(g, pivot_floor)


def tri_solve_right(x, r):
    """z with z @ r = x, i.e. x R^{-1} (multivec.py:125-146): one K6 update
    with the inverted small factor."""
    from .small import upper_inverse

    r = _small(r, "r")
    k = r.shape[0]
    if r.shape[1] != k:
        raise ValueError(f"factor must be square, got shape {r.shape}")
    X, kx, host = _tall(x, "x")
    if kx != k:
        raise ValueError(f"x has {kx} columns but the factor is {k} x {k}")
    if np.any(np.diag(r) == 0.0):
        raise ValueError("triangular factor is singular (zero diagonal)")
    if k == 0:
        return x.copy() if host else x.clone()
    out = dv.new_block(X.shape[0], X.shape[1], X.device)
    dv.update(X.shape[0], k, X, None, dv.to_device(upper_inverse(np.triu(r)), X.device), out,
              None)
    res = out[:, :k]
    return dv.to_host(res).copy() if host else res


def sym_eig(g):
    """Ascending eigenpairs of a small symmetric matrix, upper triangle read
    (multivec.py:161-171)."""
    g = _small(g, "g")
    if g.shape[0] != g.shape[1]:
        raise ValueError(f"matrix must be square, got shape {g.shape}")
    return _sym_eig(g)


def gen_sym_eig(gram_a, gram_b, want=None, pivot_floor=0.0):
    """Smallest ``want`` pairs of gram_a c = lam gram_b c (multivec.py:174-211)."""
    gram_a, gram_b = _small(gram_a, "gram_a"), _small(gram_b, "gram_b")
    k = gram_a.shape[0]
    if gram_a.shape != (k, k) or gram_b.shape != (k, k):
        raise ValueError(f"pencil blocks must be square and matching, got "
                         f"{gram_a.shape} and {gram_b.shape}")
    if want is None:
        want = k
    if not 0 < want <= k:
        raise ValueError(f"want must be in 1..{k}, got {want}")
    return _gen_sym_eig(gram_a, gram_b, want, pivot_floor)


def column_norms(x):
    """Euclidean norm of each column (multivec.py:214-217), from the K5 Gram."""
    X, k, host = _tall(x, "x")
    g = dv.gram(X.shape[0], [(X, k)], [(X, k)])
    nrm = torch.sqrt(torch.diagonal(g).clamp_min(0.0))
    return dv.to_host(nrm).copy() if host else nrm


def seeded_random_fill(n, k, seed, device=False):
    """Generator(PCG64(seed)).uniform(-1, 1, (n, k)) bit for bit
    (multivec.py:220-229), generated on the GPU (K9).  device=True returns
    the CUDA tensor instead of the host array."""
    if n < 1 or k < 1:
        raise ValueError("dimensions must be positive")
    out = dv.new_block(n, dv.even(k), _device())
    dv.seeded_fill(out, k, seed)
    res = out[:, :k]
    return res if device else dv.to_host(res).copy()
