"""Matrix-free operators and preconditioners on CUDA blocks.

Same names, attributes and call contracts as the reference
(operators.py:41-334): an operator has ``dim`` and ``spd``, is callable on an
(n, k) or (n,) block and returns the same shape, and may expose
``diagonal()``.  The difference is the data: blocks here are CUDA float64
tensors (numpy input is accepted and answered in numpy, for convenience).

The solver recognises ``Laplacian3D``, ``DiagonalOperator``,
``IdentityOperator``, ``JacobiPreconditioner`` and ``IdentityPreconditioner``
and fuses them into its kernels; any other callable is invoked on CUDA
tensors, keeping the reference's "anything that can multiply a block plugs
in" contract with no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv

__all__ = [
    "Grid3D",
    "LinearOperator",
    "MatrixFreeOperator",
    "DenseOperator",
    "DiagonalOperator",
    "IdentityOperator",
    "Laplacian3D",
    "ShiftedOperator",
    "laplacian3d",
    "shift_operator",
    "Preconditioner",
    "IdentityPreconditioner",
    "JacobiPreconditioner",
    "jacobi_preconditioner",
    "probe_diagonal",
    # the reference keeps its inner PCG in operators.py (:336-427); here it
    # lives in pcg.py and is re-exported lazily (pcg imports this module)
    "PCGBreakdown",
    "pcg_solve",
    "InnerPCGPreconditioner",
    "inner_pcg_preconditioner",
]

_PCG_NAMES = ("PCGBreakdown", "pcg_solve", "InnerPCGPreconditioner", "inner_pcg_preconditioner")


def __getattr__(name):
    if name in _PCG_NAMES:
        from . import pcg

        return getattr(pcg, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_0705_2626_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _to_block(x, dim: int, what: str, device):
    """Accept a CUDA tensor or array-like; return (2-D cuda f64 tensor,
    was_1d, was_numpy).  Mirrors the shape rules of operators.py:84-94."""
    host = not isinstance(x, torch.Tensor)
    if host:
        arr = np.asarray(x, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    else:
        if not x.is_cuda:
            x = x.to(device)
        t = x if x.dtype == torch.float64 else x.to(torch.float64)
    single = t.dim() == 1
    if single:
        t = t[:, None]
    if t.dim() != 2 or t.shape[0] != dim:
        raise ValueError(f"{what} of dimension {dim} applied to block of shape {tuple(t.shape)}")
    return t, single, host


def _from_block(y, single: bool, host: bool):
    if single:
        y = y[:, 0]
    if host:
        return y.detach().cpu().numpy()
    return y


@dataclass(frozen=True)
class Grid3D:
    """nx x ny x nz interior points; point (i, j, k) -> i + nx*(j + ny*k)
    (reference operators.py:41-67)."""

    nx: int
    ny: int
    nz: int

    def __post_init__(self):
        for name, value in (("nx", self.nx), ("ny", self.ny), ("nz", self.nz)):
            if not isinstance(value, (int, np.integer)) or value < 1:
                raise ValueError(f"{name} must be a positive integer, got {value!r}")

    @property
    def n(self):
        return self.nx * self.ny * self.nz

    def index(self, i, j, k):
        if not (0 <= i < self.nx and 0 <= j < self.ny and 0 <= k < self.nz):
            raise IndexError(f"point ({i}, {j}, {k}) outside grid {self}")
        return i + self.nx * (j + self.ny * k)


class LinearOperator:
    """Symmetric block operator on CUDA tensors (operators.py:70-101)."""

    def __init__(self, dim, spd=False, device=None):
        if dim < 1:
            raise ValueError(f"operator dimension must be positive, got {dim}")
        self.dim = int(dim)
        self.spd = bool(spd)
        self.device = torch.device(device) if device is not None else _default_device()

    def __call__(self, x):
        t, single, host = _to_block(x, self.dim, "operator", self.device)
        return _from_block(self._apply(t), single, host)

    def _apply(self, x):
        raise NotImplementedError

    def diagonal(self):
        """Matrix diagonal as a (dim,) CUDA tensor, or None."""
        return None


class MatrixFreeOperator(LinearOperator):
    """Wrap ``f(x) -> y`` on CUDA tensors (operators.py:104-121)."""

    def __init__(self, dim, apply_block, spd=False, diag=None, device=None):
        super().__init__(dim, spd=spd, device=device)
        self._apply_block = apply_block
        self._diag = None if diag is None else torch.as_tensor(
            np.asarray(diag, dtype=np.float64) if not isinstance(diag, torch.Tensor) else diag,
            dtype=torch.float64, device=self.device).clone()

    def _apply(self, x):
        y = self._apply_block(x)
        if not isinstance(y, torch.Tensor):
            y = torch.as_tensor(np.asarray(y, dtype=np.float64), device=self.device)
        if tuple(y.shape) != tuple(x.shape):
            raise ValueError(
                f"operator apply returned shape {tuple(y.shape)}, expected {tuple(x.shape)}")
        return y.to(torch.float64)

    def diagonal(self):
        return None if self._diag is None else self._diag.clone()


class DenseOperator(LinearOperator):
    """Explicit symmetric matrix (tests / small oracles; operators.py:124-140)."""

    def __init__(self, a, spd=False, device=None):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError(f"matrix must be square, got shape {a.shape}")
        if not np.allclose(a, a.T, rtol=0.0, atol=1e-13 * max(1.0, np.abs(a).max())):
            raise ValueError("matrix is not symmetric")
        super().__init__(a.shape[0], spd=spd, device=device)
        self.a = torch.as_tensor(0.5 * (a + a.T), device=self.device)

    def _apply(self, x):
        return self.a @ x

    def diagonal(self):
        return torch.diagonal(self.a).clone()


class DiagonalOperator(LinearOperator):
    """diag(d); as B it is fused into the Gram/residual kernels as a row
    weight (operators.py:143-155)."""

    def __init__(self, d, device=None):
        if isinstance(d, torch.Tensor):
            dh = d.detach().to("cpu", torch.float64).numpy()
        else:
            dh = np.asarray(d, dtype=np.float64)
        if dh.ndim != 1 or dh.size == 0:
            raise ValueError(f"diagonal must be a nonempty 1-d array, got shape {dh.shape}")
        super().__init__(dh.size, spd=bool(np.all(dh > 0.0)), device=device)
        self.d = torch.as_tensor(dh.copy(), device=self.device)

    def _apply(self, x):
        return self.d[:, None] * x

    def diagonal(self):
        return self.d.clone()


class IdentityOperator(LinearOperator):
    def __init__(self, dim, device=None):
        super().__init__(dim, spd=True, device=device)

    def _apply(self, x):
        return x.clone()

    def diagonal(self):
        return torch.ones(self.dim, dtype=torch.float64, device=self.device)


class _StencilProbe:
    """Symbolic block passed once through a MatrixFreeOperator's function to
    recognise the reference's BASELINE harness
    ``MatrixFreeOperator(n, lambda v: s * L(v), diag=6s)`` (operators.py:104-121,
    SURVEY 8c) as the scaled Laplacian it is, so it runs on the fused kernels.
    It supports exactly: ``L(probe)`` for a Laplacian3D ``L`` and one
    multiplication by a real scalar (the kernel's scale epilogue rounds the
    same single product ``s * L(v)``); anything else raises and the operator
    stays a generic callback."""

    __slots__ = ("lap", "scale", "muls")
    __array_ufunc__ = None   # numpy scalars defer to __rmul__

    def __init__(self, lap=None, scale=1.0, muls=0):
        self.lap, self.scale, self.muls = lap, scale, muls

    def __mul__(self, c):
        if self.lap is None or isinstance(c, (bool, np.bool_)) or not isinstance(
                c, (int, float, np.integer, np.floating)):
            raise TypeError("not a scaled Laplacian")
        return _StencilProbe(self.lap, self.scale * float(c), self.muls + 1)

    __rmul__ = __mul__


def as_fused_stencil(op):
    """The Laplacian3D an operator is, or None: a Laplacian3D itself, or a
    MatrixFreeOperator whose function is ``s * L(v)`` / ``L(v) * s`` / ``L(v)``
    for a Laplacian3D L of the same dimension (probed once, symbolically)."""
    if isinstance(op, Laplacian3D):
        return op
    if not isinstance(op, MatrixFreeOperator):
        return None
    try:
        r = op._apply_block(_StencilProbe())
    except Exception:
        return None
    if not isinstance(r, _StencilProbe) or r.lap is None or r.lap.dim != op.dim:
        return None
    lap = r.lap
    if type(lap) is not Laplacian3D or r.muls + (lap.scale != 1.0) > 1:
        return None   # nested scalings round twice: keep the callback
    return Laplacian3D(lap.grid, scale=r.scale, device=op.device)


class Laplacian3D(LinearOperator):
    """7-point Dirichlet Laplacian on a Grid3D, times ``scale``.

    ``scale=1`` is the reference's unscaled operator (operators.py:169-199);
    ``scale=(N+1)**2`` is the BASELINE harness s*L fused into the
    kernel's epilogue.  Applied by the TMA z-streaming kernel K1, bitwise
    equal to the reference.
    """

    def __init__(self, grid, scale=1.0, device=None):
        if not isinstance(grid, Grid3D):
            grid = Grid3D(*grid)
        super().__init__(grid.n, spd=True, device=device)
        self.grid = grid
        self.scale = float(scale)

    def __call__(self, x):
        if isinstance(x, _StencilProbe):
            if x.lap is not None:
                raise TypeError("not a scaled Laplacian")
            return _StencilProbe(self, self.scale, 0)
        return super().__call__(x)

    def apply_into(self, x: torch.Tensor, out: torch.Tensor) -> None:
        """out = A x for (n, ld) blocks with equal even leading dimension."""
        g = self.grid
        dv.stencil7(x, out, g.nx, g.ny, g.nz, self.scale)

    def stencil_gram_into(self, x, out, xb, m, kw, gram_out) -> None:
        """out = A x and gram_out = [xb[:, :m] ; x[:, :kw]]^T out[:, :kw] in
        one pass (K1+K5b)."""
        g = self.grid
        dv.stencil7_gram(x, out, g.nx, g.ny, g.nz, self.scale, xb, m, kw, gram_out)

    # widest column group one stencil launch takes (its plane tiles must fit
    # shared memory); wider blocks -- e.g. L(eye(n)) -- go in groups
    MAX_COLS = 32

    def _apply(self, x):
        n, k = x.shape
        if k > self.MAX_COLS:
            return torch.cat([self._apply(x[:, c:c + self.MAX_COLS])
                              for c in range(0, k, self.MAX_COLS)], dim=1)
        ld = dv.even(k)
        if x.stride(1) == 1 and x.stride(0) == ld and x.data_ptr() % 16 == 0 and k == ld:
            xin = x
        else:
            xin = torch.zeros((n, ld), dtype=torch.float64, device=x.device)
            xin[:, :k] = x
        out = torch.empty((n, ld), dtype=torch.float64, device=x.device)
        self.apply_into(xin, out)
        return out[:, :k] if ld != k else out

    def diagonal(self):
        return torch.full((self.dim,), 6.0 * self.scale, dtype=torch.float64,
                          device=self.device)


class ShiftedOperator(LinearOperator):
    """A + alpha B (operators.py:202-237)."""

    def __init__(self, a, b, alpha):
        if b is not None and b.dim != a.dim:
            raise ValueError(f"operator dimensions differ: A has {a.dim}, B has {b.dim}")
        super().__init__(a.dim, spd=a.spd and alpha >= 0.0 and (b is None or b.spd),
                         device=a.device)
        self.a, self.b, self.alpha = a, b, float(alpha)

    def _apply(self, x):
        y = self.a(x)
        return y + self.alpha * (x if self.b is None else self.b(x))

    def diagonal(self):
        da = self.a.diagonal()
        if da is None:
            return None
        if self.b is None:
            return da + self.alpha
        db = self.b.diagonal()
        return None if db is None else da + self.alpha * db


def laplacian3d(grid, scale=1.0):
    return Laplacian3D(grid, scale=scale)


def shift_operator(a, b, alpha):
    return ShiftedOperator(a, b, alpha)


class Preconditioner:
    """Block application of T (operators.py:250-277)."""

    def __init__(self, dim, device=None):
        if dim < 1:
            raise ValueError(f"preconditioner dimension must be positive, got {dim}")
        self.dim = int(dim)
        self.device = torch.device(device) if device is not None else _default_device()

    def __call__(self, x):
        t, single, host = _to_block(x, self.dim, "preconditioner", self.device)
        return _from_block(self._apply(t), single, host)

    def _apply(self, x):
        raise NotImplementedError


class IdentityPreconditioner(Preconditioner):
    def _apply(self, x):
        return x.clone()


class JacobiPreconditioner(Preconditioner):
    """T = diag(A)^{-1} (operators.py:285-298).  A constant diagonal (the
    Laplacian's 6s) is detected and applied as one scalar inside K4."""

    def __init__(self, diag, device=None):
        if isinstance(diag, torch.Tensor):
            dh = diag.detach().to("cpu", torch.float64).numpy()
        else:
            dh = np.asarray(diag, dtype=np.float64)
        if dh.ndim != 1:
            raise ValueError(f"diagonal must be 1-d, got shape {dh.shape}")
        if np.any(dh <= 0.0) or not np.all(np.isfinite(dh)):
            raise ValueError("Jacobi preconditioner needs a positive diagonal")
        super().__init__(dh.size, device=device)
        inv = 1.0 / dh
        self.uniform = bool(np.all(inv == inv[0]))
        self.inv_scalar = float(inv[0])
        self.inv_diag = torch.as_tensor(inv, device=self.device)

    def _apply(self, x):
        return self.inv_diag[:, None] * x


def jacobi_preconditioner(op, probe=False):
    """Jacobi from ``op.diagonal()`` (operators.py:319-334)."""
    d = op.diagonal()
    if d is None:
        if not probe:
            raise ValueError(
                "operator does not expose its diagonal; pass probe=True to "
                "recover it with dim operator applications")
        d = probe_diagonal(op)
    return JacobiPreconditioner(d, device=getattr(op, "device", None))


def probe_diagonal(op, chunk=256):
    """diag(A) from A applied to coordinate blocks (operators.py:301-316)."""
    n = op.dim
    d = torch.empty(n, dtype=torch.float64, device=op.device)
    for start in range(0, n, chunk):
        cols = min(chunk, n - start)
        e = torch.zeros((n, cols), dtype=torch.float64, device=op.device)
        idx = torch.arange(cols, device=op.device)
        e[start + idx, idx] = 1.0
        y = op(e)
        d[start:start + cols] = y[start + idx, idx]
    return d
