"""Inner-PCG preconditioner on the B200 path.

Reference: operators.py:336-427 -- ``PCGBreakdown``, ``pcg_solve``,
``InnerPCGPreconditioner``, ``inner_pcg_preconditioner``.  The reference runs
``pcg_solve`` column by column; here the k columns of a block advance
together (csrc/pcg.cu), each with its own scalars kept on the device, and
``A p`` for the built-in Laplacian is one fused stencil pass that also yields
the curvatures ``p_j^T A p_j`` (b2l_stencil7_gram with m = 0).  One host
synchronisation per preconditioner application (the breakdown flag).
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as dv
from .operators import (
    IdentityPreconditioner,
    JacobiPreconditioner,
    Laplacian3D,
    Preconditioner,
    _from_block,
    _to_block,
)

__all__ = ["PCGBreakdown", "pcg_solve", "InnerPCGPreconditioner", "inner_pcg_preconditioner"]


class PCGBreakdown(Exception):
    """Conjugate gradients hit a nonpositive curvature p.T A p, which means
    the operator (or preconditioner) is not positive definite
    (operators.py:336-338)."""


def _precond_mode(m, device):
    """(tmode, tinv, tvec) of the PCG's own preconditioner; tmode 3 = callback."""
    if m is None or isinstance(m, IdentityPreconditioner):
        return 0, 1.0, None
    if isinstance(m, JacobiPreconditioner):
        if m.uniform:
            return 1, m.inv_scalar, None
        return 2, 1.0, m.inv_diag.to(device)
    return 3, 1.0, None


def _aligned(t, k):
    return (t.dim() == 2 and t.stride(1) == 1 and t.stride(0) % 2 == 0 and t.stride(0) >= k
            and t.data_ptr() % 16 == 0 and t.dtype == torch.float64)


def pcg_block(a, m, B: torch.Tensor, max_iter: int, rtol: float = 0.0) -> torch.Tensor:
    """pcg_solve (operators.py:341-392) on every column of the CUDA (n, k)
    block B at once, from a zero start; returns the (n, k) iterate block."""
    n, k = B.shape
    dev = B.device
    ld = dv.even(k)
    if not _aligned(B, k):
        Bp = dv.new_block(n, ld, dev)
        Bp[:, :k] = B
    else:
        Bp = B
    tmode, tinv, tvec = _precond_mode(m, dev)
    X, R, P, AP = (dv.new_block(n, ld, dev) for _ in range(4))
    Z = dv.new_block(n, ld, dev) if tmode == 3 else None
    f64 = dict(dtype=torch.float64, device=dev)
    sums0 = torch.empty(2 * k, **f64)
    sums = torch.empty(2 * k, **f64)
    rz = [torch.empty(k, **f64), torch.empty(k, **f64)]
    done = [torch.zeros(k, dtype=torch.int32, device=dev) for _ in range(2)]
    G = torch.empty((k, k), **f64)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    reduce = getattr(a, "allreduce_", None) or (lambda t: t)
    fused = isinstance(a, Laplacian3D) or hasattr(a, "stencil_gram_into")

    def precond_into(src):
        z = m(src[:, :k])
        if not isinstance(z, torch.Tensor):
            z = torch.as_tensor(np.asarray(z, dtype=np.float64), device=dev)
        Z[:, :k] = z

    def apply_a():
        if fused:
            a.stencil_gram_into(P, AP, None, 0, k, G)
        else:
            y = a(P[:, :k])
            if not isinstance(y, torch.Tensor):
                y = torch.as_tensor(np.asarray(y, dtype=np.float64), device=dev)
            AP[:, :k] = y
            dv.gram(n, [(P, k)], [(AP, k)], out=G)
        reduce(G)

    if tmode == 3:
        precond_into(Bp)
    dv.pcg_init(n, k, Bp, X, R, P, Z, tmode, tinv, tvec, sums0)
    reduce(sums0)
    bb = sums0[:k].clone()
    rz[0].copy_(sums0[k:])
    cur = 0
    for step in range(max_iter):
        apply_a()
        dv.pcg_update(n, k, X, R, P, AP, G, k + 1, rz[cur], bb, done[cur], tmode, tinv, tvec,
                      sums, err)
        reduce(sums)
        if step == max_iter - 1:
            break                      # x is final; the reference's last p is unused
        if tmode == 3:
            precond_into(R)
            dv.pcg_dot(n, k, R, Z, bb, done[cur], sums)
            reduce(sums)
        dv.pcg_direction(n, k, R, P, Z, tmode, tinv, tvec, rz[cur], sums, bb, rtol, done[cur],
                         done[1 - cur], rz[1 - cur])
        cur = 1 - cur
    if int(err.item()):
        raise PCGBreakdown("nonpositive curvature p.T A p; operator is not SPD")
    return X[:, :k]


def pcg_solve(a, m, b, max_iter, rtol=0.0):
    """Preconditioned conjugate gradients for A x = b from a zero start
    (operators.py:341-392): at most ``max_iter`` steps, early stop once
    ``norm(r) <= rtol * norm(b)`` when rtol > 0.  b is an (n,) array or CUDA
    tensor; the result has the same kind."""
    host = not isinstance(b, torch.Tensor)
    bt = torch.as_tensor(np.asarray(b, dtype=np.float64)) if host else b
    if bt.dim() != 1 or bt.shape[0] != a.dim:
        raise ValueError(f"right-hand side has shape {tuple(bt.shape)}, expected ({a.dim},)")
    if max_iter < 1:
        raise ValueError(f"max_iter must be positive, got {max_iter}")
    dev = getattr(a, "device", None) or torch.device("cuda", torch.cuda.current_device())
    B = bt.to(device=dev, dtype=torch.float64)[:, None]
    x = pcg_block(a, m, B, int(max_iter), float(rtol))[:, 0]
    return x.cpu().numpy().copy() if host else x


class InnerPCGPreconditioner(Preconditioner):
    """A fixed number of PCG steps on A per column as the preconditioner
    (operators.py:395-421).  Deterministic, slightly nonlinear in its input
    (the CG step lengths depend on it), as in the reference."""

    def __init__(self, a, inner, steps):
        if steps < 1:
            raise ValueError(f"steps must be positive, got {steps}")
        if inner is not None and inner.dim != a.dim:
            raise ValueError(f"dimensions differ: operator has {a.dim}, inner "
                             f"preconditioner has {inner.dim}")
        super().__init__(a.dim, device=getattr(a, "device", None))
        self.a = a
        self.inner = inner
        self.steps = int(steps)

    def __call__(self, x):
        t, single, host = _to_block(x, self.dim, "preconditioner", self.device)
        return _from_block(self._apply(t), single, host)

    def _apply(self, x):
        return pcg_block(self.a, self.inner, x, self.steps, 0.0)


def inner_pcg_preconditioner(a, inner, steps):
    """Fixed-step PCG on A as a preconditioner; ``inner`` preconditions the
    PCG iteration itself (e.g. Jacobi, or None for plain CG)
    (operators.py:424-427)."""
    return InnerPCGPreconditioner(a, inner, steps)
