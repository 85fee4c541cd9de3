"""CPU stand-ins for the four native kernels, for testing the HOST logic of
paper_0705_2626_b200 (control flow, Gram bookkeeping, folding of Cholesky
factors, repair ladder) without a GPU.

Test infrastructure only: installed by monkeypatching inside tests; the
product package never imports this module and has no CPU fallback.
Each stand-in follows the contract in include/b200lobpcg.h on torch CPU
tensors with numpy arithmetic.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch

from oracle import lobpcg_oracle as orc


def _np(t):
    return t.detach().numpy()


def stencil7(x, out, nx, ny, nz, scale, halo=None, has_lo=False, has_hi=False):
    xa = _np(x)
    plane = nx * ny
    k = xa.shape[1]
    lo = _np(halo)[:plane] if has_lo else np.zeros((plane, k))
    hi = _np(halo)[plane:] if has_hi else np.zeros((plane, k))
    ext = np.vstack([lo, xa, hi])
    y = np.ascontiguousarray(orc.stencil7(ext, nx, ny, nz + 2, scale))
    # rows of the owned planes; z-neighbours beyond the ghosts are zero,
    # which is what the extended apply sees for the owned planes.
    out.copy_(torch.from_numpy(y[plane:plane + nz * plane]))


def gram(nrows, left, right, weighted_mask=0, weight=None, out=None, device=None, pair_mode=None):
    L = np.hstack([_np(t)[:nrows, :c] for t, c in left])
    Rs = []
    for j, (t, c) in enumerate(right):
        b = _np(t)[:nrows, :c]
        if (weighted_mask >> j) & 1:
            b = _np(weight)[:nrows, None] * b
        Rs.append(b)
    g = torch.from_numpy(L.T @ np.hstack(Rs))
    if out is not None:
        out.copy_(g)
        return out
    return g


def residual(nrows, m, x, ax, bdiag, lam_dev, tmode, tinv, tvec, wpos_dev, kw, w, want_ax,
             sums_out):
    X, AX = _np(x)[:, :m], _np(ax)[:, :m]
    lam = _np(lam_dev)
    bx = X if bdiag is None else _np(bdiag)[:, None] * X
    wf = AX - bx * lam
    s = np.concatenate([(wf * wf).sum(0), (AX * AX).sum(0) if want_ax else np.zeros(m)])
    sums_out.copy_(torch.from_numpy(s))
    if wpos_dev is not None and kw:
        pos = _np(wpos_dev)
        W = _np(w)
        for j in range(m):
            if pos[j] >= 0:
                v = wf[:, j]
                if tmode == 1:
                    v = tinv * v
                elif tmode == 2:
                    v = _np(tvec) * v
                W[:, pos[j]] = v
        if W.shape[1] > kw:
            W[:, kw:] = 0.0


def update(nrows, m, x, ax, cx, xo, axo, w=None, aw=None, kw=0, cw=None, p=None, ap=None,
           pcols=None, kp=0, cp=None, po=None, apo=None, x_plus_p=False):
    CX = _np(cx).reshape(m, m)
    have_p = (kw + kp) > 0

    def side(X, W, P, Xo, Po):
        pn = 0.0
        if have_p:
            parts = []
            if kw:
                parts.append(_np(W)[:, :kw] @ _np(cw).reshape(kw, m))
            if kp:
                parts.append(_np(P)[:, _np(pcols)[:kp]] @ _np(cp).reshape(kp, m))
            pn = parts[0] if len(parts) == 1 else parts[0] + parts[1]
            if Po is not None:
                Po.zero_()
                Po[:, :m] = torch.from_numpy(pn)
        xs = _np(X)[:, :m] @ CX
        if x_plus_p:
            xs = xs + pn
        Xo.zero_()
        Xo[:, :m] = torch.from_numpy(xs)

    side(x, w, p, xo, po)
    if ax is not None:
        side(ax, aw, ap, axo, apo)


@contextlib.contextmanager
def emulate(monkeypatch):
    """Route paper_0705_2626_b200's device wrappers to the CPU stand-ins."""
    from paper_0705_2626_b200 import _lib, device as dv, operators

    monkeypatch.setattr(dv, "stencil7", stencil7)
    monkeypatch.setattr(dv, "gram", gram)
    monkeypatch.setattr(dv, "residual", residual)
    monkeypatch.setattr(dv, "update", update)
    monkeypatch.setattr(_lib, "ensure_device", lambda i: None)
    monkeypatch.setattr(operators, "_default_device", lambda: torch.device("cpu"))
    yield
