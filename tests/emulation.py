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


def stencil7_gram(x, out, nx, ny, nz, scale, xb, m, kw, gram_out, halo=None, has_lo=False,
                  has_hi=False):
    stencil7(x, out, nx, ny, nz, scale, halo, has_lo, has_hi)
    L = np.hstack([_np(xb)[:, :m], _np(x)[:, :kw]]) if m else _np(x)[:, :kw]
    gram_out.copy_(torch.from_numpy(L.T @ _np(out)[:, :kw]))


def lobpcg_step(nrows, m, x, ax, w, aw, kw, p, ap, kp, pcols, coef, xo, axo, po, apo, lam,
                bdiag, tmode, tinv, tvec, wpos, kwn, wo, want_ax, red_out):
    c = _np(coef)
    cx = c[:m * m]
    cw = c[m * m:m * m + kw * m]
    cp = c[m * m + kw * m:m * m + kw * m + kp * m]
    update(nrows, m, x, ax, torch.from_numpy(cx.copy()), xo, axo, w=w, aw=aw, kw=kw,
           cw=torch.from_numpy(cw.copy()), p=p, ap=ap, pcols=pcols, kp=kp,
           cp=torch.from_numpy(cp.copy()), po=po, apo=apo, x_plus_p=True)
    sums = torch.zeros(2 * m, dtype=torch.float64)
    residual(nrows, m, xo, axo, bdiag, lam, tmode, tinv, tvec, wpos, kwn, wo, want_ax, sums)
    Xn, Wn, Pn, APn = (_np(t)[:, :k] for t, k in ((xo, m), (wo, kwn), (po, m), (apo, m)))
    L = np.hstack([Xn, Wn, Pn])
    B = L * (_np(bdiag)[:, None] if bdiag is not None else 1.0)
    G = L.T @ np.hstack([B, APn])
    red_out[:2 * m + G.size] = torch.from_numpy(np.concatenate([_np(sums), G.ravel()]))


def seeded_fill(out, m, seed, row0=0, low=-1.0, high=1.0):
    bg = np.random.PCG64(seed)
    if row0:
        bg.advance(row0 * m)
    vals = np.random.Generator(bg).uniform(low, high, size=(out.shape[0], m))
    out[:, :m] = torch.from_numpy(vals)


def _tapply(tmode, tinv, tvec, v):
    if tmode == 1:
        return tinv * v
    if tmode == 2:
        return _np(tvec)[:, None] * v
    return v


def pcg_init(nrows, k, b, x, r, p, z, tmode, tinv, tvec, sums_out):
    bv = _np(b)[:, :k]
    zv = _np(z)[:, :k] if tmode == 3 else _tapply(tmode, tinv, tvec, bv)
    x[:, :k] = 0.0
    r[:, :k] = torch.from_numpy(bv.copy())
    p[:, :k] = torch.from_numpy(np.ascontiguousarray(zv))
    sums_out[:] = torch.from_numpy(np.concatenate([(bv * bv).sum(0), (bv * zv).sum(0)]))


def pcg_update(nrows, k, x, r, p, ap, pap, pap_stride, rz, bb, done, tmode, tinv, tvec,
               sums_out, err):
    papv = _np(pap).ravel()[::pap_stride][:k]
    live = (_np(done)[:k] == 0) & (_np(bb)[:k] != 0.0)
    if np.any(live & (~(papv > 0) | ~np.isfinite(papv))):
        err[0] = 1
    alpha = np.where(live, _np(rz)[:k] / np.where(live, papv, 1.0), 0.0)
    X, R, P, AP = (_np(t)[:, :k] for t in (x, r, p, ap))
    Xn = np.where(live, X + alpha * P, X)
    Rn = np.where(live, R - alpha * AP, R)
    x[:, :k] = torch.from_numpy(np.ascontiguousarray(Xn))
    r[:, :k] = torch.from_numpy(np.ascontiguousarray(Rn))
    s0 = np.where(live, (Rn * _tapply(tmode, tinv, tvec, Rn)).sum(0), 0.0) if tmode != 3 else np.zeros(k)
    s1 = np.where(live, (Rn * Rn).sum(0), 0.0)
    sums_out[:] = torch.from_numpy(np.concatenate([s0, s1]))


def pcg_dot(nrows, k, r, z, bb, done, sums_out):
    live = (_np(done)[:k] == 0) & (_np(bb)[:k] != 0.0)
    R, Z = _np(r)[:, :k], _np(z)[:, :k]
    sums_out[:] = torch.from_numpy(np.concatenate([np.where(live, (R * Z).sum(0), 0.0),
                                                   np.where(live, (R * R).sum(0), 0.0)]))


def pcg_direction(nrows, k, r, p, z, tmode, tinv, tvec, rz, sums, bb, rtol, done, done_next,
                  rz_next):
    sv = _np(sums)
    rzn, rr = sv[:k], sv[k:2 * k]
    bbv, rzv = _np(bb)[:k], _np(rz)[:k]
    stop = (_np(done)[:k] != 0) | (bbv == 0.0)
    if rtol > 0:
        stop |= np.sqrt(rr) <= rtol * np.sqrt(bbv)
    stop |= rzn == 0.0
    done_next[:k] = torch.from_numpy(stop.astype(np.int32))
    rz_next[:k] = torch.from_numpy(np.where(stop, rzv, rzn))
    R, P = _np(r)[:, :k], _np(p)[:, :k]
    Z = _np(z)[:, :k] if tmode == 3 else _tapply(tmode, tinv, tvec, R)
    beta = np.where(stop, 0.0, rzn / np.where(stop, 1.0, rzv))
    p[:, :k] = torch.from_numpy(np.ascontiguousarray(np.where(stop, P, Z + beta * P)))


@contextlib.contextmanager
def emulate(monkeypatch):
    """Route paper_0705_2626_b200's device wrappers to the CPU stand-ins."""
    from paper_0705_2626_b200 import _lib, device as dv, operators

    monkeypatch.setattr(dv, "stencil7", stencil7)
    monkeypatch.setattr(dv, "gram", gram)
    monkeypatch.setattr(dv, "residual", residual)
    monkeypatch.setattr(dv, "update", update)
    monkeypatch.setattr(dv, "stencil7_gram", stencil7_gram)
    monkeypatch.setattr(dv, "lobpcg_step", lobpcg_step)
    monkeypatch.setattr(dv, "seeded_fill", seeded_fill)
    for name in ("pcg_init", "pcg_update", "pcg_dot", "pcg_direction"):
        monkeypatch.setattr(dv, name, globals()[name])
    monkeypatch.setattr(_lib, "ensure_device", lambda i: None)
    monkeypatch.setattr(operators, "_default_device", lambda: torch.device("cpu"))
    yield
