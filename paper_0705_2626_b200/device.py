"""Device plumbing: torch tensors as (n, ld) fp64 blocks, and thin typed
wrappers around each libb200lobpcg entry point.

PyTorch is used only to own device memory and streams; all arithmetic on the
long dimension happens in the native kernels.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

F64 = torch.float64

# Native kernel launches issued through this module (bench.py reports it).
LAUNCHES = [0]


def even(k: int) -> int:
    """Leading dimension for k columns: even (16-B rows, TMA), at least 2."""
    return max(2, k + (k & 1))


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_block(t: torch.Tensor, what: str = "block") -> None:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == F64):
        raise TypeError(f"{what} must be a CUDA float64 tensor")
    if t.dim() != 2 or t.stride(1) != 1 or t.stride(0) % 2 or t.stride(0) < t.shape[1]:
        raise ValueError(f"{what} must be (n, k) with unit column stride and even row stride")
    if t.data_ptr() % 16:
        raise ValueError(f"{what} must be 16-byte aligned")


def new_block(n: int, ld: int, device) -> torch.Tensor:
    return torch.zeros((n, ld), dtype=F64, device=device)


def view_block(buf: torch.Tensor, n: int, ld: int) -> torch.Tensor:
    """(n, ld) view of the first n*ld doubles of a flat buffer."""
    return buf[: n * ld].view(n, ld)


# ------------------------------------------------------------------ kernels


def stencil7(x: torch.Tensor, out: torch.Tensor, nx: int, ny: int, nz: int,
             scale: float, halo: torch.Tensor | None = None, has_lo: bool = False,
             has_hi: bool = False) -> None:
    """out = scale * L7(x) on the ld columns of (n, ld) blocks (K1)."""
    lib = _lib.load()
    ld = x.stride(0)
    if out.stride(0) != ld:
        raise ValueError("stencil7: in/out leading dimensions differ")
    _lib.check(lib.b2l_stencil7(x.data_ptr(), out.data_ptr(), nx, ny, nz, ld,
                                halo.data_ptr() if halo is not None else None,
                                int(has_lo), int(has_hi), float(scale),
                                stream_ptr(x.device)), "b2l_stencil7")
    LAUNCHES[0] += 1


def seeded_fill(out: torch.Tensor, m: int, seed: int, row0: int = 0, low: float = -1.0,
                high: float = 1.0) -> None:
    """out[:, :m] = rows row0.. of Generator(PCG64(seed)).uniform(low, high, (N, m))
    generated on the device, bit for bit (K9, multivec.py:220-229)."""
    require_block(out, "seeded_fill out")
    st = np.random.PCG64(seed).state["state"]
    mask = (1 << 64) - 1
    s, inc = int(st["state"]), int(st["inc"])
    lib = _lib.load()
    _lib.check(lib.b2l_seeded_fill(out.data_ptr(), out.stride(0), out.shape[0], m, row0 * m,
                                   s >> 64, s & mask, inc >> 64, inc & mask, float(low),
                                   float(high), stream_ptr(out.device)), "b2l_seeded_fill")
    LAUNCHES[0] += 1


def stencil7_gram(x: torch.Tensor, out: torch.Tensor, nx: int, ny: int, nz: int,
                  scale: float, xb: torch.Tensor, m: int, kw: int, gram_out: torch.Tensor,
                  halo: torch.Tensor | None = None, has_lo: bool = False,
                  has_hi: bool = False) -> None:
    """out = scale*L7(x); gram_out = [xb[:, :m] ; x[:, :kw]]^T out[:, :kw]."""
    lib = _lib.load()
    ld = x.stride(0)
    if out.stride(0) != ld:
        raise ValueError("stencil7_gram: in/out leading dimensions differ")
    _lib.check(lib.b2l_stencil7_gram(
        x.data_ptr(), out.data_ptr(), nx, ny, nz, ld,
        halo.data_ptr() if halo is not None else None, int(has_lo), int(has_hi),
        float(scale), xb.data_ptr() if xb is not None else None,
        xb.stride(0) if xb is not None else 0, int(m), int(kw), gram_out.data_ptr(),
        stream_ptr(x.device)), "b2l_stencil7_gram")
    LAUNCHES[0] += 2


def lobpcg_step(nrows, m, x, ax, w, aw, kw, p, ap, kp, pcols, coef, xo, axo, po, apo,
                lam, bdiag, tmode, tinv, tvec, wpos, kwn, wo, want_ax, red_out) -> None:
    """F1: fused update + next residual + next non-AW Gram blocks."""
    lib = _lib.load()

    def ptr(t):
        return t.data_ptr() if t is not None else None

    _lib.check(lib.b2l_lobpcg_step(
        nrows, m, ptr(x), ptr(ax), x.stride(0), ptr(w), ptr(aw),
        w.stride(0) if w is not None else 0, int(kw), ptr(p), ptr(ap), int(kp), ptr(pcols),
        ptr(coef), ptr(xo), ptr(axo), ptr(po), ptr(apo), ptr(lam), ptr(bdiag), int(tmode),
        float(tinv), ptr(tvec), ptr(wpos), int(kwn), ptr(wo),
        wo.stride(0) if wo is not None else 0, int(want_ax), ptr(red_out),
        stream_ptr(x.device)), "b2l_lobpcg_step")
    LAUNCHES[0] += 2


def _blk(t: torch.Tensor, cols: int) -> _lib.b2l_block:
    return _lib.b2l_block(t.data_ptr(), t.stride(0), cols)


def gram(nrows: int, left, right, weighted_mask: int = 0,
         weight: torch.Tensor | None = None, out: torch.Tensor | None = None,
         device=None, pair_mode=None) -> torch.Tensor:
    """Device (sum left cols, sum right cols) matrix [L]^T diag(w)^? [R] (K5).

    left/right: sequences of (tensor (n, ld), cols).  pair_mode: optional
    (len(left), len(right)) array of 0 (skip) / 1 (full) / 2 (upper only).
    """
    lib = _lib.load()
    a = sum(c for _, c in left)
    b = sum(c for _, c in right)
    dev = device if device is not None else left[0][0].device
    if out is None:
        out = torch.empty((a, b), dtype=F64, device=dev)
    L = (_lib.b2l_block * len(left))(*[_blk(t, c) for t, c in left])
    R = (_lib.b2l_block * len(right))(*[_blk(t, c) for t, c in right])
    pm = None
    if pair_mode is not None:
        pm = np.ascontiguousarray(pair_mode, dtype=np.uint8).tobytes()
        if len(pm) != len(left) * len(right):
            raise ValueError("pair_mode must be len(left) x len(right)")
    _lib.check(lib.b2l_gram(nrows, L, len(left), R, len(right), int(weighted_mask),
                            weight.data_ptr() if weight is not None else None, pm,
                            out.data_ptr(), stream_ptr(dev)), "b2l_gram")
    LAUNCHES[0] += 2
    return out


def residual(nrows: int, m: int, x: torch.Tensor, ax: torch.Tensor,
             bdiag: torch.Tensor | None, lam_dev: torch.Tensor, tmode: int,
             tinv: float, tvec: torch.Tensor | None, wpos_dev: torch.Tensor | None,
             kw: int, w: torch.Tensor | None, want_ax: bool,
             sums_out: torch.Tensor) -> None:
    """K4+K2: W[:, wpos] = T(AX - BX lam), squared norms into sums_out (2m)."""
    lib = _lib.load()
    _lib.check(lib.b2l_residual(
        nrows, m, x.data_ptr(), ax.data_ptr(), x.stride(0),
        bdiag.data_ptr() if bdiag is not None else None, lam_dev.data_ptr(),
        int(tmode), float(tinv), tvec.data_ptr() if tvec is not None else None,
        wpos_dev.data_ptr() if wpos_dev is not None else None, int(kw),
        w.data_ptr() if w is not None else None, w.stride(0) if w is not None else 0,
        int(want_ax), sums_out.data_ptr(), stream_ptr(x.device)), "b2l_residual")
    LAUNCHES[0] += 2


def update(nrows: int, m: int, x, ax, cx, xo, axo, w=None, aw=None, kw=0, cw=None,
           p=None, ap=None, pcols=None, kp=0, cp=None, po=None, apo=None,
           x_plus_p=False) -> None:
    """K6: P' = W Cw + P[:, pcols] Cp ; X' = X Cx (+P') ; A-side twins."""
    lib = _lib.load()

    def ptr(t):
        return t.data_ptr() if t is not None else None

    _lib.check(lib.b2l_update(
        nrows, m, ptr(x), ptr(ax), x.stride(0) if x is not None else 0, ptr(cx),
        ptr(w), ptr(aw), w.stride(0) if w is not None else 0, int(kw), ptr(cw),
        ptr(p), ptr(ap), p.stride(0) if p is not None else 0, ptr(pcols), int(kp), ptr(cp),
        ptr(xo), ptr(axo), xo.stride(0), ptr(po), ptr(apo),
        po.stride(0) if po is not None else 0, int(bool(x_plus_p)),
        stream_ptr(xo.device)), "b2l_update")
    LAUNCHES[0] += 1


# ------------------------------------------------ column-batched PCG (K10)


def _p(t):
    return t.data_ptr() if t is not None else None


def pcg_init(nrows, k, b, x, r, p, z, tmode, tinv, tvec, sums_out):
    lib = _lib.load()
    _lib.check(lib.b2l_pcg_init(nrows, k, b.data_ptr(), b.stride(0), x.data_ptr(),
                                r.data_ptr(), p.data_ptr(), x.stride(0), _p(z), int(tmode),
                                float(tinv), _p(tvec), sums_out.data_ptr(),
                                stream_ptr(x.device)), "b2l_pcg_init")
    LAUNCHES[0] += 2


def pcg_update(nrows, k, x, r, p, ap, pap, pap_stride, rz, bb, done, tmode, tinv, tvec,
               sums_out, err):
    lib = _lib.load()
    _lib.check(lib.b2l_pcg_update(nrows, k, x.data_ptr(), r.data_ptr(), p.data_ptr(),
                                  ap.data_ptr(), x.stride(0), pap.data_ptr(), int(pap_stride),
                                  rz.data_ptr(), bb.data_ptr(), done.data_ptr(), int(tmode),
                                  float(tinv), _p(tvec), sums_out.data_ptr(), err.data_ptr(),
                                  stream_ptr(x.device)), "b2l_pcg_update")
    LAUNCHES[0] += 2


def pcg_dot(nrows, k, r, z, bb, done, sums_out):
    lib = _lib.load()
    _lib.check(lib.b2l_pcg_dot(nrows, k, r.data_ptr(), z.data_ptr(), r.stride(0),
                               bb.data_ptr(), done.data_ptr(), sums_out.data_ptr(),
                               stream_ptr(r.device)), "b2l_pcg_dot")
    LAUNCHES[0] += 2


def pcg_direction(nrows, k, r, p, z, tmode, tinv, tvec, rz, sums, bb, rtol, done, done_next,
                  rz_next):
    lib = _lib.load()
    _lib.check(lib.b2l_pcg_direction(nrows, k, r.data_ptr(), p.data_ptr(), r.stride(0), _p(z),
                                     int(tmode), float(tinv), _p(tvec), rz.data_ptr(),
                                     sums.data_ptr(), bb.data_ptr(), float(rtol),
                                     done.data_ptr(), done_next.data_ptr(), rz_next.data_ptr(),
                                     stream_ptr(r.device)), "b2l_pcg_direction")
    LAUNCHES[0] += 1


# ------------------------------------------------------- small transfers


def to_device(a: np.ndarray, device, dtype=F64) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype,
                                                        non_blocking=False)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()
