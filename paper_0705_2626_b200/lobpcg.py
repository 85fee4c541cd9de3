"""LOBPCG with soft locking on B200: the reference's ``solve`` entry point
(lobpcg.py:343-577) with every long-dimension operation on the GPU.

Control flow, thresholds, the lock test, the basis-repair ladder, the drift
repair and the status strings are the reference's, evaluated on the host on
small matrices.  What changes is where the tall work happens and how much of
it there is per iteration (steady state, built-in operators):

  reference (numpy), per iteration           here (libb200lobpcg, sm_100a)
  -----------------------------------------  ---------------------------------
  Ritz update, 6 multiplies   :520-540       F1 b2l_lobpcg_step (one pass):
  drift gram X^T B X          :419             update, next residual + norms,
  W_full, norms, T(W_J)       :429-467         next W, every Gram block not
  b_orthonormalize(W), P_J    :176-178,490     involving A W (DMMA)
  _project_pencil 6 grams     :328-338
  a(w)                        :482           K1+K5b b2l_stencil7_gram (one
  gram(x, aw), gram(w, aw)    :325-327         pass): A W and [X W]^T A W
  Cholesky-QR, gen_sym_eig    :501-519       host fp64 (LAPACK), unchanged
  tri_solve_right (W, P, AP)  :177,491       folded into the coefficients

The Cholesky-QR factors of W and P are never applied to the tall blocks: the
Gram blocks of the normalised vectors are R^-T G R^-1 of the raw ones, and
R^-1 is folded into the update coefficients.  BX is d*X computed on the fly
for diagonal B (the reference carries BX by recurrence).  Both change
results only at rounding level (tests/test_gpu_solve.py holds the trajectory
to the reference's own 1-ulp perturbation band).

The first iteration, drift repairs and the exit refresh use the standalone
kernels (b2l_gram / b2l_residual / b2l_update); so do block sizes whose Gram
does not fit the fused kernels (m > 16) and generic operators.
"""

from __future__ import annotations

import contextlib
import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv
from .operators import (
    DiagonalOperator,
    IdentityOperator,
    IdentityPreconditioner,
    JacobiPreconditioner,
    as_fused_stencil,
)
from .small import (NativeRitz, NotSPD, RitzFailure, chol_solve, cholesky, gen_sym_eig,
                    scaled_cholesky, sym_eig)

__all__ = [
    "SolverConfig",
    "HistoryEntry",
    "SolverReport",
    "solve",
    "solve_staged",
    "device_options",
    "LOBPCGRun",
    "project_pencil",
    "Constraints",
    "apply_constraints",
    "b_orthonormalize",
]

PIVOT_FLOOR = 1e-8   # lobpcg.py:57
DRIFT_LIMIT = 1e-11  # lobpcg.py:66


@dataclass(frozen=True)
class SolverConfig:
    """Same knobs and defaults as the reference (lobpcg.py:69-98)."""

    block_size: int = 1
    tol: float = 1e-6
    max_iter: int = 200
    seed: int = 0
    lock_history: bool = True
    verbosity: int = 0
    relative_tol: bool = False
    check_invariants: bool = False

    def validate(self):
        if self.block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {self.block_size}")
        if not self.tol > 0.0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")


@dataclass(frozen=True)
class HistoryEntry:
    """Per-iteration snapshot (lobpcg.py:203-225)."""

    iteration: int
    ritz: np.ndarray | None
    residual_norms: np.ndarray | None
    active: np.ndarray
    locked_now: tuple
    fallbacks: int
    constraint_violation: float | None
    stage: int = 0


@dataclass(frozen=True)
class SolverReport:
    """Result of a solve (lobpcg.py:228-263).  ``eigenvectors`` is a host
    numpy (n, m) array unless ``device_options(return_device=True)`` is in
    effect, in which case it is the CUDA (n, m) tensor."""

    eigenvalues: np.ndarray
    eigenvectors: object
    iterations_used: int
    converged: np.ndarray
    residual_norms: np.ndarray
    lock_iterations: np.ndarray
    history: tuple
    status: str
    basis_fallbacks: int = 0
    stages: tuple = ()

    @property
    def all_converged(self):
        return bool(self.converged.all())

    @property
    def ok(self):
        return not self.status.startswith("Failed")


# Device options live outside SolverConfig so the reference signature and
# config stay untouched.
_OPTS = {"return_device": False, "timer": None, "fused": True}


@contextlib.contextmanager
def device_options(return_device: bool | None = None, timer=None, fused: bool | None = None):
    """Scoped device options.

    return_device -- keep eigenvectors on the GPU (the 464^3 x 8 block is 6.4 GB)
    timer         -- callable(name, fn) wrapping each kernel launch (bench.py
                     times kernels with CUDA events through it)
    fused         -- False forces the unfused standalone kernels (tests)
    """
    old = dict(_OPTS)
    if return_device is not None:
        _OPTS["return_device"] = bool(return_device)
    if timer is not None:
        _OPTS["timer"] = timer
    if fused is not None:
        _OPTS["fused"] = bool(fused)
    try:
        yield
    finally:
        _OPTS.clear()
        _OPTS.update(old)


def _timed(name, fn):
    t = _OPTS["timer"]
    return fn() if t is None else t(name, fn)


class _Failure(Exception):
    pass


# Gram block-pair modes (include/b200lobpcg.h): only what the host reads.
_UPPER = np.array([[2]], dtype=np.uint8)
# L = [X, W, P], R = [BX, BW, BP, AP]   (the F1 layout).  X^T B X is left
# out: Rayleigh-Ritz takes it as I and the drift check has its own Gram
_MODES_P = np.array([[0, 1, 1, 1],
                     [0, 2, 1, 1],
                     [0, 0, 2, 1]], dtype=np.uint8)
# L = [X, W], R = [BX, BW]
_MODES_NOP = np.array([[0, 1],
                       [0, 2]], dtype=np.uint8)


def _mirror_upper(g):
    return np.triu(g) + np.triu(g, 1).T


def _tilesets(a, b):
    """8x8 tile blocks (2x4 tiles each) of an a x b Gram (gram_tile.cuh)."""
    ni, nj = (a + 7) // 8, (b + 7) // 8
    return ((ni + 1) // 2) * ((nj + 3) // 4)


def _host_buf(count, dtype=torch.float64):
    return torch.empty(count, dtype=dtype, pin_memory=torch.cuda.is_available())


class _Pinned:
    """Pinned host staging for the small per-iteration transfers."""

    def __init__(self, dev, nd, ni):
        self.dev = dev
        self.hd = _host_buf(nd)
        self.dd = torch.empty(nd, dtype=torch.float64, device=dev)
        self.hi = _host_buf(ni, torch.int32)
        self.di = torch.empty(ni, dtype=torch.int32, device=dev)
        self.hd_np = self.hd.numpy()
        self.hi_np = self.hi.numpy()
        self._views = {}

    def upload(self, dparts, iparts):
        """Pack float64 / int32 arrays, one H2D copy each; returns device views.

        The pinned staging is reused by the next call: the stream orders the
        copy before any later host write only because every caller
        synchronises the stream once per iteration (LOBPCGRun.step)."""
        outs_d, outs_i = [], []
        o = 0
        for a in dparts:
            a = np.asarray(a, dtype=np.float64).ravel()
            self.hd_np[o:o + a.size] = a
            outs_d.append((o, a.size))
            o += a.size
        if o:
            self._copy(self.dd, self.hd, o)
        oi = 0
        for a in iparts:
            a = np.asarray(a, dtype=np.int32).ravel()
            self.hi_np[oi:oi + a.size] = a
            outs_i.append((oi, a.size))
            oi += a.size
        if oi:
            self._copy(self.di, self.hi, oi)
        return ([self._view(self.dd, s, k) for s, k in outs_d],
                [self._view(self.di, s, k) for s, k in outs_i])

    def _view(self, buf, s, k):
        key = (id(buf), s, k)
        v = self._views.get(key)
        if v is None:
            v = self._views[key] = buf[s:s + k]
        return v

    def _copy(self, dst, src, count):
        self._view(dst, 0, count).copy_(self._view(src, 0, count), non_blocking=True)


def _device_of(op, default=None):
    dev = getattr(op, "device", None)
    if dev is not None:
        return dev
    if default is not None:
        return default
    from . import operators

    return operators._default_device()


def _padded_block(y, device):
    """(n, k) array / tensor -> CUDA (n, even(k)) float64 block (zero pad)."""
    if isinstance(y, torch.Tensor):
        t = y.detach().to(device=device, dtype=torch.float64)
    else:
        arr = np.asarray(y, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"constraint basis must be 2-d, got shape {arr.shape}")
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    if t.dim() != 2:
        raise ValueError(f"constraint basis must be 2-d, got shape {tuple(t.shape)}")
    n, k = t.shape
    out = dv.new_block(n, dv.even(k), device)
    out[:, :k] = t
    return out


class Constraints:
    """Hard-locking basis: iterates are kept B-orthogonal to span(Y)
    (reference lobpcg.py:101-128).

    Holds Y, the cached product BY (CUDA (n, k) views of padded blocks) and
    the host Cholesky factor of Y^T B Y, so projections cost one tall Gram,
    two small triangular solves and one tall update -- no operator
    applications.
    """

    def __init__(self, y, by, yby_chol):
        dev = y.device if isinstance(y, torch.Tensor) else _device_of(None)
        self._y = _padded_block(y, dev)
        self._by = self._y if by is y else _padded_block(by, dev)
        self._k = int(y.shape[1] if hasattr(y, "shape") else np.asarray(y).shape[1])
        self.yby_chol = np.asarray(yby_chol, dtype=np.float64)

    @property
    def y(self):
        return self._y[:, :self._k]

    @property
    def by(self):
        return self._by[:, :self._k]

    @classmethod
    def from_basis(cls, y, b=None):
        """Build constraints from a basis block, computing BY and the factor
        (lobpcg.py:114-124).  Raises NotSPD if the columns of y are not
        linearly B-independent."""
        dev = _device_of(b, y.device if isinstance(y, torch.Tensor) else None)
        Y = _padded_block(y, dev)
        n, k = Y.shape[0], int(y.shape[1] if hasattr(y, "shape") else np.asarray(y).shape[1])
        if b is None or isinstance(b, IdentityOperator):
            BY = Y
        elif isinstance(b, DiagonalOperator):
            BY = b.d.to(dev)[:, None] * Y
        else:
            BY = _padded_block(b(Y[:, :k]), dev)
        g = dv.to_host(dv.gram(n, [(Y, k)], [(BY, k)]))
        r = cholesky(g)                     # NotSPD propagates (multivec.py:89-122)
        obj = cls.__new__(cls)
        obj._y, obj._by, obj._k = Y, BY, int(k)
        obj.yby_chol = r
        return obj

    @property
    def count(self):
        return self._k


def b_orthonormalize(x, bx, pivot_floor=0.0):
    """B-orthonormalize a block (lobpcg.py:147-179): returns (x', bx', r)
    with x'^T bx' = I and x ~ x' r (r upper, the column scaling included).
    Columns are scaled to unit B-norm before the Cholesky factorisation;
    raises NotSPD(pivot) for a nonpositive / non-finite B-norm or a pivot at
    or below pivot_floor.  On the device: one Gram (K5), the small factor on
    the host, one update (K6) per block; bx may alias x (B = I).  CUDA
    tensors in -> CUDA tensors out; arrays in -> arrays out."""
    host = not isinstance(x, torch.Tensor)
    shared = bx is x
    dev = x.device if not host else _device_of(None)
    X = _padded_block(x, dev)
    BX = X if shared else _padded_block(bx, dev)
    n = X.shape[0]
    k = int(x.shape[1] if hasattr(x, "shape") else np.asarray(x).shape[1])
    g = _mirror_upper(dv.to_host(dv.gram(n, [(X, k)], [(BX, k)], pair_mode=_UPPER)))
    reff, inv = scaled_cholesky(g, pivot_floor)
    M = dv.to_device(inv, dev)
    XO = dv.new_block(n, X.shape[1], dev)
    dv.update(n, k, X, None, M, XO, None)
    if shared:
        BXO = XO
    else:
        BXO = dv.new_block(n, X.shape[1], dev)
        dv.update(n, k, BX, None, M, BXO, None)
    xo, bxo = XO[:, :k], BXO[:, :k]
    if host:
        xo = dv.to_host(xo).copy()
        bxo = xo if shared else dv.to_host(bxo).copy()
    return xo, bxo, reff


def project_pencil(lam, x, ax, w, aw, bw, pj, apj, bpj, bx, exact_diagonal=False):
    """The projected pencil (gramA, gramB) on the basis [x, w, p]
    (`_project_pencil`, lobpcg.py:299-340), upper-triangular blocks only, from
    tall blocks on the GPU (K5 Grams; CUDA (n, k) tensors or host arrays).

    The diagonal blocks are Lambda and identities by construction;
    ``exact_diagonal=True`` computes them instead (lobpcg.py:317-321,
    :334-336): the reference's cross-check of the B-orthonormality the solver
    assumes.  The solver itself folds the orthonormalisation into its
    coefficients and never calls this; it is the diagnostic twin of the
    reference's private helper."""
    from . import multivec as mv

    lam = np.asarray(lam, dtype=np.float64)
    m = int(x.shape[1])
    nw = int(w.shape[1])
    npj = 0 if pj is None else int(pj.shape[1])
    dim = m + nw + npj
    ga = np.zeros((dim, dim))
    gb = np.zeros((dim, dim))
    sx, sw, sp = slice(0, m), slice(m, m + nw), slice(m + nw, dim)
    if exact_diagonal:
        ga[sx, sx] = mv.gram(x, ax)
        gb[sx, sx] = mv.gram(x, bx)
        gb[sw, sw] = mv.gram(w, bw)
    else:
        ga[sx, sx] = np.diag(lam)
        gb[sx, sx] = np.eye(m)
        gb[sw, sw] = np.eye(nw)
    ga[sw, sw] = mv.gram(w, aw)
    ga[sx, sw] = mv.gram(x, aw)
    gb[sx, sw] = mv.gram(x, bw)
    if npj:
        ga[sx, sp] = mv.gram(x, apj)
        ga[sw, sp] = mv.gram(w, apj)
        gb[sx, sp] = mv.gram(x, bpj)
        gb[sw, sp] = mv.gram(w, bpj)
        ga[sp, sp] = mv.gram(pj, apj)
        gb[sp, sp] = mv.gram(pj, bpj) if exact_diagonal else np.eye(npj)
    return ga, gb


def apply_constraints(x, constraints, b=None):
    """x - Y (Y^T B Y)^{-1} (BY)^T x  (lobpcg.py:131-144); b is accepted for
    call-site symmetry and not consulted.  x: CUDA (n, k) tensor (returned
    as a new tensor) or array (returned as numpy)."""
    if constraints is None or constraints.count == 0:
        return x
    host = not isinstance(x, torch.Tensor)
    X = _padded_block(x, constraints._y.device)
    n, k = X.shape[0], int(x.shape[1] if hasattr(x, "shape") else np.asarray(x).shape[1])
    out = dv.new_block(n, X.shape[1], X.device)
    _project_into(X, k, constraints, out)
    res = out[:, :k]
    return dv.to_host(res).copy() if host else res


def _project_into(X, k, cons, out, reduce=None):
    """out[:, :k] = X - Y chol_solve(R, (BY)^T X) on the device (K5 + K6)."""
    n, c = X.shape[0], cons.count
    g = dv.gram(n, [(cons._by, c)], [(X, k)])
    if reduce is not None:
        reduce(g)
    coef = chol_solve(cons.yby_chol, dv.to_host(g))
    eye = dv.to_device(np.eye(k), X.device)
    mc = dv.to_device(-coef, X.device)
    dv.update(n, k, X, None, eye, out, None, w=cons._y, kw=c, cw=mc, x_plus_p=True)


class LOBPCGRun:
    """One LOBPCG solve on the device, stepped iteration by iteration.

    ``solve`` drives it to completion; bench.py steps it to time individual
    iterations.  Mirrors lobpcg.py:375-577 in control flow.
    """

    def __init__(self, a, b=None, t=None, y=None, x0=None, config=None):
        cfg = config if config is not None else SolverConfig()
        cfg.validate()
        self.cfg = cfg
        m = cfg.block_size
        n = a.dim
        ncons = 0 if y is None else y.count
        if m > n - ncons:
            raise ValueError(f"block size {m} exceeds the constrained problem dimension "
                             f"{n} - {ncons}")
        self.cons = y if ncons else None
        self.a, self.b, self.t = a, b, t
        # z-slab runs (distributed.SlabLaplacian3D): blocks hold this rank's
        # rows; every small reduction is summed over ranks before the host
        # reads it, so all ranks take identical decisions
        self.n_global = n
        rows = int(getattr(a, "local_rows", n))
        self._allreduce = getattr(a, "allreduce_", None)
        self.m, self.n = m, rows
        self.dev = getattr(a, "device", None) or torch.device("cuda", torch.cuda.current_device())
        _lib.load()
        _lib.ensure_device(self.dev.index if self.dev.index is not None else 0)

        # ---- operator kinds
        # the built-in stencil, or the reference harness MatrixFreeOperator(n,
        # lambda v: s * L(v)) recognised as one (operators.as_fused_stencil)
        lap = as_fused_stencil(a)
        if lap is not None and lap is not a:
            self.a = a = lap
        self.fused_a = lap is not None
        # B: none / identity (BX = X), diagonal (a row weight streamed by the
        # kernels, never materialised), or any other callable on CUDA (n, k)
        # float64 blocks -- then BX, BW, BP are carried by recurrence as the
        # reference does (lobpcg.py:396, :476, :533-538)
        self.bdiag = None
        self.b_generic = None
        if b is not None and not isinstance(b, IdentityOperator):
            bdim = getattr(b, "dim", n)
            if bdim != n:
                raise ValueError(f"B has dimension {bdim}, expected {n}")
            if isinstance(b, DiagonalOperator):
                self.bdiag = b.d.to(self.dev)
            elif callable(b):
                self.b_generic = b
            else:
                raise TypeError("b must be an operator or a callable on (n, k) blocks")
        self.tmode, self.tinv, self.tvec, self.t_generic = 0, 1.0, None, None
        if t is None or isinstance(t, IdentityPreconditioner):
            pass
        elif isinstance(t, JacobiPreconditioner):
            if t.uniform:
                self.tmode, self.tinv = 1, t.inv_scalar
            else:
                self.tmode, self.tvec = 2, t.inv_diag.to(self.dev)
        else:
            self.t_generic = t
        fused = _OPTS["fused"]
        # F1 holds the whole next-step Gram in one CTA; stencil+Gram likewise
        # (hard constraints project W between the residual and A W: F1 forms
        # W' inside its pass, so a constrained run takes the unfused kernels)
        self.use_f1 = (fused and _tilesets(3 * m, 4 * m) <= 8 and self.cons is None
                       and self.b_generic is None)
        self.use_sgram = fused and self.fused_a and _tilesets(2 * m, m) <= 8

        # ---- initial block (lobpcg.py:386-393)
        if x0 is not None:
            if isinstance(x0, torch.Tensor):
                # copied straight into the X block below (one H2D from a
                # pinned host tensor, no intermediate device copy); the
                # finiteness check runs on the device after the copy
                x0t = x0.detach()
                if tuple(x0t.shape) not in ((n, m), (rows, m)):
                    raise ValueError(f"x0 has shape {tuple(x0t.shape)}, expected ({n}, {m})")
            else:
                # no host copy (the block is copied to the device below) and
                # the finiteness check runs on the device after the upload
                xh = np.asarray(x0, dtype=np.float64)
                # a z-slab run also accepts this rank's rows only
                if xh.shape not in ((n, m), (rows, m)):
                    raise ValueError(f"x0 has shape {xh.shape}, expected ({n}, {m})")
                x0t = xh
        else:
            # seeded block generated on the device (K9), bit for bit
            # Generator(PCG64(seed)).uniform(-1, 1, (n, m)) (multivec.py:220-229);
            # a z-slab rank generates its own rows only
            x0t = None
        if rows != n and x0t is not None and x0t.shape[0] == n:
            r0 = a.part.z0 * a.plane
            x0t = x0t[r0:r0 + rows]
        if b is not None and self.bdiag is not None and self.bdiag.numel() == n and rows != n:
            r0 = a.part.z0 * a.plane
            self.bdiag = self.bdiag[r0:r0 + rows].contiguous()
        n = rows

        if self.cons is not None:
            c = self.cons
            if c._y.shape[0] not in (self.n_global, rows):
                raise ValueError(f"constraint basis has {c._y.shape[0]} rows, expected {self.n_global}")
            if c._y.shape[0] != rows:       # z-slab: this rank's rows of Y and BY
                r0 = a.part.z0 * a.plane
                loc = Constraints.__new__(Constraints)
                loc._y, loc._by = c._y[r0:r0 + rows], c._by[r0:r0 + rows]
                loc._k, loc.yby_chol = c._k, c.yby_chol
                self.cons = loc
        ld = dv.even(m)
        self.ld = ld
        dev = self.dev
        self.X, self.AX, self.X2, self.AX2 = (dv.new_block(n, ld, dev) for _ in range(4))
        self.P, self.AP, self.P2, self.AP2 = (dv.new_block(n, ld, dev) for _ in range(4))
        self.BX = self.BX2 = self.BP = self.BP2 = self.BWbuf = None
        if self.b_generic is not None:
            self.BX, self.BX2, self.BP, self.BP2 = (dv.new_block(n, ld, dev) for _ in range(4))
            self.BWbuf = torch.zeros(n * ld, dtype=torch.float64, device=dev)
        self.Wbufs = [torch.zeros(n * ld, dtype=torch.float64, device=dev) for _ in range(2)]
        self.wcur = 0
        self.AWbuf = torch.zeros(n * ld, dtype=torch.float64, device=dev)
        self.sums = torch.zeros(2 * m, dtype=torch.float64, device=dev)
        nred = 2 * m + (3 * m) * (4 * m)
        # F1's reductions and the stencil pass's Gram share one buffer, so a
        # z-slab run sums both over the ranks with a single all-reduce
        self._redg2 = torch.zeros(nred + (2 * m) * m, dtype=torch.float64, device=dev)
        self.red = self._redg2[:nred]
        self.g2 = self._redg2[nred:]
        self.h_red = _host_buf(nred)
        self.h_g2 = _host_buf((2 * m) * m)
        self.h_g1 = _host_buf((3 * m) * (4 * m))
        self.h_red_np = self.h_red.numpy()
        self.h_g2_np = self.h_g2.numpy()
        self._wviews = {}
        self._triu = np.triu_indices(m)
        self._eye_triu = np.eye(m)[self._triu]
        self._tol_vec = np.full(m, cfg.tol)
        self._iota = np.arange(m)
        self._iota32 = np.arange(m, dtype=np.int32)
        self.pin = _Pinned(dev, 3 * m * m + 2 * m + 8, 3 * m + 8)
        if x0t is None:
            row0 = a.part.z0 * a.plane if rows != self.n_global else 0
            dv.seeded_fill(self.X, m, cfg.seed, row0)
        else:
            src = x0t if isinstance(x0t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x0t))
            self.X[:, :m].copy_(src, non_blocking=src.device.type == "cpu" and src.is_pinned())
            if not bool(torch.isfinite(self.X[:, :m]).all()):
                raise ValueError("x0 contains non-finite entries")

        self.active = np.ones(m, dtype=bool)
        self.lock_iteration = np.full(m, -1, dtype=np.int64)
        self.have_p = False
        self.history = []
        self.pending = 0
        self._ritz = NativeRitz(self.m)
        self.total_fallbacks = 0
        self.failure = None
        self.norms = np.zeros(m)
        self.it = 0
        self.done = False
        self.drift_repairs = 0
        # stall watch for the implicit-AX refresh (see _refresh_ax_if_stalled)
        self.ax_refreshes = 0
        self._force_repair = False
        self._stall_best = np.full(m, np.inf)
        self._stall_it = 0
        self.f1_pending = False    # self.red holds F1 results for this step
        self.sg_pending = False    # self.g2 / AW hold the stencil pass for this step

        self._initial()
        self._native_setup()

    # ------------------------------------------------------------ helpers
    def _reduce(self, t):
        """Sum a device reduction over the z-slab ranks (identity on one)."""
        if self._allreduce is not None:
            self._allreduce(t)
        return t

    def _gram(self, *args, **kw):
        return self._reduce(dv.gram(*args, **kw))

    def _residual(self, *args):
        dv.residual(*args)
        self._reduce(args[-1])

    def _wmask(self, nblocks):
        return ((1 << nblocks) - 1) if self.bdiag is not None else 0

    def _bx(self):
        """The block holding B X for the kernels: X itself for B = I and
        diagonal B (the kernels weight it by d), the carried BX otherwise."""
        return self.BX if self.b_generic is not None else self.X

    def _apply_b(self, src, dst, k):
        """dst[:, :k] = B src[:, :k] through the user's callback (generic B),
        shape-checked like every operator output."""
        y = self.b_generic(src[:, :k])
        if not isinstance(y, torch.Tensor):
            y = torch.as_tensor(np.asarray(y, dtype=np.float64), device=self.dev)
        if tuple(y.shape) != (self.n, k):
            raise ValueError(f"B returned shape {tuple(y.shape)}, expected ({self.n}, {k})")
        dst[:, :k] = y.to(device=self.dev, dtype=torch.float64)
        if dst.shape[1] > k:
            dst[:, k:] = 0.0

    def _bwview(self, k):
        return dv.view_block(self.BWbuf, self.n, dv.even(k))

    def _wview(self, k, which=None):
        key = (self.wcur if which is None else which, k)
        v = self._wviews.get(key)
        if v is None:
            buf = self.Wbufs[key[0]]
            ldw = dv.even(k)
            v = (dv.view_block(buf, self.n, ldw), dv.view_block(self.AWbuf, self.n, ldw))
            self._wviews[key] = v
        return v

    def _fetch(self, dev_t, host_t, count):
        """D2H of the first `count` doubles through pinned memory (syncs)."""
        host_t[:count].copy_(dev_t.reshape(-1)[:count], non_blocking=True)
        if self.dev.type == "cuda":
            torch.cuda.current_stream(self.dev).synchronize()
        return host_t[:count].numpy().copy()

    def _gram_xx(self):
        """X^T B X (upper triangle computed, mirrored on the host)."""
        if self.b_generic is not None:
            # X^T (BX) in full: the carried BX makes it symmetric only to
            # rounding, and the reference's drift test reads every entry
            g = _timed("gram_drift", lambda: self._gram(self.n, [(self.X, self.m)],
                                                     [(self.BX, self.m)]))
            return dv.to_host(g)
        g = _timed("gram_drift", lambda: self._gram(self.n, [(self.X, self.m)], [(self.X, self.m)],
                                                 self._wmask(1), self.bdiag, pair_mode=_UPPER))
        return _mirror_upper(dv.to_host(g))

    def _rotate_x(self, M, with_a=True):
        """X, AX (, BX) <- X M, AX M (, BX M) (no P involvement)."""
        Md = dv.to_device(M, self.dev)
        if with_a:
            dv.update(self.n, self.m, self.X, self.AX, Md, self.X2, self.AX2)
            self.AX, self.AX2 = self.AX2, self.AX
        else:
            dv.update(self.n, self.m, self.X, None, Md, self.X2, None)
        self.X, self.X2 = self.X2, self.X
        if self.b_generic is not None:
            dv.update(self.n, self.m, self.BX, None, Md, self.BX2, None)
            self.BX, self.BX2 = self.BX2, self.BX

    def _refresh_ritz(self, gxx):
        """_refresh_ritz (lobpcg.py:280-296) from the raw Gram X^T B X."""
        _, minv = scaled_cholesky(gxx)             # NotSPD propagates
        self._rotate_x(minv)
        gxa = dv.to_host(self._gram(self.n, [(self.X, self.m)], [(self.AX, self.m)],
                                 pair_mode=_UPPER))
        lam, q = sym_eig(gxa)
        self._rotate_x(q)
        self.lam = lam

    def _apply_a_plain(self, src, dst, k):
        """dst[:, :k] = A src[:, :k] (K1 for the built-in Laplacian)."""
        if self.fused_a:
            _timed("stencil", lambda: self.a.apply_into(src, dst))
        else:
            y = self.a(src[:, :k])
            if not isinstance(y, torch.Tensor) or tuple(y.shape) != (self.n, k):
                raise ValueError("operator apply returned a block of the wrong shape")
            dst[:, :k] = y

    def _initial(self):
        m, n = self.m, self.n
        if self.cons is not None:                   # lobpcg.py:394
            _project_into(self.X, m, self.cons, self.X2, self._reduce)
            self.X, self.X2 = self.X2, self.X
        if self.b_generic is not None:
            self._apply_b(self.X, self.BX, m)        # bx = b(x) (lobpcg.py:396)
        gxx = self._gram_xx()
        try:
            _, minv = scaled_cholesky(gxx)
        except NotSPD as err:
            raise ValueError(f"initial block is B-degenerate at column {err.pivot}") from err
        # X (, BX) <- X R_eff^{-1} (b_orthonormalize, lobpcg.py:398)
        self._rotate_x(minv, with_a=False)
        self._apply_a_plain(self.X, self.AX, m)      # lobpcg.py:403
        gxa = dv.to_host(self._gram(n, [(self.X, m)], [(self.AX, m)], pair_mode=_UPPER))
        lam, q = sym_eig(gxa)                        # lobpcg.py:404
        self._rotate_x(q)
        self.lam = lam

    # ---------------------------------------------------- native fast path
    def _native_setup(self):
        """b2l_fast_iteration drives the steady state when every piece of the
        step is one of the fused kernels (built-in stencil, diagonal or no B,
        Jacobi/identity T, no constraints, one GPU)."""
        cfg, m = self.cfg, self.m
        self._native = None
        slab = getattr(self.a, "native_slab", None)
        if not (self.dev.type == "cuda" and self.use_f1 and self.use_sgram and self.fused_a
                and self.b_generic is None
                and (self._allreduce is None or slab is not None)
                and self.t_generic is None and self.cons is None
                and not cfg.check_invariants and cfg.verbosity < 2):
            return
        dev = self.dev
        st = _lib.b2l_iter_state()
        # a z-slab rank steps its own planes; the library exchanges the halo
        # and sums the reductions over the ranks inside the step
        g = getattr(self.a, "local_grid", self.a.grid)
        st.slab = slab
        st.n, st.m, st.ldx = self.n, m, self.ld
        st.nx, st.ny, st.nz, st.scale = g.nx, g.ny, g.nz, self.a.scale
        st.tmode, st.tinv = self.tmode, self.tinv
        st.tvec = self.tvec.data_ptr() if self.tvec is not None else None
        st.bdiag = self.bdiag.data_ptr() if self.bdiag is not None else None
        st.tol, st.relative_tol, st.max_iter = cfg.tol, int(cfg.relative_tol), cfg.max_iter
        st.drift_limit, st.pivot_floor = DRIFT_LIMIT, PIVOT_FLOOR
        self._n_coef = torch.empty(3 * m * m, dtype=torch.float64, device=dev)
        self._n_lam = torch.empty(m, dtype=torch.float64, device=dev)
        self._n_pcols = torch.empty(2 * m, dtype=torch.int32, device=dev)
        self._n_stage = _host_buf(3 * m * m + m)
        self._n_istage = _host_buf(2 * m, torch.int32)
        st.aw = self.AWbuf.data_ptr()
        st.red_dev, st.g2_dev = self.red.data_ptr(), self.g2.data_ptr()
        st.coef_dev, st.lam_dev = self._n_coef.data_ptr(), self._n_lam.data_ptr()
        st.pcols_dev = self._n_pcols.data_ptr()
        st.h_red, st.h_g2 = self.h_red.data_ptr(), self.h_g2.data_ptr()
        st.h_stage, st.h_istage = self._n_stage.data_ptr(), self._n_istage.data_ptr()
        self._n_norms = np.zeros(m)
        self._n_newly = np.zeros(m, dtype=bool)
        self._n_lamnext = np.zeros(m)
        st.norms = self._n_norms.ctypes.data
        st.newly = self._n_newly.ctypes.data
        st.lam_next = self._n_lamnext.ctypes.data
        self._native = st

    def _native_step(self):
        """One steady-state iteration in b2l_fast_iteration.  Returns the
        step() result, or None when the drift test needs the repair path."""
        st, cfg, m = self._native, self.cfg, self.m
        lam = np.ascontiguousarray(self.lam, dtype=np.float64)
        active = np.ascontiguousarray(self.active, dtype=bool)
        self.lam, self.active = lam, active
        kst = int(active.sum())
        st.x, st.ax, st.p, st.ap = (t.data_ptr() for t in (self.X, self.AX, self.P, self.AP))
        st.x2, st.ax2, st.p2, st.ap2 = (t.data_ptr() for t in (self.X2, self.AX2, self.P2,
                                                                  self.AP2))
        st.w_cur = self.Wbufs[self.wcur].data_ptr()
        st.w_next = self.Wbufs[1 - self.wcur].data_ptr()
        st.lam = lam.ctypes.data
        st.active = active.ctypes.data
        st.lock_iteration = self.lock_iteration.ctypes.data
        st.it, st.have_p, st.kst = self.it, int(self.have_p), kst
        st.drift_limit = -1.0 if self._force_repair else DRIFT_LIMIT
        self._force_repair = False
        st.stream = torch.cuda.current_stream(self.dev).cuda_stream
        lib = _lib.load()
        rc = lib.b2l_fast_iteration(ctypes.byref(st))
        if rc == _lib.ITER_DRIFT:
            return None
        if rc < 0 and rc != _lib.EDEGENERATE:
            _lib.check(rc, "b2l_fast_iteration")
        it = self.it
        norms = self._n_norms.copy()
        newly = self._n_newly
        self.norms = norms
        self.f1_pending = self.sg_pending = False
        if st.repaired:
            # the drift test fired and the step repaired the block on the
            # device (lam now holds the repaired Ritz values): the repaired
            # blocks sit in the "next" buffers
            self.drift_repairs += 1
            self._swap_blocks()
            if cfg.verbosity >= 2:
                print(f"  it {it:4d}  Ritz block re-orthonormalized (drift {st.drift:.1e})")
        self.history.append(HistoryEntry(
            iteration=it,
            ritz=lam.copy() if cfg.lock_history else None,
            residual_norms=norms.copy() if cfg.lock_history else None,
            active=active.copy(),
            locked_now=tuple(int(i) for i in np.flatnonzero(newly)) if newly.any() else (),
            fallbacks=self.pending,
            constraint_violation=None,
        ))
        self.total_fallbacks += self.pending
        self.pending = 0
        if rc == _lib.ITER_DONE:
            self.done = True
            return False
        if rc == _lib.EDEGENERATE:
            self.pending += st.fallbacks
            self.failure = "BasisDegeneracy"
            self.done = True
            return False
        # ITER_OK: the next F1 and stencil pass are queued
        self.pending += st.fallbacks
        self._swap_blocks()
        self.have_p = True
        self.lam = self._n_lamnext.copy()
        self.f1_pending = self.sg_pending = True
        self.it += 1
        return True

    def _swap_blocks(self):
        self.X, self.X2 = self.X2, self.X
        self.AX, self.AX2 = self.AX2, self.AX
        self.P, self.P2 = self.P2, self.P
        self.AP, self.AP2 = self.AP2, self.AP
        self.wcur = 1 - self.wcur

    # ---------------------------------------------------------- iteration
    STALL_WINDOW = 100   # iterations without any active residual halving

    def _refresh_ax_if_stalled(self):
        """AX and AP are carried by recurrence (the reference never recomputes
        them, lobpcg.py:520-540).  The fused path folds the orthonormalisation
        of W and P into the update coefficients, so `A P_orth` is formed as
        `(A P_raw) M_p`: when two active columns of one cluster make P nearly
        dependent, that product and `P_raw M_p` lose `eps cond(P)` to
        cancellation independently and the recurrence drifts by
        `eps cond(P) |A|` per step.  Once the drift exceeds the tolerance the
        computed residuals cannot fall below it (Ritz values freeze, slightly
        BELOW the exact eigenvalues) and the run stalls.  Watch for exactly
        that -- no active column has halved its best residual for
        STALL_WINDOW iterations -- and then recompute AX = A X and AP = A P
        (two applies): more accurate than the recurrence, never less."""
        if self.it == 0 or self.norms is None:
            return
        act = self.active
        if not act.any():
            return
        better = act & (self.norms < 0.5 * self._stall_best)
        if better.any() or not np.isfinite(self._stall_best[act]).all():
            self._stall_best = np.where(act, np.minimum(self._stall_best, self.norms),
                                        self._stall_best)
            self._stall_it = self.it
            return
        if self.it - self._stall_it < self.STALL_WINDOW or not self.have_p:
            return
        if self.b_generic is not None or self._allreduce is not None:
            return   # B-side recurrences / slab runs: not covered here
        self._apply_a_plain(self.X, self.AX, self.m)
        self._apply_a_plain(self.P, self.AP, self.m)
        # ... and have this step run the reference's own repair
        # (_refresh_ritz, lobpcg.py:280-296) on them: the pencil's X block is
        # the carried diag(Lambda) (lobpcg.py:323), which is only as good as
        # the recurrences; the repair re-diagonalises the fresh X^T A X
        self._force_repair = True
        self.ax_refreshes += 1
        self._stall_it = self.it
        self._stall_best = np.where(act, self.norms, self._stall_best)
        if self.cfg.verbosity >= 2:
            print(f"  it {self.it:4d}  A X and A P recomputed (stalled residuals)")

    def step(self):
        """One pass of the hot loop body (lobpcg.py:418-540).  Returns False
        once the loop has exited (converged, max_iter or failure)."""
        if self.done:
            return False
        self._refresh_ax_if_stalled()
        fetched = False
        if self._native is not None and self.f1_pending and self.sg_pending \
                and _OPTS["timer"] is None:
            res = self._native_step()
            if res is not None:
                return res
            fetched = True            # drift: the reductions are in h_red / h_g2
        elif self._native is not None and self._native.red_on_host and self.f1_pending:
            # the passes the native step queued write their reductions
            # straight into the pinned h_red / h_g2 (device-mapped), not into
            # self.red / self.g2: read them there (a timer entered mid-run
            # sends the step down this path)
            torch.cuda.current_stream(self.dev).synchronize()
            self._native.red_on_host = 0
            fetched = True
        cfg, m, n = self.cfg, self.m, self.n
        it = self.it
        try:
            jprev = np.flatnonzero(self.active)
            kst = jprev.size
            G1 = sums = G2 = None
            g2_rows = m + kst
            if self.f1_pending:
                # F1 of the previous step already produced this step's drift
                # Gram, residual norms, W and every non-AW Gram block; the
                # stencil pass queued right behind it produced A W and
                # [X W]^T A W.  One host synchronisation for both.
                a, b = 2 * m + kst, 3 * m + kst
                nred = 2 * m + a * b
                if not fetched:
                    if self.sg_pending and self._allreduce is not None:
                        # one all-reduce over [red | g2] (the unused tail of
                        # red between nred and its capacity rides along)
                        self._reduce(self._redg2[:self.red.numel() + g2_rows * kst])
                    else:
                        self._reduce(self.red[:nred])
                        if self.sg_pending:
                            self._reduce(self.g2[:g2_rows * kst])
                    self.h_red[:nred].copy_(self.red[:nred], non_blocking=True)
                    if self.sg_pending:
                        self.h_g2[:g2_rows * kst].copy_(self.g2[:g2_rows * kst],
                                                        non_blocking=True)
                    if self.dev.type == "cuda":
                        torch.cuda.current_stream(self.dev).synchronize()
                # views of the pinned staging buffers (rewritten only after
                # the next synchronisation)
                red = self.h_red_np[:nred]
                sums = red[:2 * m]
                G1 = red[2 * m:].reshape(a, b)
                gxx = None
                if self.sg_pending:
                    G2 = self.h_g2_np[:g2_rows * kst].reshape(g2_rows, kst)
            else:
                gxx = self._gram_xx()
            self.f1_pending = False
            self.sg_pending = False
            # drift check (lobpcg.py:419-428): max |X^T B X - I| over the
            # upper triangle (the Gram is symmetric)
            gu = G1[:m, :m] if gxx is None else gxx
            drift = float(np.abs(gu[self._triu] - self._eye_triu).max())
            forced, self._force_repair = self._force_repair, False
            if gxx is None and (drift > DRIFT_LIMIT or forced or cfg.check_invariants):
                gxx = _mirror_upper(gu)
            if drift > DRIFT_LIMIT or forced:
                try:
                    self._refresh_ritz(gxx)
                except NotSPD:
                    raise _Failure("BasisDegeneracy")
                self.drift_repairs += 1
                G1 = sums = G2 = None
                if cfg.verbosity >= 2:
                    print(f"  it {it:4d}  Ritz block re-orthonormalized (drift {drift:.1e})")

            W, AW = self._wview(kst)
            if sums is None:
                # residual + T(W) for the active set (lobpcg.py:429-430, :466-467)
                pos = np.full(m, -1, dtype=np.int32)
                pos[jprev] = np.arange(kst, dtype=np.int32)
                (lam_d,), (pos_d,) = self.pin.upload([self.lam], [pos])
                _timed("residual", lambda: self._residual(
                    n, m, self._bx(), self.AX, self.bdiag, lam_d, self.tmode, self.tinv, self.tvec,
                    pos_d, kst, W, cfg.relative_tol, self.sums))
                sums = self._fetch(self.sums, self.h_red, 2 * m)

            # lock test (lobpcg.py:429-437)
            norms = np.sqrt(sums[:m])
            if cfg.relative_tol:
                thresholds = cfg.tol * np.sqrt(sums[m:2 * m])
            else:
                thresholds = self._tol_vec
            newly = self.active & (norms < thresholds)
            # clusters in the pencil eigensolve: eigenvalue gaps below a tenth
            # of the smallest lock threshold (rr.cu align_clusters;
            # b2l_fast_iteration sets the same value)
            self._ritz.align = 0.1 * float(np.min(thresholds))
            self.lock_iteration[newly] = it
            self.active = self.active & ~newly
            self.norms = norms
            violation = None
            if self.cons is not None:                # lobpcg.py:438-439
                violation = self._violation()
            self.history.append(HistoryEntry(
                iteration=it,
                ritz=self.lam.copy() if cfg.lock_history else None,
                residual_norms=norms.copy() if cfg.lock_history else None,
                active=self.active.copy(),
                locked_now=tuple(int(i) for i in np.flatnonzero(newly)) if newly.any() else (),
                fallbacks=self.pending,
                constraint_violation=violation,
            ))
            self.total_fallbacks += self.pending
            self.pending = 0
            if cfg.verbosity >= 2:
                print(f"  it {it:4d}  active {int(self.active.sum()):3d}  "
                      f"max resid {norms.max():.3e}")
            if not self.active.any() or it == cfg.max_iter:
                self.done = True
                return False
            if cfg.check_invariants:
                self._check_state(gxx)

            J = np.flatnonzero(self.active)
            # W columns of J
            sel = self._iota[:kst] if J.size == kst else np.searchsorted(jprev, J)
            if self.t_generic is not None:
                W, AW, kst, sel = self._generic_precondition(W, sel, J.size)
                G1 = G2 = None                       # F1 saw the raw residual
                g2_rows = m + kst
            elif self.b_generic is not None and J.size != kst:
                # b(w) sees the active columns only, as in the reference
                W, AW, kst, sel = self._compact_w(W, sel, J.size)
                g2_rows = m + kst
            if self.cons is not None:
                # w = apply_constraints(w, y) (lobpcg.py:475), into the other W buffer
                nxt = 1 - self.wcur
                Wn, AW = self._wview(kst, nxt)
                _project_into(W, kst, self.cons, Wn, self._reduce)
                self.wcur = nxt
                W = Wn
            BW = None
            if self.b_generic is not None:
                BW = self._bwview(kst)               # bw = b(w) (lobpcg.py:476)
                self._apply_b(W, BW, kst)

            # A W (+ [X W]^T A W in the same pass for the built-in stencil)
            g2 = self.g2[:g2_rows * kst].view(g2_rows, kst)
            G1dev = None
            if G1 is None:
                # G1 = [X W P]^T B [X W P (AP)] first: it does not need A W,
                # so its half of Rayleigh-Ritz (the Cholesky-QRs and the
                # pencil's B factor) runs on the host while A W and G2 are
                # still on the GPU
                if self.have_p:
                    L = [(self.X, m), (W, kst), (self.P, m)]
                    if BW is not None:
                        R = [(self.BX, m), (BW, kst), (self.BP, m), (self.AP, m)]
                    else:
                        R = L + [(self.AP, m)]
                    G1dev = _timed("gram", lambda: self._gram(n, L, R, self._wmask(3), self.bdiag,
                                                           pair_mode=_MODES_P))
                else:
                    L = [(self.X, m), (W, kst)]
                    R = [(self.BX, m), (BW, kst)] if BW is not None else L
                    G1dev = _timed("gram", lambda: self._gram(n, L, R, self._wmask(2), self.bdiag,
                                                           pair_mode=_MODES_NOP))
            g1_ready = None
            if G1dev is not None and G2 is None and self.dev.type == "cuda":
                cnt = G1dev.numel()
                self.h_g1[:cnt].copy_(G1dev.reshape(-1), non_blocking=True)
                g1_ready = torch.cuda.Event()
                g1_ready.record(torch.cuda.current_stream(self.dev))
            if G2 is None:
                self._launch_aw(W, AW, kst, g2)
            begun = False
            if g1_ready is not None:
                g1_ready.synchronize()
                G1 = self.h_g1[:cnt].numpy().reshape(G1dev.shape)
                self._ritz.begin(m, kst, self.have_p, G1, J, sel, PIVOT_FLOOR)
                begun = True
            elif G1dev is not None:
                G1 = dv.to_host(G1dev)
            if G2 is None:
                if self.use_sgram:
                    self._reduce(g2)   # the callback path reduced inside self._gram
                G2 = self._fetch(g2, self.h_g2, g2_rows * kst).reshape(g2_rows, kst)
            self._rayleigh_ritz(G1, G2, J, sel, kst, W, AW, begun=begun, BW=BW)
        except _Failure as f:
            self.failure = str(f)
            self.done = True
            return False
        self.it += 1
        return True

    def _launch_aw(self, W, AW, kst, g2):
        """A W on the stored columns of W and G2 = [X W]^T A W (K1+K5b for
        the built-in stencil; callback + K5 otherwise)."""
        m, n = self.m, self.n
        if self.use_sgram:
            _timed("stencil", lambda: self.a.stencil_gram_into(W, AW, self.X, m, kst, g2))
        else:
            self._apply_a_plain(W, AW, kst)
            _timed("gram_aw", lambda: self._gram(n, [(self.X, m), (W, kst)], [(AW, kst)],
                                              out=g2))

    def _compact_w(self, W, sel, kj):
        """The active columns sel of W, compacted into the other W buffer."""
        nxt = 1 - self.wcur
        Wn, AWn = self._wview(kj, nxt)
        Wn.zero_()
        Wn[:, :kj] = W[:, torch.as_tensor(sel, device=self.dev)]
        self.wcur = nxt
        return Wn, AWn, kj, np.arange(kj)

    def _generic_precondition(self, W, sel, kj):
        """User preconditioner callback on the active residual block
        (lobpcg.py:466-474): shape and finiteness are checked as in the
        reference, and the result becomes the compact W."""
        n = self.n
        wj = W[:, torch.as_tensor(sel, device=self.dev)]
        out = self.t_generic(wj)
        if not isinstance(out, torch.Tensor):
            out = torch.as_tensor(np.asarray(out, dtype=np.float64), device=self.dev)
        if tuple(out.shape) != (n, kj):
            raise ValueError(f"preconditioner returned shape {tuple(out.shape)}, expected ({n}, {kj})")
        if not bool(torch.isfinite(out).all()):
            raise ValueError("preconditioner returned non-finite entries")
        W, AW = self._wview(kj)
        W.zero_()
        W[:, :kj] = out.to(torch.float64)
        return W, AW, kj, np.arange(kj)

    def _rayleigh_ritz(self, G1, G2, J, sel, kst, W, AW, begun=False, BW=None):
        """Rayleigh-Ritz on the projected blocks (lobpcg.py:475-519) in the
        native host routine b2l_rayleigh_ritz (or its second half when
        `begun`), then the device update."""
        m, n = self.m, self.n
        try:
            if begun:
                lam_new, coef, pcols, fb = self._ritz.finish(m, G2, self.lam)
            else:
                lam_new, coef, pcols, fb = self._ritz(m, kst, self.have_p, G1, G2, self.lam, J,
                                                      sel, PIVOT_FLOOR)
        except RitzFailure as f:
            self.pending += f.fallbacks
            raise _Failure("BasisDegeneracy")
        self.pending += fb
        kp = pcols.size
        cx = coef[:m * m].reshape(m, m)
        cw_raw = coef[m * m:m * m + kst * m].reshape(kst, m)
        cp_raw = coef[m * m + kst * m:].reshape(kp, m)

        if self.use_f1:
            # next iteration's W holds the current active set J
            if J.size == m:
                wpos = self._iota32
            else:
                wpos = np.full(m, -1, dtype=np.int32)
                wpos[J] = np.arange(J.size, dtype=np.int32)
            (coef_d, lam_d), (pc_d, wpos_d) = self.pin.upload(
                [coef, lam_new],
                [pcols if kp else np.zeros(1, np.int32), wpos])
            nxt = 1 - self.wcur
            Wn, _ = self._wview(J.size, nxt)
            tmode = 0 if self.t_generic is not None else self.tmode
            _timed("step", lambda: dv.lobpcg_step(
                n, m, self.X, self.AX, W, AW, kst, self.P if kp else None,
                self.AP if kp else None, kp, pc_d, coef_d, self.X2, self.AX2, self.P2,
                self.AP2, lam_d, self.bdiag, tmode, self.tinv, self.tvec, wpos_d, J.size, Wn,
                self.cfg.relative_tol, self.red))
            self.wcur = nxt
            self.f1_pending = True
        else:
            (cx_d, cw_d, cp_d), (pc_d,) = self.pin.upload(
                [cx, cw_raw, cp_raw if kp else np.zeros(1)],
                [pcols if kp else np.zeros(1, np.int32)])
            _timed("update", lambda: dv.update(
                n, m, self.X, self.AX, cx_d, self.X2, self.AX2, w=W, aw=AW, kw=kst, cw=cw_d,
                p=self.P if kp else None, ap=self.AP if kp else None, pcols=pc_d, kp=kp,
                cp=cp_d, po=self.P2, apo=self.AP2, x_plus_p=True))
            if BW is not None:
                # BP' = BW Cw + BP_J Cp, BX' = BX Cx + BP' (lobpcg.py:533-538)
                _timed("update", lambda: dv.update(
                    n, m, self.BX, None, cx_d, self.BX2, None, w=BW, kw=kst, cw=cw_d,
                    p=self.BP if kp else None, pcols=pc_d, kp=kp, cp=cp_d, po=self.BP2,
                    x_plus_p=True))
                self.BX, self.BX2 = self.BX2, self.BX
                self.BP, self.BP2 = self.BP2, self.BP
        self.X, self.X2 = self.X2, self.X
        self.AX, self.AX2 = self.AX2, self.AX
        self.P, self.P2 = self.P2, self.P
        self.AP, self.AP2 = self.AP2, self.AP
        self.have_p = True
        if self.use_f1 and self.use_sgram and self.t_generic is None:
            # queue the next step's stencil pass right behind F1: it needs
            # only W' and X', and its columns are a superset of the next
            # active set, so the lock test can run after it
            k_next = J.size
            Wn, AWn = self._wview(k_next)
            g2n = self.g2[:(m + k_next) * k_next].view(m + k_next, k_next)
            self._launch_aw(Wn, AWn, k_next, g2n)
            self.sg_pending = True
        self.lam = lam_new

    def _violation(self):
        """max |(BY)^T X| (lobpcg.py:438-439)."""
        c = self.cons
        g = dv.to_host(self._gram(self.n, [(c._by, c.count)], [(self.X, self.m)]))
        return float(np.abs(g).max())

    def _check_state(self, gxx):
        """_check_state (lobpcg.py:266-277)."""
        err = np.abs(gxx - np.eye(self.m)).max()
        if err > 1e-10:
            raise RuntimeError(f"block lost B-orthonormality: max deviation {err:.3e}")
        if self.cons is not None:
            gx = dv.to_host(self._gram(self.n, [(self.X, self.m)], [(self.X, self.m)]))
            scale = max(1.0, float(np.sqrt(np.diag(gx)).max()))
            viol = self._violation()
            if viol > 1e-10 * scale:
                raise RuntimeError(
                    f"block lost constraint orthogonality: max violation {viol:.3e}")

    # -------------------------------------------------------------- finish
    def report(self):
        """Exit refresh + status (lobpcg.py:542-577)."""
        cfg, m, n = self.cfg, self.m, self.n
        self.total_fallbacks += self.pending
        self.pending = 0
        failure = self.failure
        norms = self.norms
        if failure is None:
            try:
                self._refresh_ritz(self._gram_xx())
                lam_d = dv.to_device(self.lam, self.dev)
                self._residual(n, m, self._bx(), self.AX, self.bdiag, lam_d, 0, 1.0, None, None, 0,
                            None, False, self.sums)
                norms = np.sqrt(dv.to_host(self.sums)[:m])
            except NotSPD:
                failure = "BasisDegeneracy"
        converged = ~self.active
        if failure is not None:
            status = f"Failed({failure})"
        elif self.total_fallbacks:
            status = f"BasisFallback({self.total_fallbacks})"
        elif converged.all():
            status = "Converged"
        else:
            status = "MaxIterReached"
        if cfg.verbosity >= 1:
            print(f"[blockeig] {status}: {int(converged.sum())}/{m} converged in "
                  f"{self.history[-1].iteration} iterations, max residual {norms.max():.3e}")
        vecs = self.X[:, :m]
        if _OPTS["return_device"]:
            vecs = vecs.clone()
        else:
            # D2H into page-locked memory (torch's caching host allocator
            # recycles it across solves): ~50 GB/s instead of the ~2 GB/s of a
            # pageable copy into fresh numpy pages; the array owns the buffer
            host = torch.empty((n, m), dtype=torch.float64, pin_memory=self.dev.type == "cuda")
            host.copy_(vecs)
            vecs = host.numpy()
        return SolverReport(
            eigenvalues=self.lam.copy(),
            eigenvectors=vecs,
            iterations_used=self.history[-1].iteration,
            converged=converged,
            residual_norms=norms,
            lock_iterations=self.lock_iteration.copy(),
            history=tuple(self.history),
            status=status,
            basis_fallbacks=self.total_fallbacks,
        )


def solve(a, b=None, t=None, y=None, x0=None, config=None):
    """Compute the m smallest eigenpairs of A x = lambda B x on the GPU.

    Same signature, semantics and report as the reference ``solve``
    (lobpcg.py:343).  ``a``, ``b``, ``t`` are operators of this package (or
    any callables on CUDA (n, k) float64 tensors).
    """
    run = LOBPCGRun(a, b=b, t=t, y=y, x0=x0, config=config)
    while run.step():
        pass
    return run.report()


def solve_staged(a, b=None, t=None, total_wanted=1, stage_block=1, config=None):
    """Compute total_wanted eigenpairs in stages of stage_block at a time
    (lobpcg.py:580-653): each stage is a ``solve`` with every previously
    accepted eigenvector hard-locked into the constraints; stage seeds are
    config.seed + stage; stops at the first stage that fails or stalls.  The
    report concatenates the stages (eigenpairs sorted ascending, history
    entries stamped with their stage, iterations summed, per-stage reports
    in ``stages``).  The accumulated basis stays on the GPU between stages."""
    cfg = config if config is not None else SolverConfig()
    cfg.validate()
    if stage_block < 1:
        raise ValueError(f"stage_block must be >= 1, got {stage_block}")
    if total_wanted < stage_block:
        raise ValueError(
            f"total_wanted ({total_wanted}) must be >= stage_block ({stage_block})")
    want_device = _OPTS["return_device"]
    reports = []
    constraints = None
    basis = None
    remaining = total_wanted
    stage = 0
    while remaining > 0:
        mcur = min(stage_block, remaining)
        stage_cfg = dataclasses.replace(cfg, block_size=mcur, seed=cfg.seed + stage)
        with device_options(return_device=True):
            report = solve(a, b=b, t=t, y=constraints, config=stage_cfg)
        reports.append(report)
        if not (report.ok and report.all_converged):
            break
        vecs = report.eigenvectors
        basis = vecs if basis is None else torch.cat([basis, vecs], dim=1)
        constraints = Constraints.from_basis(basis, b)
        remaining -= mcur
        stage += 1

    def host(v):
        return v if want_device else dv.to_host(v).copy()

    reports = [dataclasses.replace(r, eigenvectors=host(r.eigenvectors)) for r in reports]
    values = np.concatenate([r.eigenvalues for r in reports])
    order = np.argsort(values, kind="stable")
    if want_device:
        vectors = torch.cat([r.eigenvectors for r in reports], dim=1)[:, torch.as_tensor(order)]
    else:
        vectors = np.hstack([r.eigenvectors for r in reports])[:, order]
    converged = np.concatenate([r.converged for r in reports])[order]
    residuals = np.concatenate([r.residual_norms for r in reports])[order]
    locks = np.concatenate([r.lock_iterations for r in reports])[order]
    history = tuple(dataclasses.replace(entry, stage=s)
                    for s, r in enumerate(reports) for entry in r.history)
    fallbacks = sum(r.basis_fallbacks for r in reports)
    failed = [r.status for r in reports if not r.ok]
    if failed:
        status = failed[0]
    elif not converged.all():
        status = "MaxIterReached"
    elif fallbacks:
        status = f"BasisFallback({fallbacks})"
    else:
        status = "Converged"
    return SolverReport(
        eigenvalues=values[order],
        eigenvectors=vectors,
        iterations_used=sum(r.iterations_used for r in reports),
        converged=converged,
        residual_norms=residuals,
        lock_iterations=locks,
        history=history,
        status=status,
        basis_fallbacks=fallbacks,
        stages=tuple(reports),
    )
