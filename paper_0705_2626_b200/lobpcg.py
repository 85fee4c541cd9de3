"""LOBPCG with soft locking on B200: the reference's ``solve`` entry point
(lobpcg.py:343-577) with every long-dimension operation on the GPU.

Control flow, thresholds, the lock test, the basis-repair ladder, the drift
repair and the status strings are the reference's, evaluated on the host on
small matrices.  What changes is where the tall work happens and how much of
it there is per iteration:

  reference (numpy)                      here (libb200lobpcg, sm_100a)
  ------------------------------------   ----------------------------------
  drift gram X^T B X        :419          K5 gram (1 pass over X)
  W_full, norms, T(W_J)     :429-467      K4+K2 residual kernel (1 pass)
  b_orthonormalize(W), P    :176-178,490  host Cholesky of Gram sub-blocks;
   (gram + tri_solve_right)                R^{-1} folded into the pencil and
                                           the update coefficients -- W, P,
                                           AP are never rewritten
  a(w)                      :482          K1 fused stencil on raw W
  _project_pencil 8 grams   :299-340      K5 one multi-block gram pass
  gen_sym_eig + ladder      :501-519      host (scipy LAPACK), unchanged
  Ritz update 6 multiplies  :520-540      K6 one fused update pass

BX is d*X computed on the fly for diagonal B (the reference carries BX by
recurrence); this changes results only at rounding level.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from . import device as dv
from .operators import (
    DiagonalOperator,
    IdentityOperator,
    IdentityPreconditioner,
    JacobiPreconditioner,
    Laplacian3D,
)
from .small import NotSPD, gen_sym_eig, scaled_cholesky, sym_eig

__all__ = [
    "SolverConfig",
    "HistoryEntry",
    "SolverReport",
    "solve",
    "solve_staged",
    "device_options",
    "LOBPCGRun",
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
_OPTS = {"return_device": False, "timer": None}


@contextlib.contextmanager
def device_options(return_device: bool | None = None, timer=None):
    """Scoped device options: ``return_device`` keeps eigenvectors on the GPU
    (the 464^3 x 8 block is 6.4 GB); ``timer`` is a callable(name, fn) hook
    used by bench.py to time individual kernels with CUDA events."""
    old = dict(_OPTS)
    if return_device is not None:
        _OPTS["return_device"] = bool(return_device)
    if timer is not None:
        _OPTS["timer"] = timer
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
# L = [X, W, P], R = [X, W, P, AW, AP]  (P^T AW is never used)
_MODES_P = np.array([[2, 1, 1, 1, 1],
                     [0, 2, 1, 1, 1],
                     [0, 0, 2, 0, 1]], dtype=np.uint8)
# L = [X, W], R = [X, W, AW]
_MODES_NOP = np.array([[2, 1, 1],
                       [0, 2, 1]], dtype=np.uint8)


def _mirror_upper(g):
    return np.triu(g) + np.triu(g, 1).T


class LOBPCGRun:
    """One LOBPCG solve on the device, stepped iteration by iteration.

    ``solve`` drives it to completion; bench.py steps it to time individual
    iterations.  Mirrors lobpcg.py:375-577 line for line in control flow.
    """

    def __init__(self, a, b=None, t=None, y=None, x0=None, config=None):
        cfg = config if config is not None else SolverConfig()
        cfg.validate()
        if y is not None and getattr(y, "count", 0) > 0:
            raise NotImplementedError(
                "hard-locking constraints (y) are not on the B200 path yet")
        self.cfg = cfg
        m = cfg.block_size
        n = a.dim
        if m > n:
            raise ValueError(f"block size {m} exceeds the constrained problem dimension {n} - 0")
        self.a, self.b, self.t = a, b, t
        self.m, self.n = m, n
        self.dev = getattr(a, "device", None) or torch.device("cuda", torch.cuda.current_device())
        _lib.load()
        _lib.ensure_device(self.dev.index if self.dev.index is not None else 0)

        # ---- operator kinds
        self.fused_a = isinstance(a, Laplacian3D)
        self.bdiag = None
        if b is not None and not isinstance(b, IdentityOperator):
            if not isinstance(b, DiagonalOperator):
                raise NotImplementedError("only diagonal B (DiagonalOperator) is supported on the B200 path")
            if b.dim != n:
                raise ValueError(f"B has dimension {b.dim}, expected {n}")
            self.bdiag = b.d.to(self.dev)
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

        # ---- initial block (lobpcg.py:386-393)
        if x0 is not None:
            if isinstance(x0, torch.Tensor):
                x0t = x0.detach().to(self.dev, torch.float64)
                if tuple(x0t.shape) != (n, m):
                    raise ValueError(f"x0 has shape {tuple(x0t.shape)}, expected ({n}, {m})")
                if not bool(torch.isfinite(x0t).all()):
                    raise ValueError("x0 contains non-finite entries")
            else:
                xh = np.array(x0, dtype=np.float64, copy=True)
                if xh.shape != (n, m):
                    raise ValueError(f"x0 has shape {xh.shape}, expected ({n}, {m})")
                if not np.all(np.isfinite(xh)):
                    raise ValueError("x0 contains non-finite entries")
                x0t = xh
        else:
            x0t = np.random.Generator(np.random.PCG64(cfg.seed)).uniform(-1.0, 1.0, size=(n, m))

        ld = dv.even(m)
        self.ld = ld
        dev = self.dev
        self.X = dv.new_block(n, ld, dev)
        self.AX = dv.new_block(n, ld, dev)
        self.X2 = dv.new_block(n, ld, dev)
        self.AX2 = dv.new_block(n, ld, dev)
        self.P = dv.new_block(n, ld, dev)
        self.AP = dv.new_block(n, ld, dev)
        self.P2 = dv.new_block(n, ld, dev)
        self.AP2 = dv.new_block(n, ld, dev)
        self.Wbuf = torch.zeros(n * ld, dtype=torch.float64, device=dev)
        self.AWbuf = torch.zeros(n * ld, dtype=torch.float64, device=dev)
        self.sums = torch.zeros(2 * m, dtype=torch.float64, device=dev)
        if isinstance(x0t, torch.Tensor):
            self.X[:, :m] = x0t
        else:
            self.X[:, :m].copy_(torch.from_numpy(x0t))

        self.active = np.ones(m, dtype=bool)
        self.lock_iteration = np.full(m, -1, dtype=np.int64)
        self.have_p = False
        self.history = []
        self.pending = 0
        self.total_fallbacks = 0
        self.failure = None
        self.norms = np.zeros(m)
        self.it = 0
        self.done = False
        self.drift_repairs = 0

        self._initial()

    # ------------------------------------------------------------ helpers
    def _wmask(self, nblocks):
        return ((1 << nblocks) - 1) if self.bdiag is not None else 0

    def _gram_xx(self):
        """X^T B X (upper triangle computed, mirrored on the host)."""
        g = _timed("gram_drift", lambda: dv.gram(self.n, [(self.X, self.m)], [(self.X, self.m)],
                                                 self._wmask(1), self.bdiag, pair_mode=_UPPER))
        return _mirror_upper(dv.to_host(g))

    def _apply_a(self, src, dst, k):
        """dst[:, :k] = A src[:, :k] for (n, ld) blocks (K1 when fused)."""
        if self.fused_a:
            _timed("stencil", lambda: self.a.apply_into(src, dst))
        else:
            y = self.a(src[:, :k])
            if not isinstance(y, torch.Tensor) or tuple(y.shape) != (self.n, k):
                raise ValueError("operator apply returned a block of the wrong shape")
            dst[:, :k] = y

    def _rotate_x(self, M):
        """X, AX <- X M, AX M (no P involvement)."""
        Md = dv.to_device(M, self.dev)
        dv.update(self.n, self.m, self.X, self.AX, Md, self.X2, self.AX2)
        self.X, self.X2 = self.X2, self.X
        self.AX, self.AX2 = self.AX2, self.AX

    def _refresh_ritz(self, gxx):
        """_refresh_ritz (lobpcg.py:280-296) from the raw Gram X^T B X."""
        _, minv = scaled_cholesky(gxx)             # NotSPD propagates
        self._rotate_x(minv)
        gxa = dv.to_host(dv.gram(self.n, [(self.X, self.m)], [(self.AX, self.m)],
                                 pair_mode=_UPPER))
        lam, q = sym_eig(gxa)
        self._rotate_x(q)
        self.lam = lam

    def _initial(self):
        m, n = self.m, self.n
        gxx = self._gram_xx()
        try:
            _, minv = scaled_cholesky(gxx)
        except NotSPD as err:
            raise ValueError(f"initial block is B-degenerate at column {err.pivot}") from err
        # X <- X R_eff^{-1} (b_orthonormalize, lobpcg.py:398)
        Md = dv.to_device(minv, self.dev)
        dv.update(n, m, self.X, None, Md, self.X2, None)
        self.X, self.X2 = self.X2, self.X
        self._apply_a(self.X, self.AX, m)             # lobpcg.py:403
        gxa = dv.to_host(dv.gram(n, [(self.X, m)], [(self.AX, m)], pair_mode=_UPPER))
        lam, q = sym_eig(gxa)                          # lobpcg.py:404
        self._rotate_x(q)
        self.lam = lam

    # ---------------------------------------------------------- iteration
    def step(self):
        """One pass of the hot loop body (lobpcg.py:418-540).  Returns False
        once the loop has exited (converged, max_iter or failure)."""
        if self.done:
            return False
        cfg, m, n = self.cfg, self.m, self.n
        it = self.it
        try:
            # drift check (lobpcg.py:419-428)
            gxx = self._gram_xx()
            drift = np.abs(gxx - np.eye(m)).max()
            if drift > DRIFT_LIMIT:
                try:
                    self._refresh_ritz(gxx)
                except NotSPD:
                    raise _Failure("BasisDegeneracy")
                self.drift_repairs += 1
                if cfg.verbosity >= 2:
                    print(f"  it {it:4d}  Ritz block re-orthonormalized (drift {drift:.1e})")

            # residual + lock (lobpcg.py:429-437); W written for the active set
            jprev = np.flatnonzero(self.active)
            kst = jprev.size
            ldw = dv.even(kst)
            W = dv.view_block(self.Wbuf, n, ldw)
            AW = dv.view_block(self.AWbuf, n, ldw)
            pos = np.full(m, -1, dtype=np.int32)
            pos[jprev] = np.arange(kst, dtype=np.int32)
            lam_d = dv.to_device(self.lam, self.dev)
            pos_d = dv.to_device(pos, self.dev, torch.int32)
            _timed("residual", lambda: dv.residual(
                n, m, self.X, self.AX, self.bdiag, lam_d, self.tmode, self.tinv, self.tvec,
                pos_d, kst, W, cfg.relative_tol, self.sums))
            sums = dv.to_host(self.sums)
            norms = np.sqrt(sums[:m])
            if cfg.relative_tol:
                thresholds = cfg.tol * np.sqrt(sums[m:])
            else:
                thresholds = np.full(m, cfg.tol)
            newly = self.active & (norms < thresholds)
            self.lock_iteration[newly] = it
            self.active = self.active & ~newly
            self.norms = norms
            self.history.append(HistoryEntry(
                iteration=it,
                ritz=self.lam.copy() if cfg.lock_history else None,
                residual_norms=norms.copy() if cfg.lock_history else None,
                active=self.active.copy(),
                locked_now=tuple(int(i) for i in np.flatnonzero(newly)),
                fallbacks=self.pending,
                constraint_violation=None,
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
                self._check_state()

            J = np.flatnonzero(self.active)
            sel = np.searchsorted(jprev, J)          # W columns of J
            if self.t_generic is not None:
                W, AW, kst, ldw, sel = self._generic_precondition(W, sel, J.size)

            # AW = A W on the raw (un-orthonormalized) residuals
            self._apply_a(W, AW, kst)

            # one Gram pass for every block product of the step
            hp = self.have_p
            L = [(self.X, m), (W, kst)] + ([(self.P, m)] if hp else [])
            R = [(self.X, m), (W, kst)] + ([(self.P, m)] if hp else []) + [(AW, kst)] + \
                ([(self.AP, m)] if hp else [])
            nb = 3 if hp else 2
            mode = _MODES_P if hp else _MODES_NOP
            G = dv.to_host(_timed("gram", lambda: dv.gram(n, L, R, self._wmask(nb), self.bdiag,
                                                          pair_mode=mode)))
            self._rayleigh_ritz(G, J, sel, kst, W, AW)
        except _Failure as f:
            self.failure = str(f)
            self.done = True
            return False
        self.it += 1
        return True

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
        ldw = dv.even(kj)
        W = dv.view_block(self.Wbuf, n, ldw)
        AW = dv.view_block(self.AWbuf, n, ldw)
        W.zero_()
        W[:, :kj] = out.to(torch.float64)
        return W, AW, kj, ldw, np.arange(kj)

    def _rayleigh_ritz(self, G, J, sel, kst, W, AW):
        m, n = self.m, self.n
        hp = self.have_p
        # row/col offsets of the blocks inside G
        rX, rW, rP = 0, m, m + kst
        cX, cW = 0, m
        cP = m + kst
        cAW = m + kst + (m if hp else 0)
        cAP = cAW + kst

        # W: Cholesky-QR with column dropping on the J sub-block
        # (lobpcg.py:475-481, :182-200), W never rewritten
        keep = list(range(J.size))
        mw = None
        while keep:
            ks = sel[keep]
            gww = G[rW + ks][:, cW + ks]
            try:
                _, minv = scaled_cholesky(gww, PIVOT_FLOOR)
                mw = minv
                break
            except NotSPD as err:
                del keep[err.pivot]
        self.pending += J.size - len(keep)
        if not keep:
            raise _Failure("BasisDegeneracy")
        wcols = sel[keep]                 # stored W columns in the basis

        # P_J: Cholesky-QR with floor; NotSPD drops P (lobpcg.py:484-494)
        mp = None
        if hp:
            try:
                gpp = G[rP + J][:, cP + J]
                _, mp = scaled_cholesky(gpp, PIVOT_FLOOR)
            except NotSPD:
                mp = None
                self.pending += 1

        # raw Gram sub-blocks
        gXAW = G[rX:rX + m][:, cAW + wcols]
        gXBW = G[rX:rX + m][:, cW + wcols]
        gWAW = G[rW + wcols][:, cAW + wcols]
        if hp:
            gXAP = G[rX:rX + m][:, cAP + J]
            gWAP = G[rW + wcols][:, cAP + J]
            gXBP = G[rX:rX + m][:, cP + J]
            gWBP = G[rW + wcols][:, cP + J]
            gPAP = G[rP + J][:, cAP + J]

        # Rayleigh-Ritz with the repair ladder (lobpcg.py:501-519)
        use_p = mp is not None
        while True:
            kw = mw.shape[1]
            kp = J.size if use_p else 0
            d = m + kw + kp
            ga = np.zeros((d, d))
            gb = np.zeros((d, d))
            sx, sw, sp = slice(0, m), slice(m, m + kw), slice(m + kw, d)
            ga[sx, sx] = np.diag(self.lam)
            gb[sx, sx] = np.eye(m)
            ga[sw, sw] = mw.T @ gWAW @ mw
            gb[sw, sw] = np.eye(kw)
            ga[sx, sw] = gXAW @ mw
            gb[sx, sw] = gXBW @ mw
            if kp:
                ga[sx, sp] = gXAP @ mp
                ga[sw, sp] = mw.T @ gWAP @ mp
                gb[sx, sp] = gXBP @ mp
                gb[sw, sp] = mw.T @ gWBP @ mp
                ga[sp, sp] = mp.T @ gPAP @ mp
                gb[sp, sp] = np.eye(kp)
            try:
                lam_new, c = gen_sym_eig(ga, gb, m, PIVOT_FLOOR)
                break
            except NotSPD as err:
                self.pending += 1
                if use_p:
                    use_p = False
                elif m <= err.pivot < m + kw and kw > 1:
                    keepc = np.arange(kw) != err.pivot - m
                    mw = mw[:, keepc]
                else:
                    raise _Failure("BasisDegeneracy")
        kw = mw.shape[1]
        cx = c[:m]
        cw = c[m:m + kw]
        cp = c[m + kw:]
        # fold the orthonormalization into raw-block coefficients
        cw_raw = np.zeros((kst, m))
        cw_raw[wcols] = mw @ cw
        if use_p:
            cp_raw = mp @ cp
            pcols = J.astype(np.int32)
        else:
            cp_raw = np.zeros((0, m))
            pcols = np.zeros(0, dtype=np.int32)
        dev = self.dev
        cxd = dv.to_device(cx, dev)
        cwd = dv.to_device(cw_raw, dev)
        cpd = dv.to_device(cp_raw, dev) if cp_raw.size else cxd
        pcd = dv.to_device(pcols, dev, torch.int32) if pcols.size else pos_dummy(dev)
        _timed("update", lambda: dv.update(
            n, m, self.X, self.AX, cxd, self.X2, self.AX2, w=W, aw=AW, kw=kst, cw=cwd,
            p=self.P if use_p else None, ap=self.AP if use_p else None, pcols=pcd,
            kp=pcols.size, cp=cpd, po=self.P2, apo=self.AP2, x_plus_p=True))
        self.X, self.X2 = self.X2, self.X
        self.AX, self.AX2 = self.AX2, self.AX
        self.P, self.P2 = self.P2, self.P
        self.AP, self.AP2 = self.AP2, self.AP
        self.have_p = True
        self.lam = lam_new

    def _check_state(self):
        g = self._gram_xx()
        err = np.abs(g - np.eye(self.m)).max()
        if err > 1e-10:
            raise RuntimeError(f"block lost B-orthonormality: max deviation {err:.3e}")

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
                dv.residual(n, m, self.X, self.AX, self.bdiag, lam_d, 0, 1.0, None, None, 0,
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
        vecs = vecs.clone() if _OPTS["return_device"] else dv.to_host(vecs).copy()
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


_DUMMY = {}


def pos_dummy(dev):
    t = _DUMMY.get(dev)
    if t is None:
        t = _DUMMY[dev] = torch.zeros(2, dtype=torch.int32, device=dev)
    return t


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
    """Staged solves with hard locking (lobpcg.py:580-653) -- needs the
    constraint path, which is not on the B200 path yet."""
    raise NotImplementedError("solve_staged needs hard-locking constraints (SURVEY 8f rank 1)")
