"""Host fp64 algebra on the small projected matrices (<= 3m x 3m).

The reference does this on the host too (multivec.py:89-211, scipy LAPACK).
Here the LAPACK routines are called directly (scipy.linalg.lapack: dpotrf,
dtrtrs, dtrtri, dsyevr) to keep the per-iteration host latency -- which sits
on the critical path between the two device passes -- small.

The reference writes its Cholesky out row by row so that a failure names its
pivot (the first numerically dependent column), which drives the basis-repair
ladder of lobpcg.py:182-200 and :501-519.  dpotrf computes the same factor;
the first pivot that is non-positive, non-finite or below the relative floor
is recovered from its diagonal (pivot_j = R_jj^2 vs floor * G_jj), so the
NotSPD(pivot) contract is unchanged.  The symmetric eigensolver of these
helpers (multivec API, drift repair, exit refresh) is dsyevr, the driver
scipy.linalg.eigh (the reference's call) uses.  The per-iteration
Rayleigh-Ritz step itself runs in the library (NativeRitz ->
b2l_rayleigh_ritz, csrc/rr.cu): native congruence + tridiagonal QR with the
eigenvectors of numerically degenerate clusters aligned to the current Ritz
vectors, LAPACK above a 64 x 64 pencil.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import lapack

# Pencils above 64 x 64 (m >= 22) go through scipy's LAPACK / BLAS, whose
# OpenBLAS is multithreaded: on these sizes the thread hand-offs cost more
# than they save (C5: 44.8 -> 43.1 ms per iteration on the B200 host) and the
# rounding depends on the host's core count.  Those calls run with one BLAS
# thread (scoped: the caller's setting is restored), so the Rayleigh-Ritz
# step is single-threaded and host-independent, as the reference's solve is.
_BLAS_LIMIT_M = 22
_tp_ctl = None


def _one_blas_thread():
    """Scope the BLAS thread pool to one thread (threadpoolctl).  The limit is
    process-wide while it is held (OpenBLAS has one pool), so other host
    threads' BLAS calls run single-threaded meanwhile.  Without threadpoolctl
    the caller's setting stays (rounding then follows the host's core
    count, as the reference's own BLAS calls do)."""
    global _tp_ctl
    if _tp_ctl is None:
        try:
            from threadpoolctl import ThreadpoolController

            _tp_ctl = ThreadpoolController()
        except ImportError:
            _tp_ctl = False
    if _tp_ctl is False:
        return _NoLimit()
    return _tp_ctl.limit(limits=1, user_api="blas")


class _NoLimit:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_potrf = lapack.dpotrf
_trtrs = lapack.dtrtrs
_trtri = lapack.dtrtri
_syevr = lapack.dsyevr


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
    if k == 0:
        return np.zeros((0, 0))
    r, info = _potrf(g, lower=0, clean=1, overwrite_a=0)
    if info < 0:
        raise ValueError(f"dpotrf: illegal argument {-info}")
    ok = k if info == 0 else info - 1          # leading pivots dpotrf accepted
    piv = np.diag(r)[:ok] ** 2
    gd = np.diag(g)[:ok]
    bad = ~(piv > pivot_floor * gd) | ~np.isfinite(piv)
    if bad.any():
        raise NotSPD(int(np.flatnonzero(bad)[0]))
    if info > 0:
        raise NotSPD(info - 1)
    return r


def sym_eig(g: np.ndarray):
    """Ascending eigenpairs of a symmetric matrix, upper triangle read
    (scipy.linalg.eigh(g, lower=False), multivec.py:161-171)."""
    g = np.asarray(g, dtype=np.float64)
    w, v, _, _, info = _syevr(g, compute_v=1, range="A", lower=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"dsyevr failed ({info})")
    return w, v


def _lsolve_t(r, b):
    """R^{-T} b for upper R (dtrtrs, trans='T')."""
    x, info = _trtrs(r, b, lower=0, trans=1)
    if info != 0:
        raise np.linalg.LinAlgError(f"dtrtrs failed ({info})")
    return x


def gen_sym_eig(ga: np.ndarray, gb: np.ndarray, want: int, pivot_floor: float = 0.0):
    """Smallest ``want`` pairs of ga c = lam gb c via gb = R^T R
    (multivec.py:174-211); only upper triangles are read."""
    ga = np.triu(ga) + np.triu(ga, 1).T
    r = cholesky(gb, pivot_floor)
    t = _lsolve_t(r, ga)
    t = _lsolve_t(r, np.ascontiguousarray(t.T))
    t = 0.5 * (t + t.T)
    vals, vecs = sym_eig(t)
    c, info = _trtrs(r, vecs[:, :want], lower=0, trans=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"dtrtrs failed ({info})")
    return vals[:want], c


def chol_solve(r: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """(R^T R) z = rhs for upper R (multivec.chol_solve, multivec.py:149-158)."""
    r = np.asarray(r, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    if r.ndim != 2 or r.shape[0] != r.shape[1]:
        raise ValueError(f"factor must be square, got shape {r.shape}")
    if r.shape[0] == 0:
        return rhs.copy()
    u = _lsolve_t(r, rhs)
    z, info = _trtrs(r, u, lower=0, trans=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"dtrtrs failed ({info})")
    return z


def upper_inverse(r: np.ndarray) -> np.ndarray:
    """R^{-1} for an upper-triangular R (used to fold Cholesky-QR factors
    into the Gram blocks and update coefficients instead of rewriting the
    tall block, which the reference does with tri_solve_right)."""
    k = r.shape[0]
    if k == 0:
        return np.zeros((0, 0))
    inv, info = _trtri(r, lower=0, unitdiag=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"dtrtri failed ({info})")
    return np.triu(inv)


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


class RitzFailure(Exception):
    """b2l_rayleigh_ritz exhausted the repair ladder (BasisDegeneracy)."""

    def __init__(self, fallbacks):
        super().__init__("BasisDegeneracy")
        self.fallbacks = int(fallbacks)


class NativeRitz:
    """Host Rayleigh-Ritz step in the native library (b2l_rayleigh_ritz):
    W / P Cholesky-QR with the column-drop and P-drop ladders, the projected
    pencil, the generalised eigensolve with its retry ladder and the
    coefficient folding of lobpcg.py:475-540, in one call.  Output buffers are
    reused across iterations."""

    def __init__(self, m):
        import ctypes as C

        from . import _lib

        self._C = C
        self._lib = _lib
        self.m = m
        self.lam = np.zeros(m)
        self.coef = np.zeros(3 * m * m)
        self.pcols = np.zeros(m, dtype=np.int32)
        self._kp = C.c_int()
        self._fb = C.c_int()
        # absolute eigenvalue gap of a numerically degenerate cluster
        # (b2l_set_rr_align): the solver sets a tenth of its smallest lock
        # threshold before each step; 0 = no alignment
        self.align = 0.0

    def _scope(self):
        return _one_blas_thread() if self.m >= _BLAS_LIMIT_M else _NoLimit()

    def __call__(self, m, kst, have_p, g1, g2, lam, jact, sel, pivot_floor):
        C, L = self._C, self._lib
        lib = L.load()
        g1 = np.ascontiguousarray(g1, dtype=np.float64)
        g2 = np.ascontiguousarray(g2, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        jact = np.ascontiguousarray(jact, dtype=np.int32)
        sel = np.ascontiguousarray(sel, dtype=np.int32)
        dp, ip = L.c_dp, L.c_ip
        lib.b2l_set_rr_align(float(self.align))
        with self._scope():
            rc = lib.b2l_rayleigh_ritz(
                m, kst, int(have_p), g1.ctypes.data_as(dp), g1.shape[1], g2.ctypes.data_as(dp),
                lam.ctypes.data_as(dp), jact.ctypes.data_as(ip), jact.size,
                sel.ctypes.data_as(ip), float(pivot_floor), self.lam.ctypes.data_as(dp),
                self.coef.ctypes.data_as(dp), self.pcols.ctypes.data_as(ip), C.byref(self._kp),
                C.byref(self._fb))
        if rc == L.EDEGENERATE:
            raise RitzFailure(self._fb.value)
        L.check(rc, "b2l_rayleigh_ritz")
        kp = self._kp.value
        ncoef = m * m + kst * m + kp * m
        return (self.lam.copy(), self.coef[:ncoef].copy(), self.pcols[:kp].copy(),
                self._fb.value)

    def begin(self, m, kst, have_p, g1, jact, sel, pivot_floor):
        """The G1-only half (b2l_rayleigh_ritz_begin); `finish` completes it."""
        C, L = self._C, self._lib
        lib = L.load()
        self._g1 = np.ascontiguousarray(g1, dtype=np.float64)
        jact = np.ascontiguousarray(jact, dtype=np.int32)
        sel = np.ascontiguousarray(sel, dtype=np.int32)
        self._kst = kst
        with self._scope():
            rc = lib.b2l_rayleigh_ritz_begin(
                m, kst, int(have_p), self._g1.ctypes.data_as(L.c_dp), self._g1.shape[1],
                jact.ctypes.data_as(L.c_ip), jact.size, sel.ctypes.data_as(L.c_ip),
                float(pivot_floor), C.byref(self._fb))
        self._begin_rc = rc
        if rc != 0 and rc != L.EDEGENERATE:
            L.check(rc, "b2l_rayleigh_ritz_begin")

    def finish(self, m, g2, lam):
        """The G2 half: same return value as __call__."""
        C, L = self._C, self._lib
        lib = L.load()
        if self._begin_rc == L.EDEGENERATE:
            raise RitzFailure(self._fb.value)
        g2 = np.ascontiguousarray(g2, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        dp, ip = L.c_dp, L.c_ip
        lib.b2l_set_rr_align(float(self.align))
        with self._scope():
            rc = lib.b2l_rayleigh_ritz_finish(
                g2.ctypes.data_as(dp), lam.ctypes.data_as(dp), self.lam.ctypes.data_as(dp),
                self.coef.ctypes.data_as(dp), self.pcols.ctypes.data_as(ip), C.byref(self._kp),
                C.byref(self._fb))
        if rc == L.EDEGENERATE:
            raise RitzFailure(self._fb.value)
        L.check(rc, "b2l_rayleigh_ritz_finish")
        kp = self._kp.value
        ncoef = m * m + self._kst * m + kp * m
        return (self.lam.copy(), self.coef[:ncoef].copy(), self.pcols[:kp].copy(),
                self._fb.value)
