"""CPU oracle for the LOBPCG hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package
``blockeig`` (``/root/reference/pkg/src/blockeig``) for the one path this
repository accelerates: LOBPCG with soft locking on the matrix-free 7-point
Laplacian (identity or Jacobi preconditioner, identity or diagonal B).

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``, and only as the
checker or as the timed CPU baseline.  The product package
``paper_0705_2626_b200`` never imports it; the GPU path has no CPU fallback.

Parity pin: ``run_lobpcg`` reproduces the reference's golden trajectory
``pkg/demos/convergence_history.csv`` (20^3, m=10, Jacobi, tol 1e-6, seed 2)
bit for bit -- see ``tests/test_oracle.py`` and ``tests/golden/``.  It uses the
same numpy/scipy primitives in the same order as the reference so that the
floating-point results are identical, not merely close.

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import eigh, solve_triangular

PIVOT_FLOOR = 1e-8   # lobpcg.py:57
DRIFT_LIMIT = 1e-11  # lobpcg.py:66


class PivotFailure(Exception):
    """Cholesky pivot failure carrying the zero-based pivot (multivec.py:34-48)."""

    def __init__(self, pivot):
        super().__init__(f"pivot {pivot}")
        self.pivot = int(pivot)


# --------------------------------------------------------------------------
# operators (operators.py)


def stencil7(x, nx, ny, nz, scale=None):
    """7-point Dirichlet Laplacian on an (n, k) block, x fastest.

    Restates ``Laplacian3D._apply`` (operators.py:184-196): y = 6 f, then the
    six neighbour subtractions in the fixed order x-, x+, y-, y+, z-, z+.  With
    ``scale`` the result is multiplied by it afterwards, which is what the
    harness ``MatrixFreeOperator(n, lambda v: s * L(v))`` (operators.py:104-121)
    computes.  Like the reference it returns an F-order (n, k) view: the
    memory order matters for bitwise parity because OpenBLAS picks its
    summation order from operand layout.
    """
    x = np.asarray(x, dtype=np.float64)
    k = x.shape[1]
    f = np.ascontiguousarray(x.T).reshape(k, nz, ny, nx)
    y = 6.0 * f
    y[:, :, :, 1:] -= f[:, :, :, :-1]
    y[:, :, :, :-1] -= f[:, :, :, 1:]
    y[:, :, 1:, :] -= f[:, :, :-1, :]
    y[:, :, :-1, :] -= f[:, :, 1:, :]
    y[:, 1:, :, :] -= f[:, :-1, :, :]
    y[:, :-1, :, :] -= f[:, 1:, :, :]
    out = y.reshape(k, nz * ny * nx).T
    if scale is not None:
        out = scale * out
    return out


def closed_form_smallest(nx, ny, nz, m, scale=1.0):
    """m smallest eigenvalues of the (scaled) Dirichlet 7-point Laplacian.

    Formula of problems.py:44-82 (4 sum sin^2(i pi / 2(n+1))), restricted to
    modes with every index <= m, which always contain the m smallest
    (SURVEY 8c shortcut), so it stays cheap at 464^3.
    """
    def axis(cnt):
        modes = np.arange(1, min(cnt, m) + 1)
        return 4.0 * np.sin(modes * np.pi / (2.0 * (cnt + 1))) ** 2

    tx, ty, tz = axis(nx), axis(ny), axis(nz)
    vals = (tx[:, None, None] + ty[None, :, None] + tz[None, None, :]).ravel()
    return np.sort(vals)[:m] * scale


def seeded_block(n, k, seed):
    """Reference initial block, multivec.py:220-229 (PCG64 uniform(-1,1))."""
    return np.random.Generator(np.random.PCG64(seed)).uniform(-1.0, 1.0, size=(n, k))


# --------------------------------------------------------------------------
# small dense algebra (multivec.py)


def chol_upper(g, floor=0.0):
    """Row-by-row upper Cholesky with relative pivot floor (multivec.py:89-122)."""
    g = np.asarray(g, dtype=np.float64)
    k = g.shape[0]
    r = np.zeros((k, k))
    for j in range(k):
        piv = g[j, j] - r[:j, j] @ r[:j, j]
        if not (piv > floor * g[j, j]) or not np.isfinite(piv):
            raise PivotFailure(j)
        d = np.sqrt(piv)
        r[j, j] = d
        if j + 1 < k:
            r[j, j + 1:] = (g[j, j + 1:] - r[:j, j] @ r[:j, j + 1:]) / d
    return r


def right_solve(x, r):
    """Z with Z r = X (multivec.py:125-146)."""
    if r.shape[0] == 0:
        return x.copy()
    return solve_triangular(r, x.T, trans="T", lower=False).T


def pencil_smallest(ga, gb, want, floor=0.0):
    """Smallest ``want`` eigenpairs of ga c = lam gb c, upper triangles only
    (multivec.py:174-211)."""
    ga = np.triu(ga) + np.triu(ga, 1).T
    r = chol_upper(gb, floor)
    t = solve_triangular(r, ga, trans="T", lower=False)
    t = solve_triangular(r, t.T, trans="T", lower=False)
    t = 0.5 * (t + t.T)
    w, v = eigh(t, lower=False)
    return w[:want], solve_triangular(r, v[:, :want], trans="N", lower=False)


def col_norms(x):
    return np.linalg.norm(x, axis=0)  # multivec.py:214-217


# --------------------------------------------------------------------------
# LOBPCG (lobpcg.py)


def normalize_block(x, bx, floor=0.0):
    """Scaled Cholesky-QR, lobpcg.py:147-179. Returns (x', bx', r_eff)."""
    same = bx is x
    sq = np.einsum("ij,ij->j", x, bx)
    badmask = ~(sq > 0.0) | ~np.isfinite(sq)
    if badmask.any():
        raise PivotFailure(int(np.flatnonzero(badmask)[0]))
    sc = np.sqrt(sq)
    xs = x / sc
    bxs = xs if same else bx / sc
    r = chol_upper(xs.T @ bxs, floor)
    xo = right_solve(xs, r)
    return xo, (xo if same else right_solve(bxs, r)), r * sc[None, :]


def normalize_dropping(w, bw):
    """lobpcg.py:182-200: drop each failing pivot column and retry."""
    same = bw is w
    total = w.shape[1]
    keep = list(range(total))
    while keep:
        wk = w[:, keep]
        bwk = wk if same else bw[:, keep]
        try:
            wo, bwo, _ = normalize_block(wk, bwk, PIVOT_FLOOR)
            return wo, bwo, total - len(keep)
        except PivotFailure as e:
            del keep[e.pivot]
    return w[:, :0], bw[:, :0], total


def exact_ritz(x, ax, bx, bop):
    """lobpcg.py:280-296 (no operator applications); bop is None for B = I."""
    x, bx, r = normalize_block(x, bx)
    ax = right_solve(ax, r)
    lam, q = eigh(x.T @ ax, lower=False)
    x = x @ q
    ax = ax @ q
    bx = x if bop is None else bx @ q
    return x, ax, bx, lam


def assemble_pencil(lam, x, w, aw, bw, p, ap, bp):
    """Upper blocks of the projected pencil on [x, w, p] (lobpcg.py:299-340)."""
    m, kw = x.shape[1], w.shape[1]
    kp = 0 if p is None else p.shape[1]
    d = m + kw + kp
    ga = np.zeros((d, d))
    gb = np.zeros((d, d))
    X, W, P = slice(0, m), slice(m, m + kw), slice(m + kw, d)
    ga[X, X] = np.diag(lam)
    gb[X, X] = np.eye(m)
    ga[W, W] = w.T @ aw
    gb[W, W] = np.eye(kw)
    ga[X, W] = x.T @ aw
    gb[X, W] = x.T @ bw
    if kp:
        ga[X, P] = x.T @ ap
        ga[W, P] = w.T @ ap
        gb[X, P] = x.T @ bp
        gb[W, P] = w.T @ bp
        ga[P, P] = p.T @ ap
        gb[P, P] = np.eye(kp)
    return ga, gb


@dataclass
class OracleResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    iterations_used: int
    converged: np.ndarray
    residual_norms: np.ndarray
    lock_iterations: np.ndarray
    status: str
    basis_fallbacks: int
    hist_ritz: list = field(default_factory=list)
    hist_resid: list = field(default_factory=list)
    hist_active: list = field(default_factory=list)
    iter_times: list = field(default_factory=list)
    drift_repairs: int = 0


def run_lobpcg(apply_a, n, m, *, bdiag=None, apply_b=None, tinv=None, apply_t=None, x0=None,
               tol=1e-6, max_iter=200, seed=0, relative_tol=False,
               record=True, timer=False):
    """Restatement of ``solve`` (lobpcg.py:343-577) without hard constraints.

    apply_a: callable (n,k)->(n,k).  bdiag: (n,) diagonal of B or None;
    apply_b: a generic B callable instead (BX, BW, BP carried by recurrence,
    lobpcg.py:396, :476, :533-538).
    tinv: (n,) array or scalar applied as ``tinv[:, None] * w`` (Jacobi,
    operators.py:297-298); apply_t: generic callable alternative.
    ``timer=True`` records a perf_counter stamp at the top of every
    iteration (used by bench.py's CPU baseline only).
    """
    bop = apply_b if apply_b is not None else (
        None if bdiag is None else (lambda v: bdiag[:, None] * v))
    if x0 is not None:
        x = np.array(x0, dtype=np.float64, copy=True)
    else:
        x = seeded_block(n, m, seed)
    bx = bop(x) if bop else x
    x, bx, _ = normalize_block(x, bx)
    ax = apply_a(x)
    lam, q = eigh(x.T @ ax, lower=False)
    x = x @ q
    ax = ax @ q
    bx = x if bop is None else bx @ q

    res = OracleResult(None, None, 0, None, None, None, "", 0)
    active = np.ones(m, dtype=bool)
    lock_it = np.full(m, -1, dtype=np.int64)
    p = ap = bp = None
    pend = 0
    fallbacks = 0
    fail = None
    norms = np.zeros(m)
    last_it = 0
    for it in range(max_iter + 1):
        if timer:
            res.iter_times.append(time.perf_counter())
        drift = np.abs(x.T @ bx - np.eye(m)).max()
        if drift > DRIFT_LIMIT:
            try:
                x, ax, bx, lam = exact_ritz(x, ax, bx, bop)
                res.drift_repairs += 1
            except PivotFailure:
                fail = "BasisDegeneracy"
                break
        wfull = ax - bx * lam
        norms = col_norms(wfull)
        thr = tol * col_norms(ax) if relative_tol else np.full(m, tol)
        newly = active & (norms < thr)
        lock_it[newly] = it
        active = active & ~newly
        last_it = it
        if record:
            res.hist_ritz.append(lam.copy())
            res.hist_resid.append(norms.copy())
            res.hist_active.append(active.copy())
        fallbacks += pend
        pend = 0
        if not active.any() or it == max_iter:
            break

        J = np.flatnonzero(active)
        w = wfull[:, J]
        if apply_t is not None:
            w = np.asarray(apply_t(w), dtype=np.float64)
        elif tinv is not None:
            w = tinv[:, None] * w if np.ndim(tinv) else tinv * w
        bw = bop(w) if bop else w
        w, bw, dropped = normalize_dropping(w, bw)
        pend += dropped
        if w.shape[1] == 0:
            fail = "BasisDegeneracy"
            break
        aw = apply_a(w)

        pj = apj = bpj = None
        if p is not None:
            pj, apj = p[:, J], ap[:, J]
            bpj = pj if bop is None else bp[:, J]
            try:
                pj, bpj, reff = normalize_block(pj, bpj, PIVOT_FLOOR)
                apj = right_solve(apj, reff)
            except PivotFailure:
                pj = apj = bpj = None
                pend += 1

        while True:
            ga, gb = assemble_pencil(lam, x, w, aw, bw, pj, apj, bpj)
            try:
                lam_new, c = pencil_smallest(ga, gb, m, PIVOT_FLOOR)
                break
            except PivotFailure as e:
                pend += 1
                if pj is not None:
                    pj = apj = bpj = None
                elif m <= e.pivot < m + w.shape[1] and w.shape[1] > 1:
                    sel = np.arange(w.shape[1]) != e.pivot - m
                    w, aw = w[:, sel], aw[:, sel]
                    bw = w if bop is None else bw[:, sel]
                else:
                    fail = "BasisDegeneracy"
                    break
        if fail is not None:
            break
        kw = w.shape[1]
        cx, cw, cp = c[:m], c[m:m + kw], c[m + kw:]
        pn = w @ cw
        apn = aw @ cw
        if pj is not None:
            pn += pj @ cp
            apn += apj @ cp
        if bop is None:
            bpn = pn
        else:
            bpn = bw @ cw
            if pj is not None:
                bpn += bpj @ cp
        x = x @ cx + pn
        ax = ax @ cx + apn
        bx = x if bop is None else bx @ cx + bpn
        p, ap, bp = pn, apn, (pn if bop is None else bpn)
        lam = lam_new

    fallbacks += pend
    if fail is None:
        try:
            x, ax, bx, lam = exact_ritz(x, ax, bx, bop)
            norms = col_norms(ax - bx * lam)
        except PivotFailure:
            fail = "BasisDegeneracy"
    conv = ~active
    if fail is not None:
        status = f"Failed({fail})"
    elif fallbacks:
        status = f"BasisFallback({fallbacks})"
    elif conv.all():
        status = "Converged"
    else:
        status = "MaxIterReached"
    res.eigenvalues = lam.copy()
    res.eigenvectors = x
    res.iterations_used = last_it
    res.converged = conv
    res.residual_norms = norms
    res.lock_iterations = lock_it
    res.status = status
    res.basis_fallbacks = fallbacks
    return res


def laplacian_case(N, m, *, precond="jacobi", scaled=True, bseed=None, x0=None,
                   tol=1e-6, max_iter=200, seed=0, record=True, timer=False):
    """The BASELINE harness: A = s L7 with s=(N+1)^2 exact, Jacobi
    = 1/(6s), optional B = diag(U[1,2]) from PCG64(bseed)."""
    n = N ** 3
    s = float((N + 1) ** 2) if scaled else None
    diag = 6.0 * (s if s is not None else 1.0)
    bdiag = None
    if bseed is not None:
        bdiag = np.random.Generator(np.random.PCG64(bseed)).uniform(1.0, 2.0, n)
    tinv = None
    if precond == "jacobi":
        tinv = 1.0 / np.full(n, diag)
    return run_lobpcg(lambda v: stencil7(v, N, N, N, s), n, m, bdiag=bdiag,
                      tinv=tinv, x0=x0, tol=tol, max_iter=max_iter, seed=seed,
                      record=record, timer=timer)
