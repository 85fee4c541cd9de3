#!/usr/bin/env python3
"""Seeds 1 and 2 of the BASELINE shapes (SURVEY 8c harness rules: "also run
seeds 1 and 2"), from the REAL reference package, at matched iterations.

Run in the build container only (imports blockeig from /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_seeds.py

Cases (every run ends MaxIterReached, so the comparison is at a matched
iteration count, before the trajectories of degenerate clusters decorrelate):
  c1  32^3 scaled, m=4,  no T,   tol 1e-6, 120 it   (BASELINE configs[0] shape)
  c2  48^3 scaled, m=10, Jacobi, tol 1e-8,  60 it   (configs[1] shape, reduced grid)
  c3  40^3 scaled, m=16, Jacobi, tol 1e-6,  60 it   (configs[2] shape, reduced grid)
  c5  24^3 scaled, m=32, Jacobi, B = diag(U[1,2]) from PCG64(1000 + seed),
      tol 1e-6, 40 it                                (configs[4] shape, reduced)
Output: seeds12.npz with <case>_s<seed>_{eigenvalues, residual_norms,
hist_ritz, hist_resid, status, iterations_used, converged}.
"""
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
from blockeig import (  # noqa: E402
    DiagonalOperator,
    MatrixFreeOperator,
    SolverConfig,
    jacobi_preconditioner,
    laplacian3d,
    solve,
)

OUT = Path(__file__).parent

CASES = {   # name: (N, m, jacobi, diag_b, tol, max_iter)
    "c1": (32, 4, False, False, 1e-6, 120),
    "c2": (48, 10, True, False, 1e-8, 60),
    "c3": (40, 16, True, False, 1e-6, 60),
    "c5": (24, 32, True, True, 1e-6, 40),
}


def scaled_laplacian(N):
    s = float((N + 1) ** 2)
    L = laplacian3d((N, N, N))
    return MatrixFreeOperator(N ** 3, lambda v: s * L(v), spd=True,
                              diag=np.full(N ** 3, 6.0 * s))


def main():
    out = {}
    for name, (N, m, jac, diag_b, tol, max_iter) in CASES.items():
        for seed in (1, 2):
            A = scaled_laplacian(N)
            b = None
            if diag_b:
                bd = np.random.Generator(np.random.PCG64(1000 + seed)).uniform(1.0, 2.0, N ** 3)
                b = DiagonalOperator(bd)
            t0 = time.time()
            rep = solve(A, b=b, t=jacobi_preconditioner(A) if jac else None,
                        config=SolverConfig(block_size=m, tol=tol, max_iter=max_iter, seed=seed))
            k = f"{name}_s{seed}_"
            out[k + "eigenvalues"] = rep.eigenvalues
            out[k + "residual_norms"] = rep.residual_norms
            out[k + "hist_ritz"] = np.array([h.ritz for h in rep.history])
            out[k + "hist_resid"] = np.array([h.residual_norms for h in rep.history])
            out[k + "status"] = np.array(rep.status)
            out[k + "iterations_used"] = np.int64(rep.iterations_used)
            out[k + "converged"] = rep.converged
            print(name, seed, rep.status, rep.iterations_used, int(rep.converged.sum()),
                  f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(OUT / "seeds12.npz", **out)
    pencil_fixture()


def pencil_fixture():
    """The reference's private `_project_pencil` (lobpcg.py:299-340) on seeded
    random blocks, with and without exact_diagonal -> project_pencil.npz."""
    from blockeig.lobpcg import _project_pencil

    r = np.random.Generator(np.random.PCG64(77))
    n, m, nw, npj = 501, 4, 3, 2
    blocks = {k: r.standard_normal((n, c)) for k, c in
              [("x", m), ("ax", m), ("bx", m), ("w", nw), ("aw", nw), ("bw", nw),
               ("pj", npj), ("apj", npj), ("bpj", npj)]}
    lam = r.uniform(1.0, 5.0, m)
    out = dict(blocks, lam=lam)
    for exact in (False, True):
        ga, gb = _project_pencil(lam, blocks["x"], blocks["ax"], blocks["w"], blocks["aw"],
                                 blocks["bw"], blocks["pj"], blocks["apj"], blocks["bpj"],
                                 blocks["bx"], exact_diagonal=exact)
        out[f"ga_{int(exact)}"], out[f"gb_{int(exact)}"] = ga, gb
    ga, gb = _project_pencil(lam, blocks["x"], blocks["ax"], blocks["w"], blocks["aw"],
                             blocks["bw"], None, None, None, blocks["bx"])
    out["ga_nop"], out["gb_nop"] = ga, gb
    np.savez_compressed(OUT / "project_pencil.npz", **out)


if __name__ == "__main__":
    main()
