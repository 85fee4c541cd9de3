"""Every BASELINE.json configuration on one GPU through the public solve().

For each config: wall time of solve() (time-to-tol on converging runs,
time-to-max_iter otherwise; X0 generated on the device by K9 inside the
call, eigenvectors kept on the device), iterations/s, status, and
size-independent checks made with plain torch fp64 outside the product path:

  * residual_check  max_j | ||A x_j - lam_j B x_j|| - reported_j | / max(reported_j, tol)
                    (A x recomputed with a torch 7-point stencil)
  * orth            max |X^T B X - I|
  * ritz_monotone   Ritz values never increase between iterations (the
                    Rayleigh-Ritz space contains the previous X), up to 1e-10 rel
  * closed_form     max rel error of the converged columns vs the closed form
                    (B = I only)

Usage: python tools/bench_configs.py [C1 C1t C2 C3 C4 C5 W1 ...] > out.jsonl
(C1t = C1 with max_iter 1000, the converging time-to-tol run; W1 = the
weak-scaling 232^3 single-GPU point.)  Diagnostic/benchmark tool: the
numbers it prints are summarised in profiles/.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

CONFIGS = {
    # name: (N, m, jacobi, tol, max_iter, diagonal B)
    "C1": (32, 4, False, 1e-6, 200, False),
    "C1t": (32, 4, False, 1e-6, 1000, False),
    "C2": (128, 10, True, 1e-8, 300, False),
    "C3": (256, 16, True, 1e-6, 300, False),
    "C4": (464, 8, True, 1e-6, 50, False),
    "W1": (232, 8, True, 1e-6, 50, False),
    "C5": (192, 64, True, 1e-6, 200, True),
}


def lap7(x, N, s):
    """s * L7 x for x (N^3, k), x fastest, zero Dirichlet (torch fp64)."""
    k = x.shape[1]
    v = x.view(N, N, N, k)
    y = 6.0 * v
    y[:, :, 1:] -= v[:, :, :-1]
    y[:, :, :-1] -= v[:, :, 1:]
    y[:, 1:] -= v[:, :-1]
    y[:, :-1] -= v[:, 1:]
    y[1:] -= v[:-1]
    y[:-1] -= v[1:]
    return (s * y).view(-1, k)


def run(name):
    N, m, jac, tol, max_iter, diag_b = CONFIGS[name]
    s = float((N + 1) ** 2)
    A = pk.Laplacian3D((N, N, N), scale=s)
    T = pk.jacobi_preconditioner(A) if jac else None
    B = None
    d = None
    if diag_b:
        dh = np.random.Generator(np.random.PCG64(1000)).uniform(1.0, 2.0, N ** 3)
        B = pk.DiagonalOperator(dh)
        d = B.d
    cfg = pk.SolverConfig(block_size=m, tol=tol, max_iter=max_iter, seed=0)
    torch.cuda.synchronize()
    with pk.device_options(return_device=True):
        # solve() = LOBPCGRun + step loop + report, timed phase by phase
        t0 = time.perf_counter()
        run_ = pk.LOBPCGRun(A, b=B, t=T, config=cfg)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        while run_.step():
            pass
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rep = run_.report()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        dt = t3 - t0
    del run_
    # per-kernel CUDA-event times over a few steps (timer mode: Python-driven steps)
    ktimes = {}

    def timer(nm, fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        ktimes.setdefault(nm, []).append((a, b))
        return r

    with pk.device_options(return_device=True):
        r2 = pk.LOBPCGRun(A, b=B, t=T, config=cfg)
        for _ in range(2):
            r2.step()
        with pk.device_options(timer=timer):
            for _ in range(3):
                r2.step()
        torch.cuda.synchronize()
    del r2
    kern = {k: round(sum(a.elapsed_time(b) for a, b in v) / 3, 4) for k, v in ktimes.items()}
    X = rep.eigenvectors
    lam = torch.as_tensor(rep.eigenvalues, device=X.device)
    AX = lap7(X, N, s)
    BX = X if d is None else d[:, None] * X
    R = AX - BX * lam[None, :]
    rn = torch.linalg.vector_norm(R, dim=0).cpu().numpy()
    del AX, R
    G = X.T @ BX
    orth = float((G - torch.eye(m, device=X.device, dtype=G.dtype)).abs().max())
    del BX, G
    rep_rn = np.asarray(rep.residual_norms)
    resid_check = float(np.max(np.abs(rn - rep_rn) / np.maximum(rep_rn, tol)))
    ritz = np.array([h.ritz for h in rep.history])
    mono = float(np.max((ritz[1:] - ritz[:-1]) / np.abs(ritz[:-1]))) if len(ritz) > 1 else 0.0
    out = {
        "config": name, "N": N, "n": N ** 3, "m": m, "jacobi": jac, "diag_B": diag_b,
        "tol": tol, "max_iter": max_iter, "status": rep.status,
        "iterations": rep.iterations_used, "converged": int(np.sum(rep.converged)),
        "solve_s": dt, "it_per_s": rep.iterations_used / dt,
        "setup_s": t1 - t0, "loop_s": t2 - t1, "report_s": t3 - t2,
        "loop_ms_per_it": 1e3 * (t2 - t1) / max(rep.iterations_used, 1),
        "kernel_ms_per_step": kern,
        "residual_check": resid_check, "orth": orth, "ritz_max_increase_rel": mono,
        "lam_head": [float(v) for v in rep.eigenvalues[:4]],
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
    }
    if not diag_b:
        exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
        conv = np.asarray(rep.converged, dtype=bool)
        out["closed_form_rel_err_converged"] = (
            float(np.max(np.abs(rep.eigenvalues[conv] - exact[conv]) / exact[conv]))
            if conv.any() else None)
        out["closed_form_rel_err_all"] = float(np.max(np.abs(rep.eigenvalues - exact) / exact))
    del X, rep
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    return out


def main():
    names = sys.argv[1:] or ["C1", "C1t", "C2", "C3", "C4", "C5"]
    # warm-up (kernel attributes, tensor maps, allocator)
    pk.solve(pk.Laplacian3D((16, 16, 16)), config=pk.SolverConfig(block_size=4, max_iter=3))
    for nm in names:
        print(json.dumps(run(nm)), flush=True)


if __name__ == "__main__":
    main()
