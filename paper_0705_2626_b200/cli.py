"""``blockeig-bench`` on the B200 path (reference cli.py).

Same flags, defaults, exit codes and output files as the reference driver
(cli.py:108-211 flags, :275-294 JSON record, :297-304 history CSV
``iter,j,ritz,resid,active``, :58-96 LOBX eigenvector container), so runs can
be scripted and chained exactly like the reference's:

    python -m paper_0705_2626_b200.cli -n 64 64 64 -vrand 8 -tol 1e-8 \\
        -json run.json -csv hist.csv -out_evecs modes.bin
    python -m paper_0705_2626_b200.cli -n 64 64 64 -vrand 8 -constraints modes.bin

B200 additions (absent from the reference): ``-scaled 1`` applies the
BASELINE harness scale s = (N+1)^2 to the operator (the analytic
column is scaled with it), ``-device K`` picks the GPU, and ``-ngpu P`` runs
the z-slab partition when launched with P ranks under torchrun.

Exit codes: 0 full convergence, 2 partial convergence (budget exhausted),
1 errors (flags, files, solver failure).
"""

from __future__ import annotations

import argparse
import json
import os
import struct
import sys
import time
from dataclasses import dataclass

import numpy as np

__all__ = ["main", "sweep", "build_parser", "save_eigenvectors", "load_eigenvectors",
           "EXIT_OK", "EXIT_ERROR", "EXIT_PARTIAL"]

EXIT_OK, EXIT_ERROR, EXIT_PARTIAL = 0, 1, 2

SWEEP_DEFAULTS = {
    "inner_iter": (0, 1, 2, 5, 10, 15, 20),
    "block_size": (1, 2, 4, 8, 16),
}

# LOBX eigenvector container (cli.py:58-96): little-endian header
# magic "LOBX", u32 version = 1, u64 n, u64 k; then n*k f64 column-major.
_LOBX = struct.Struct("<4sIQQ")
_LOBX_MAGIC, _LOBX_VERSION = b"LOBX", 1


def save_eigenvectors(path, x):
    """Write an (n, k) block (numpy or CUDA tensor) as a LOBX file."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    block = np.asarray(x, dtype=np.float64)
    if block.ndim != 2:
        raise ValueError(f"eigenvector block must be 2-d, got shape {block.shape}")
    rows, cols = block.shape
    with open(path, "wb") as fh:
        fh.write(_LOBX.pack(_LOBX_MAGIC, _LOBX_VERSION, rows, cols))
        fh.write(np.asfortranarray(block).astype("<f8", copy=False).tobytes(order="F"))


def load_eigenvectors(path):
    """Read a LOBX file back as an (n, k) float64 array."""
    with open(path, "rb") as fh:
        head = fh.read(_LOBX.size)
        if len(head) < _LOBX.size:
            raise ValueError(f"{path}: truncated header")
        magic, version, rows, cols = _LOBX.unpack(head)
        if magic != _LOBX_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}")
        if version != _LOBX_VERSION:
            raise ValueError(f"{path}: unsupported version {version}")
        body = fh.read()
    if len(body) != 8 * rows * cols:
        raise ValueError(f"{path}: payload holds {len(body)} bytes, expected {8 * rows * cols}")
    return np.frombuffer(body, dtype="<f8").astype(np.float64).reshape((rows, cols), order="F")


class _ArgParser(argparse.ArgumentParser):
    """Malformed flags exit with code 1 (not argparse's 2)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_ERROR)


def build_parser():
    p = _ArgParser(prog="blockeig-bench", allow_abbrev=False,
                   description="Block preconditioned eigensolver benchmark on the 3-d "
                               "7-point Dirichlet Laplacian (B200 path).")
    add = p.add_argument
    add("-n", nargs=3, type=int, default=[10, 10, 10], metavar=("NX", "NY", "NZ"),
        help="grid dimensions (default 10 10 10)")
    add("-vrand", "-n_eigs", dest="m", type=int, default=5, metavar="M",
        help="block size: number of eigenpairs, started from M random vectors (default 5)")
    add("-seed", type=int, default=0, help="random seed for the initial block")
    add("-tol", type=float, default=1e-6, help="per-vector residual tolerance (default 1e-6)")
    add("-itr", type=int, default=200, metavar="K", help="maximum outer iterations (default 200)")
    add("-pcgitr", type=int, default=0, metavar="P",
        help="inner PCG steps per preconditioner application; 0 applies the base "
             "preconditioner directly (default 0)")
    add("-precond", choices=("none", "jacobi"), default="jacobi",
        help="base preconditioner (default jacobi)")
    add("-verb", type=int, default=1, help="0 silent, 1 summary, 2 per-iteration (default 1)")
    add("-full_out", type=int, choices=(0, 1), default=0,
        help="1 puts the per-iteration history into the JSON record (default 0)")
    add("-json", dest="json_path", metavar="PATH", help="write the run record as JSON")
    add("-csv", dest="csv_path", metavar="PATH",
        help="write the per-iteration history (or the sweep table) as CSV")
    add("-constraints", dest="constraints_path", metavar="PATH",
        help="LOBX eigenvectors of a prior run to hard-lock (the solve targets the next "
             "eigenpairs up)")
    add("-out_evecs", dest="out_evecs_path", metavar="PATH",
        help="write the computed eigenvectors (LOBX) for a later -constraints run")
    add("-sweep", choices=tuple(SWEEP_DEFAULTS), help="parameter sweep instead of one solve")
    add("-sweep_values", metavar="V1,V2,...",
        help="values of the swept parameter (defaults: inner_iter 0,1,2,5,10,15,20; "
             "block_size 1,2,4,8,16)")
    # B200 additions
    add("-scaled", type=int, choices=(0, 1), default=0,
        help="1: operator s*L with s = (NX+1)^2 (the BASELINE harness scale)")
    add("-device", type=int, default=None, metavar="K", help="CUDA device (default: current)")
    add("-ngpu", type=int, default=1, metavar="P",
        help="z-slab ranks; must match WORLD_SIZE when launched with torchrun")
    return p


def _check(parser, a):
    if min(a.n) < 1:
        parser.error(f"-n dimensions must be positive, got {a.n}")
    if a.m < 1:
        parser.error(f"block size must be positive, got {a.m}")
    if not a.tol > 0.0:
        parser.error(f"-tol must be positive, got {a.tol}")
    if a.itr < 1:
        parser.error(f"-itr must be positive, got {a.itr}")
    if a.pcgitr < 0:
        parser.error(f"-pcgitr must be nonnegative, got {a.pcgitr}")
    if a.verb < 0:
        parser.error(f"-verb must be nonnegative, got {a.verb}")
    if a.ngpu < 1:
        parser.error(f"-ngpu must be positive, got {a.ngpu}")


@dataclass
class _Env:
    """Device / rank context of one CLI invocation."""

    rank: int = 0
    world: int = 1

    @property
    def lead(self):
        return self.rank == 0


def _setup(a) -> _Env:
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.ngpu != world:
        raise ValueError(f"-ngpu {a.ngpu} but {world} rank(s) launched "
                         "(use torchrun --nproc-per-node for P > 1)")
    if world > 1:
        import torch.distributed as dist

        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return _Env(dist.get_rank(), world)
    if a.device is not None:
        torch.cuda.set_device(a.device)
    return _Env()


def _operator(a, env: _Env):
    from . import operators as ops

    grid = ops.Grid3D(*a.n)
    scale = float((a.n[0] + 1) ** 2) if a.scaled else 1.0
    if env.world > 1:
        from .distributed import SlabLaplacian3D

        return SlabLaplacian3D(grid, scale=scale), grid, scale
    return ops.Laplacian3D(grid, scale=scale), grid, scale


def _precond(op, kind, steps):
    from .operators import jacobi_preconditioner
    from .pcg import inner_pcg_preconditioner

    base = jacobi_preconditioner(op) if kind == "jacobi" else None
    return base if steps == 0 else inner_pcg_preconditioner(op, base, steps)


def _precond_name(kind, steps):
    return f"pcg:{steps}" if steps > 0 else kind


def _echo(a):
    return {"n": [int(v) for v in a.n], "m": int(a.m), "seed": int(a.seed),
            "tol": float(a.tol), "itr": int(a.itr), "pcgitr": int(a.pcgitr),
            "precond": a.precond, "preconditioner": _precond_name(a.precond, a.pcgitr),
            "verb": int(a.verb), "full_out": int(a.full_out),
            "constraints": a.constraints_path, "out_evecs": a.out_evecs_path}


def _rows(report):
    out = []
    for h in report.history:
        if h.ritz is None:
            continue
        out.extend({"iter": int(h.iteration), "j": j, "ritz": float(h.ritz[j]),
                    "resid": float(h.residual_norms[j]), "active": bool(h.active[j])}
                   for j in range(h.ritz.size))
    return out


def _write_csv(path, report):
    lines = ["iter,j,ritz,resid,active"]
    lines += [f"{r['iter']},{r['j']},{r['ritz']!r},{r['resid']!r},{int(r['active'])}"
              for r in _rows(report)]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def _write_json(path, record):
    with open(path, "w") as fh:
        json.dump(record, fh, indent=2)
        fh.write("\n")


def _table(a, report, analytic, t_setup, t_solve):
    desc = _precond_name(a.precond, a.pcgitr)
    print(f"grid {'x'.join(map(str, a.n))}  m {a.m}  precond {desc}  seed {a.seed}  "
          f"tol {a.tol:g}")
    print(f"{'':>4} {'eigenvalue':>22} {'analytic':>22} {'rel err':>10} conv")
    for j, lam in enumerate(report.eigenvalues):
        conv = "yes" if report.converged[j] else "NO"
        if analytic is None:
            print(f"{j:>4} {lam:>22.15f} {'-':>22} {'-':>10} {conv}")
        else:
            ref = analytic[j]
            print(f"{j:>4} {lam:>22.15f} {ref:>22.15f} {abs(lam - ref) / abs(ref):>10.2e} {conv}")
    print(f"status {report.status}  iterations {report.iterations_used}  "
          f"setup {t_setup:.3f}s  solve {t_solve:.3f}s")


def _gather_rows(env: _Env, x, n):
    """Full (n, k) eigenvector block on rank 0 from the z-slab pieces."""
    if env.world == 1:
        return x
    import torch
    import torch.distributed as dist

    xt = torch.as_tensor(np.ascontiguousarray(x)).cuda()
    counts = torch.tensor([xt.shape[0]], device=xt.device)
    allc = [torch.zeros_like(counts) for _ in range(env.world)]
    dist.all_gather(allc, counts)
    rmax = int(max(int(c) for c in allc))
    pad = torch.zeros((rmax, xt.shape[1]), dtype=xt.dtype, device=xt.device)
    pad[:xt.shape[0]] = xt
    parts = [torch.empty_like(pad) for _ in range(env.world)]
    dist.all_gather(parts, pad)
    full = torch.cat([p[:int(c)] for p, c in zip(parts, allc)]).cpu().numpy()
    assert full.shape[0] == n
    return full


def sweep(kind, a):
    """One solve per value of the swept knob (fixed seed); prints / writes
    the summary table (cli.py:334-407).  Returns the exit code."""
    from .lobpcg import SolverConfig, solve

    if a.sweep_values is not None:
        try:
            values = [int(v) for v in a.sweep_values.split(",") if v.strip()]
        except ValueError:
            print(f"bad -sweep_values: {a.sweep_values!r}", file=sys.stderr)
            return EXIT_ERROR
    else:
        values = list(SWEEP_DEFAULTS[kind])
    if not values:
        print("empty sweep range", file=sys.stderr)
        return EXIT_ERROR
    if kind == "block_size" and min(values) < 1:
        print("block sizes must be positive", file=sys.stderr)
        return EXIT_ERROR
    if kind == "inner_iter" and min(values) < 0:
        print("inner iteration counts must be nonnegative", file=sys.stderr)
        return EXIT_ERROR
    env = _setup(a)
    op, _, _ = _operator(a, env)
    key = "pcgitr" if kind == "inner_iter" else "block_size"
    table = []
    for v in values:
        m, steps = (a.m, v) if kind == "inner_iter" else (v, a.pcgitr)
        cfg = SolverConfig(block_size=m, tol=a.tol, max_iter=a.itr, seed=a.seed, verbosity=0,
                           lock_history=False)
        t0 = time.perf_counter()
        rep = solve(op, t=_precond(op, a.precond, steps), config=cfg)
        table.append({key: v, "iterations": int(rep.iterations_used),
                      "solve_sec": float(time.perf_counter() - t0), "status": rep.status})
    if env.lead:
        if a.verb >= 1:
            print(f"{key:>10} {'iterations':>10} {'solve_sec':>10}  status")
            for r in table:
                print(f"{r[key]:>10} {r['iterations']:>10} {r['solve_sec']:>10.3f}  {r['status']}")
        if a.csv_path:
            with open(a.csv_path, "w") as fh:
                fh.write(f"{key},iterations,solve_sec\n")
                fh.writelines(f"{r[key]},{r['iterations']},{r['solve_sec']!r}\n" for r in table)
        if a.json_path:
            _write_json(a.json_path, {"sweep": kind, "config": _echo(a), "rows": table})
    return EXIT_ERROR if any(r["status"].startswith("Failed") for r in table) else EXIT_OK


def _single(a):
    from .lobpcg import Constraints, SolverConfig, solve
    from .problems import exact_eigenvalues

    t0 = time.perf_counter()
    env = _setup(a)
    op, grid, scale = _operator(a, env)
    t = _precond(op, a.precond, a.pcgitr)
    cons = None
    if a.constraints_path:
        basis = load_eigenvectors(a.constraints_path)
        if basis.shape[0] != grid.n:
            raise ValueError(f"constraint vectors have dimension {basis.shape[0]}, "
                             f"but the grid has {grid.n} points")
        cons = Constraints.from_basis(basis)
    cfg = SolverConfig(block_size=a.m, tol=a.tol, max_iter=a.itr, seed=a.seed,
                       verbosity=a.verb if a.verb >= 2 else 0)
    t_setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    rep = solve(op, t=t, y=cons, config=cfg)
    t_solve = time.perf_counter() - t1

    skip = cons.count if cons is not None else 0
    analytic = None
    if skip + a.m <= grid.n:
        analytic = exact_eigenvalues(grid, skip + a.m, scale=scale)[skip:]
    vecs = _gather_rows(env, rep.eigenvectors, grid.n) if a.out_evecs_path else None
    if env.lead:
        if a.verb >= 1:
            _table(a, rep, analytic, t_setup, t_solve)
        if a.json_path:
            rel = (None if analytic is None else
                   [float(abs(x - y) / abs(y)) for x, y in zip(rep.eigenvalues, analytic)])
            _write_json(a.json_path, {
                "config": _echo(a),
                "eigenvalues": [float(v) for v in rep.eigenvalues],
                "analytic": None if analytic is None else [float(v) for v in analytic],
                "rel_errors": rel,
                "iterations": int(rep.iterations_used),
                "history": _rows(rep) if a.full_out else [],
                "setup_sec": float(t_setup),
                "solve_sec": float(t_solve),
                "status": rep.status,
            })
        if a.csv_path:
            _write_csv(a.csv_path, rep)
        if a.out_evecs_path:
            save_eigenvectors(a.out_evecs_path, vecs)
    return rep


def main(argv=None):
    parser = build_parser()
    try:
        a = parser.parse_args(argv)
        _check(parser, a)
    except SystemExit as exc:
        return exc.code if exc.code is not None else EXIT_ERROR
    from .small import NotSPD

    try:
        if a.sweep:
            return sweep(a.sweep, a)
        rep = _single(a)
    except (ValueError, OSError, NotSPD) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
    if not rep.ok:
        print(f"error: solver reported {rep.status}", file=sys.stderr)
        return EXIT_ERROR
    return EXIT_OK if rep.all_converged else EXIT_PARTIAL


if __name__ == "__main__":
    sys.exit(main())
