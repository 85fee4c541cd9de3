"""Constrained solves with random dense constraints: `python tools/cons_check.py ours`
on the GPU, `... ref` in the build container (imports the reference from
/root/reference): both end BasisFallback / MaxIterReached.  Diagnostic."""
import sys, numpy as np
which = sys.argv[1]
if which == "ref":
    sys.path.insert(0, "/root/reference/pkg/src")
    import blockeig as pk
else:
    sys.path.insert(0, "/root/repo")
    import paper_0705_2626_b200 as pk
for dims, m, nc, seed in [((8, 9, 10), 4, 3, 7), ((6, 7, 5), 2, 5, 1), ((12, 10, 9), 6, 2, 3), ((10, 10, 10), 3, 1, 9)]:
    n = int(np.prod(dims))
    a = pk.laplacian3d(dims)
    y = np.random.default_rng(100 + seed).standard_normal((n, nc))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a), y=pk.Constraints.from_basis(y),
                   config=pk.SolverConfig(block_size=m, tol=1e-6, max_iter=800, seed=seed))
    print(dims, m, nc, seed, rep.status, rep.iterations_used, np.round(rep.eigenvalues[:3], 8))
