"""C1@1000 over 2K operator perturbations (scale (N+1)^2 (1 + k 2^-52),
k = +-1..K; K = 16 by default, 64 for the c1_band128 fixture) on the native
loop: the converged fraction, how often the second column locks by iteration
215, the iteration counts -- compared with the reference's own distribution
(make_golden.py --c1-band32 / --c1-band128).  Diagnostic only.
    python tools/c1_band32.py [K] [out.json]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N = 32
base = float((N + 1) ** 2)
out = []
for k in list(range(-K, 0)) + list(range(1, K + 1)):
    a = pk.Laplacian3D((N, N, N), scale=base * (1.0 + k * 2.0 ** -52))
    rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=1000, seed=0))
    out.append((k, int(rep.iterations_used), rep.status, [int(x) for x in rep.lock_iterations]))
conv = sum(1 for o in out if o[2] == "Converged")
early = sum(1 for o in out if sorted(o[3])[1] <= 215)
its = sorted(o[1] for o in out)
print(json.dumps({"converged": conv, "second_lock_le_215": early, "median_it": its[len(its) // 2],
                  "q25_it": its[len(its) // 4], "q75_it": its[3 * len(its) // 4],
                  "runs": len(out)}))
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(json.dumps(out))
