"""Phase breakdown of one public solve() at C2 (setup, iterations, report).

Diagnostic only (not part of the product): run on the GPU box with
`python tools/profile_solve.py`."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200 import lobpcg as lb  # noqa: E402

N, M = 128, 10
s = float((N + 1) ** 2)
A = pk.Laplacian3D((N,) * 3, scale=s)
T = pk.jacobi_preconditioner(A)
cfg = pk.SolverConfig(block_size=M, tol=1e-8, max_iter=300, seed=0)
x0 = np.random.Generator(np.random.PCG64(0)).uniform(-1.0, 1.0, size=(N ** 3, M))


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


orig_init, orig_initial, orig_native = lb.LOBPCGRun.__init__, lb.LOBPCGRun._initial, lb.LOBPCGRun._native_setup
marks = {}


def initial(self):
    marks["alloc+upload"] = tick()
    orig_initial(self)
    marks["initial"] = tick()


lb.LOBPCGRun._initial = initial
for rep in range(3):
    marks.clear()
    t0 = tick()
    run = lb.LOBPCGRun(A, t=T, x0=x0, config=cfg)
    t1 = tick()
    n_it = 0
    first = None
    while run.step():
        n_it += 1
        if first is None:
            first = tick()
    t2 = tick()
    r = run.report()
    t3 = tick()
    print(f"rep {rep}: ctor {1e3*(t1-t0):.1f} ms (alloc+upload {1e3*(marks['alloc+upload']-t0):.1f}, "
          f"initial {1e3*(marks['initial']-marks['alloc+upload']):.1f}, native setup "
          f"{1e3*(t1-marks['initial']):.1f}); first step {1e3*(first-t1):.2f} ms; loop {1e3*(t2-t1):.1f} ms "
          f"for {n_it} steps ({1e3*(t2-first)/(n_it-1):.3f} ms/step after the first); report {1e3*(t3-t2):.1f} ms; "
          f"total {1e3*(t3-t0):.1f} ms, {r.iterations_used} it, {r.status}")
    del run, r
    # pinned x0 variant
xp = torch.from_numpy(x0).pin_memory()
t0 = tick()
r = pk.solve(A, t=T, x0=xp, config=cfg)
t1 = tick()
print(f"pinned x0 tensor: total {1e3*(t1-t0):.1f} ms")
t0 = tick(); xd = torch.from_numpy(x0).cuda(); t1 = tick()
print(f"plain H2D of x0 (pageable): {1e3*(t1-t0):.1f} ms; pinned H2D:", end=" ")
t0 = tick(); xd = xp.cuda(non_blocking=True); t1 = tick()
print(f"{1e3*(t1-t0):.1f} ms")
t0 = tick(); h = xd.cpu(); t1 = tick()
print(f"D2H pageable: {1e3*(t1-t0):.1f} ms")

# host-side phases of the native steady-state iteration (B2L_ITER_PROFILE=1)
import ctypes  # noqa: E402
from paper_0705_2626_b200 import _lib  # noqa: E402

lib = _lib.load()
buf = (ctypes.c_double * 8)()
lib.b2l_iter_profile(buf, 1)
run = lb.LOBPCGRun(A, t=T, x0=x0, config=cfg)
t0 = tick()
while run.step():
    pass
t1 = tick()
on = lib.b2l_iter_profile(buf, 0)
c = max(buf[0], 1)
print(f"profile on={on}: {int(buf[0])} native steps, {1e3*(t1-t0)/run.it:.3f} ms/step; per step us: "
      f"fetch-enqueue {buf[1]/c:.1f}, sync-wait {buf[2]/c:.1f}, drift+lock {buf[3]/c:.1f}, "
      f"RR first half {buf[6]/c:.1f}, wait G2 {buf[7]/c:.1f}, RR second half {buf[4]/c:.1f}, "
      f"uploads+launches {buf[5]/c:.1f}")
