"""Host/device race probe: the C2 run stepped with an optional device-side
sleep queued before every step (the host then runs far ahead of the GPU), and
with the native fast path on/off.  Prints the Ritz-history hash per variant;
all must agree.  Diagnostic only."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0705_2626_b200 as pk  # noqa: E402
from paper_0705_2626_b200 import lobpcg as lb  # noqa: E402

N, m, its = 128, 10, int(sys.argv[1]) if len(sys.argv) > 1 else 40
s = float((N + 1) ** 2)
a = pk.Laplacian3D((N, N, N), scale=s)
T = pk.jacobi_preconditioner(a)
cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=its, seed=0)


def run(sleep, native=True, sleep_inside=False, sync_each=False, sync_at=()):
    r = lb.LOBPCGRun(a, t=T, config=cfg)
    if -1 in sync_at:
        torch.cuda.synchronize()
    if sync_at:
        orig_step0 = r.step
        cnt = [0]

        def stepped_at():
            out = orig_step0()
            if cnt[0] in sync_at:
                torch.cuda.synchronize()
            cnt[0] += 1
            return out
        r.step = stepped_at
    if sync_each:
        orig_step = r.step

        def stepped():
            out = orig_step()
            torch.cuda.synchronize()
            return out
        r.step = stepped
    if not native:
        r._native = None
    if sleep_inside:
        orig = r._native_step

        def wrapped():
            torch.cuda._sleep(sleep)
            return orig()
        r._native_step = wrapped
    while True:
        if sleep and not sleep_inside:
            torch.cuda._sleep(sleep)
        if not r.step():
            break
    h = np.array([e.ritz for e in r.history])
    return hashlib.sha1(h.tobytes()).hexdigest()[:12], h


VARIANTS = {"plain": dict(sleep=0), "sync-each-step": dict(sleep=0, sync_each=True),
            "sync-ctor": dict(sleep=0, sync_at=(-1,)), "sync-s0": dict(sleep=0, sync_at=(0,)),
            "sync-s1": dict(sleep=0, sync_at=(1,)), "sync-s0s1": dict(sleep=0, sync_at=(0, 1))}
order = sys.argv[2].split(",") if len(sys.argv) > 2 else None
base = None
if order:
    for name in order:
        hsh, h = run(**VARIANTS[name])
        if base is None:
            base = h
        d = np.flatnonzero(np.any(h != base, axis=1))
        print(f"{name:20s} {hsh} first diff vs first: {d[0] if d.size else None}", flush=True)
    sys.exit(0)
for name, kw in [("plain", dict(sleep=0)), ("plain2", dict(sleep=0)),
                 ("sleep-before-step", dict(sleep=2_000_000)),
                 ("sleep-in-native", dict(sleep=2_000_000, sleep_inside=True)),
                 ("python-path", dict(sleep=0, native=False)),
                 ("python-path-sleep", dict(sleep=2_000_000, native=False))]:
    hsh, h = run(**kw)
    if base is None:
        base = h
    d = np.flatnonzero(np.any(h != base, axis=1))
    print(f"{name:20s} {hsh} first diff vs plain: {d[0] if d.size else None}", flush=True)
