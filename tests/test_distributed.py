"""z-slab decomposition exercised on CPU: world_size 2 over gloo,
with the native kernels replaced by their CPU stand-ins (tests/emulation.py).

Checks the host-side multi-GPU logic the B200 path uses unchanged with NCCL:
the slab partition, the bit-identical slab initial block, the one-plane halo
exchange feeding the stencil, and the sum all-reduce of every small
reduction -- a 2-rank solve must reproduce the single-process solve.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _MP:
    def setattr(self, obj, name, value):
        setattr(obj, name, value)


def _solve(grid, m, scale, max_iter, tol):
    import paper_0705_2626_b200 as pk
    from paper_0705_2626_b200.distributed import SlabLaplacian3D

    a = SlabLaplacian3D(grid, scale=scale)
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=tol, max_iter=max_iter, seed=3))
    return a, rep


def _worker(rank, world, port, grid, m, scale, max_iter, tol, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tests.emulation import emulate

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        with emulate(_MP()):
            a, rep = _solve(grid, m, scale, max_iter, tol)
            q.put((rank, a.part.z0, a.part.z1, rep.eigenvalues, rep.iterations_used,
                   rep.status, rep.eigenvectors, np.array(rep.lock_iterations)))
    finally:
        dist.destroy_process_group()


def test_slab_partition_covers_grid():
    from paper_0705_2626_b200.distributed import SlabPartition

    for nz, world in [(128, 8), (464, 8), (10, 3), (7, 7)]:
        parts = [SlabPartition(nz, world, r) for r in range(world)]
        assert parts[0].z0 == 0 and parts[-1].z1 == nz
        for p, q in zip(parts, parts[1:]):
            assert p.z1 == q.z0 and p.planes >= 1


def test_slab_initial_block_is_bitwise_slice():
    from paper_0705_2626_b200.distributed import SlabPartition, slab_initial_block
    from paper_0705_2626_b200.operators import Grid3D

    g = Grid3D(6, 5, 9)
    m = 3
    full = np.random.Generator(np.random.PCG64(11)).uniform(-1.0, 1.0, size=(g.n, m))
    for r in range(3):
        p = SlabPartition(g.nz, 3, r)
        blk = slab_initial_block(g, p, m, 11)
        assert np.array_equal(blk, full[p.z0 * 30:p.z1 * 30])


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_slab_solve_matches_single_process(monkeypatch, world):
    """world 3 and 4 give interior ranks (both neighbours): halo from below
    and above into the same ghost buffer."""
    from tests.emulation import emulate

    grid, m, scale, max_iter, tol = (10, 9, 12), 4, 169.0, 80, 1e-8
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, m, scale, max_iter, tol, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process reference (world 1, same emulated kernels)
    with emulate(monkeypatch):
        import paper_0705_2626_b200 as pk

        a = pk.Laplacian3D(grid, scale=scale)
        ref = pk.solve(a, t=pk.jacobi_preconditioner(a),
                       config=pk.SolverConfig(block_size=m, tol=tol, max_iter=max_iter, seed=3))
    bounds = [(r[1], r[2]) for r in res]
    assert bounds == [((k * 12) // world, ((k + 1) * 12) // world) for k in range(world)]
    r0 = res[0]
    for r in res[1:]:   # every rank took identical decisions on identical bits
        assert np.array_equal(r[3], r0[3]) and r[4] == r0[4] and r[5] == r0[5]
        assert np.array_equal(r[7], r0[7])
    assert r0[5] == ref.status
    assert abs(r0[4] - ref.iterations_used) <= 1
    np.testing.assert_allclose(r0[3], ref.eigenvalues, rtol=1e-10)
    # the slabs stacked are the global Ritz block (up to column signs)
    x = np.vstack([r[6] for r in res])
    for j in range(m):
        c = abs(float(x[:, j] @ ref.eigenvectors[:, j]))
        assert c == pytest.approx(1.0, abs=1e-6)
