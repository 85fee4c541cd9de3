"""z-slab path on one GPU.  gpurun gives one GPU, so the
multi-rank exchange itself is covered by the gloo tests
(tests/test_distributed.py, worlds 2-4); here:

  * the interior + edge launches of the overlapped stencil pass
    (b2l_stencil7_gram_split, the compute half of b2l_slab_stencil7_gram)
    for every rank of a virtual 2/3/4/5-way split, with each rank's halo taken
    from its neighbours' rows: A W bitwise equal to the global stencil, the
    per-rank Grams summing to the global Gram;
  * the library's NCCL communicator on one rank (b2l_slab_create with an
    NCCL id, world 1) driving the native steady-state iteration with its
    all-reduces: the trajectory equals the plain single-GPU solve bit for bit.
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_0705_2626_b200 import _lib

    return _lib.load()


def _blk(n, ld, k, gen):
    t = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    t[:, :k] = torch.from_numpy(gen.uniform(-1, 1, (n, k))).cuda()
    return t


@pytest.mark.parametrize("dims,ld,m,kw,world", [
    ((40, 36, 30), 10, 10, 10, 2), ((40, 36, 30), 10, 10, 9, 3), ((33, 17, 23), 16, 16, 13, 4),
    ((24, 20, 10), 8, 8, 8, 5), ((24, 20, 7), 2, 0, 1, 3)])
def test_split_stencil_gram_matches_global(lib, dims, ld, m, kw, world):
    from paper_0705_2626_b200 import device as dv
    from paper_0705_2626_b200.distributed import SlabPartition

    nx, ny, nz = dims
    plane = nx * ny
    gen = np.random.Generator(np.random.PCG64(sum(dims) + world))
    W = _blk(nx * ny * nz, ld, kw, gen)
    X = _blk(nx * ny * nz, max(ld, 2), max(m, 1), gen)
    AW = torch.empty_like(W)
    G = torch.empty((m + kw, kw), dtype=torch.float64, device="cuda")
    s = 17.0
    dv.stencil7_gram(W, AW, nx, ny, nz, s, X if m else None, m, kw, G)
    Gsum = torch.zeros_like(G)
    st = dv.stream_ptr()
    for r in range(world):
        p = SlabPartition(nz, world, r)
        r0, r1 = p.z0 * plane, p.z1 * plane
        w = W[r0:r1].clone()
        x = X[r0:r1].clone()
        out = torch.full_like(w, float("nan"))
        halo = torch.zeros((2 * plane, ld), dtype=torch.float64, device="cuda")
        lo, hi = r > 0, r < world - 1
        if lo:
            halo[:plane] = W[r0 - plane:r0]
        if hi:
            halo[plane:] = W[r1:r1 + plane]
        g = torch.empty_like(G)
        rc = lib.b2l_stencil7_gram_split(w.data_ptr(), out.data_ptr(), nx, ny, p.planes, ld,
                                         halo.data_ptr(), int(lo), int(hi), s,
                                         x.data_ptr() if m else None, x.stride(0), m, kw,
                                         g.data_ptr(), st)
        assert rc == 0, lib.b2l_last_error()
        torch.cuda.synchronize()
        assert torch.equal(out[:, :kw], AW[r0:r1, :kw]), r
        Gsum += g
    ref = G.cpu().numpy()
    scale = np.abs(ref).max()
    np.testing.assert_allclose(Gsum.cpu().numpy(), ref, rtol=0, atol=1e-13 * scale)


def test_slab_apply_matches_stencil(lib):
    """b2l_slab_stencil7 on a world-1 context (no neighbours) is K1."""
    import paper_0705_2626_b200 as pk
    from paper_0705_2626_b200.distributed import SlabLaplacian3D

    N = 20
    s = float((N + 1) ** 2)
    a = SlabLaplacian3D((N, N, N), scale=s, comm="nccl")
    assert a.native_slab is not None
    x = np.random.Generator(np.random.PCG64(3)).uniform(-1, 1, (N ** 3, 5))
    np.testing.assert_array_equal(a(x), pk.Laplacian3D((N, N, N), scale=s)(x))


def test_native_slab_iteration_world1_bitwise(lib):
    """The z-slab native step (NCCL all-reduces on the communication stream,
    red_on_host = 3) on one rank reproduces the single-GPU run bit for bit."""
    import paper_0705_2626_b200 as pk
    from paper_0705_2626_b200.distributed import SlabLaplacian3D

    N, m = 40, 10
    s = float((N + 1) ** 2)
    cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=60, seed=0)
    a1 = pk.Laplacian3D((N, N, N), scale=s)
    ref = pk.solve(a1, t=pk.jacobi_preconditioner(a1), config=cfg)
    a = SlabLaplacian3D((N, N, N), scale=s, comm="nccl")
    run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a), config=cfg)
    assert run._native is not None and run._native.slab
    states = set()
    while run.step():
        states.add(int(run._native.red_on_host))
    rep = run.report()
    assert 3 in states
    assert rep.status == ref.status and rep.iterations_used == ref.iterations_used
    assert np.array_equal(np.array([h.ritz for h in rep.history]),
                          np.array([h.ritz for h in ref.history]))
    assert np.array_equal(rep.eigenvalues, ref.eigenvalues)


def test_slab_allreduce_world1(lib):
    from paper_0705_2626_b200.distributed import SlabLaplacian3D

    a = SlabLaplacian3D((8, 8, 8), comm="nccl")
    t = torch.arange(37, dtype=torch.float64, device="cuda")
    a.allreduce_(t)
    torch.cuda.synchronize()
    assert torch.equal(t, torch.arange(37, dtype=torch.float64, device="cuda"))
    w, r, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert lib.b2l_slab_info(a.native_slab, ctypes.byref(w), ctypes.byref(r), ctypes.byref(c)) == 0
    assert (w.value, r.value, c.value) == (1, 0, 1)
