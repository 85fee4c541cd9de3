"""z-slab domain decomposition of the 7-point Laplacian over GPUs.

One process per GPU (torch.distributed, NCCL over NVLink on B200; gloo on CPU
for tests).  Rank r owns the z-planes [floor(r N/P), floor((r+1) N/P)): a
contiguous row range of every point-major (n, ld) block, because z varies
slowest (reference operators.py:63-67).  Per iteration the path needs exactly
two kinds of exchange:

  * a one-plane halo of W before each stencil apply (send the first owned
    plane down, the last one up; receive the neighbours' planes into the
    (2 * nx * ny, ld) ghost buffer the stencil kernel reads);
  * a sum all-reduce of every small reduction the host consumes (Gram
    blocks, residual norms), so each rank solves the same small problem on
    identical bits and no broadcast of coefficients is needed.

Row-local work (update, residual, preconditioner, diagonal B) needs no
communication.  The reference is single-process; the paper ran
the same decomposition through MPI inside hypre.

On CUDA both exchanges run inside libb200lobpcg (b2l_slab_*, csrc/slab.cu):
an NCCL communicator of its own (its id broadcast over torch.distributed),
the halo posted on a communication stream under the interior stencil planes,
and the steady-state iteration (b2l_fast_iteration) with both all-reduces
inside it.  On CPU tensors (the gloo tests) the same exchanges go through
torch.distributed point-to-point and all_reduce.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .operators import Grid3D, Laplacian3D

__all__ = ["SlabPartition", "SlabLaplacian3D", "slab_initial_block"]


@dataclass(frozen=True)
class SlabPartition:
    """Planes [z0, z1) of an nz-plane grid owned by `rank` of `world`."""

    nz: int
    world: int
    rank: int

    @property
    def z0(self) -> int:
        return (self.rank * self.nz) // self.world

    @property
    def z1(self) -> int:
        return ((self.rank + 1) * self.nz) // self.world

    @property
    def planes(self) -> int:
        return self.z1 - self.z0

    def bounds(self, r: int) -> tuple[int, int]:
        return (r * self.nz) // self.world, ((r + 1) * self.nz) // self.world


def slab_initial_block(grid: Grid3D, part: SlabPartition, m: int, seed: int) -> np.ndarray:
    """This rank's rows of the reference initial block
    Generator(PCG64(seed)).uniform(-1, 1, (n, m)) (multivec.py:220-229),
    bit-identical to the global fill: element (i, j) is draw i*m + j of the
    PCG64 stream, so the slab starts at draw row0*m (advance())."""
    plane = grid.nx * grid.ny
    row0 = part.z0 * plane
    rows = part.planes * plane
    bg = np.random.PCG64(seed)
    if row0:
        bg.advance(row0 * m)
    return np.random.Generator(bg).uniform(-1.0, 1.0, size=(rows, m))


class SlabLaplacian3D(Laplacian3D):
    """The scaled 7-point Laplacian of a global Grid3D, applied to this rank's
    z-slab.  ``dim`` stays the global n (the reference contract);
    ``local_rows`` is the slab's row count.  Blocks passed to it hold the
    slab's rows only."""

    def __init__(self, grid, scale=1.0, group=None, device=None, comm="auto"):
        """comm: "auto" -- the library's NCCL communicator on CUDA devices,
        torch.distributed on CPU tensors; "nccl" / "torch" force one."""
        if not isinstance(grid, Grid3D):
            grid = Grid3D(*grid)
        super().__init__(grid, scale=scale, device=device)
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.part = SlabPartition(grid.nz, world, rank)
        if self.part.planes < 1:
            raise ValueError(f"{world} ranks for {grid.nz} planes: a rank would own none")
        self.local_grid = Grid3D(grid.nx, grid.ny, self.part.planes)
        self.local_rows = self.local_grid.n
        self.plane = grid.nx * grid.ny
        self._halo = {}
        self._slab = None
        if comm not in ("auto", "nccl", "torch"):
            raise ValueError(f"comm must be 'auto', 'nccl' or 'torch', got {comm!r}")
        if comm == "nccl" or (comm == "auto" and self.device.type == "cuda"):
            self._slab = self._create_native(world, rank)

    def _create_native(self, world, rank):
        """b2l_slab_create with an NCCL id made on the group's first rank and
        broadcast over torch.distributed (any backend)."""
        lib = _lib.load()
        _lib.check(lib.b2l_nccl_load(None), "b2l_nccl_load")
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(lib.b2l_nccl_unique_id(uid, 128), "b2l_nccl_unique_id")
        if world > 1:
            box = [uid.raw if rank == 0 else None]
            src = dist.get_global_rank(self.group, 0) if self.group is not None else 0
            dist.broadcast_object_list(box, src=src, group=self.group)
            uid = ctypes.create_string_buffer(box[0], 128)
        handle = ctypes.c_void_p()
        g = self.local_grid
        _lib.check(lib.b2l_slab_create(uid, world, rank, g.nx, g.ny, g.nz, ctypes.byref(handle)),
                   "b2l_slab_create")
        weakref.finalize(self, lib.b2l_slab_destroy, handle.value)
        return handle.value

    @property
    def native_slab(self):
        """The library's z-slab context (b2l_slab*) or None (torch comm)."""
        return self._slab

    # ---------------------------------------------------------- comm hooks
    @property
    def world(self) -> int:
        return self.part.world

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over ranks (no-op on one rank without a communicator)."""
        if self._slab is not None:
            from . import device as dv

            if not t.is_contiguous():
                raise ValueError("allreduce_ needs a contiguous tensor")
            _lib.check(_lib.load().b2l_slab_allreduce(self._slab, t.data_ptr(), t.numel(),
                                                      dv.stream_ptr(t.device)),
                       "b2l_slab_allreduce")
        elif self.part.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def halo(self, w: torch.Tensor):
        """Exchange the boundary planes of the (local_rows, ld) block w.

        Returns (halo, has_lo, has_hi): halo is a (2*plane, ld) buffer holding
        the plane below the slab (rows [0, plane)) and above it (rows
        [plane, 2*plane)).  Grouped non-blocking send/recv, ordered on the
        current stream by the backend."""
        p = self.part
        has_lo, has_hi = p.rank > 0, p.rank < p.world - 1
        if p.world == 1:
            return None, False, False
        ld = w.stride(0)
        key = (ld, w.device)
        hb = self._halo.get(key)
        if hb is None:
            hb = self._halo[key] = torch.zeros((2 * self.plane, ld), dtype=torch.float64,
                                               device=w.device)
        pl = self.plane
        ops = []
        if has_lo:
            ops.append(dist.P2POp(dist.isend, w[:pl].contiguous(), p.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, hb[:pl], p.rank - 1, self.group))
        if has_hi:
            ops.append(dist.P2POp(dist.isend, w[w.shape[0] - pl:].contiguous(), p.rank + 1,
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, hb[pl:], p.rank + 1, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return hb, has_lo, has_hi

    # ---------------------------------------------------------------- apply
    def apply_into(self, x: torch.Tensor, out: torch.Tensor) -> None:
        from . import device as dv

        if self._slab is not None:
            # halo on the communication stream under the interior planes
            _lib.check(_lib.load().b2l_slab_stencil7(self._slab, x.data_ptr(), out.data_ptr(),
                                                     x.stride(0), self.scale,
                                                     dv.stream_ptr(x.device)),
                       "b2l_slab_stencil7")
            dv.LAUNCHES[0] += 2
            return
        g = self.local_grid
        hb, lo, hi = self.halo(x)
        dv.stencil7(x, out, g.nx, g.ny, g.nz, self.scale, hb, lo, hi)

    def stencil_gram_into(self, x, out, xb, m, kw, gram_out) -> None:
        """out = A x on the slab and gram_out = [xb ; x]^T out (local part)."""
        from . import device as dv

        if self._slab is not None:
            _lib.check(_lib.load().b2l_slab_stencil7_gram(
                self._slab, x.data_ptr(), out.data_ptr(), x.stride(0), self.scale,
                xb.data_ptr() if xb is not None else None, xb.stride(0) if xb is not None else 0,
                int(m), int(kw), gram_out.data_ptr(), dv.stream_ptr(x.device)),
                "b2l_slab_stencil7_gram")
            dv.LAUNCHES[0] += 3
            return
        g = self.local_grid
        hb, lo, hi = self.halo(x)
        dv.stencil7_gram(x, out, g.nx, g.ny, g.nz, self.scale, xb, m, kw, gram_out, hb, lo, hi)

    def _apply(self, x):
        n_l, k = x.shape
        if n_l != self.local_rows:
            raise ValueError(f"slab operator expects {self.local_rows} rows, got {n_l}")
        return super()._apply(x)

    def __call__(self, x):
        # the slab operator works on slab blocks: dim checks use local rows
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(
            np.asarray(x, dtype=np.float64), device=self.device)
        single = t.dim() == 1
        if single:
            t = t[:, None]
        y = self._apply(t.to(self.device, torch.float64))
        y = y[:, 0] if single else y
        return y if isinstance(x, torch.Tensor) else y.detach().cpu().numpy()

    def diagonal(self):
        return torch.full((self.local_rows,), 6.0 * self.scale, dtype=torch.float64,
                          device=self.device)
