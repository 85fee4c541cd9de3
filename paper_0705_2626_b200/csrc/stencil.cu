// K1: fused block 7-point Laplacian, z-streaming with TMA (sm_100a).
//
// Replaces Laplacian3D._apply (reference operators.py:184-196) and the harness
// scaling s*L(x) (operators.py:104-121).  Blocks are point-major (n, ld) fp64,
// point p = i + nx*(j + ny*k) (operators.py:63-67), so one grid point's k
// columns are ld contiguous doubles.
//
// Each CTA owns a TX x TY column of the xy-plane and a chunk of z-planes.  It
// streams input planes (with a one-point xy halo) through an NST-deep ring of
// shared-memory stages filled by 4-D TMA tile loads; the TMA zero-fills
// out-of-range x/y/z coordinates, which IS the homogeneous Dirichlet boundary.
// The z-1 and z centre values live in registers, so each output element reads
// 5 values from shared memory.  Output planes are written back by TMA stores
// from a double-buffered staging tile.
//
// Arithmetic order is exactly the reference's: ((((((6c - x-) - x+) - y-) -
// y+) - z-) - z+) then * scale, with explicit _rn intrinsics (no FMA
// contraction), so the result is bitwise equal to the numpy reference.
#include "stencil.cuh"

namespace b2l {


template <int EPT, int NST>
__global__ void __launch_bounds__(256)
    stencil7_kernel(const __grid_constant__ CUtensorMap tin,
                    const __grid_constant__ CUtensorMap thalo,
                    const __grid_constant__ CUtensorMap tout, StencilGeom g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw;
  auto stage = [&](int s) -> double* {
    return reinterpret_cast<double*>(base + s * g.stage_stride);
  };
  double* outbuf0 = reinterpret_cast<double*>(base + NST * g.stage_stride);
  double* outbuf1 =
      reinterpret_cast<double*>(base + NST * g.stage_stride + g.out_stride);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + NST * g.stage_stride +
                                              2 * g.out_stride);

  const int tid = threadIdx.x;
  const int tx0 = (blockIdx.x % g.tiles_x) * g.TX;
  const int ty0 = (blockIdx.x / g.tiles_x) * g.TY;
  int z0, z1;
  stencil_zrange(g, z0, z1);
  if (z0 >= z1) return;
  const int nplanes = (z1 - z0) + 2;  // planes z0-1 .. z1

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int q) {
    const int z = z0 - 1 + q;
    const int s = q % NST;
    mbar_expect_tx(&bar[s], g.stage_bytes);
    if (z < 0 && g.has_lo)
      tma_load_4d(stage(s), &thalo, &bar[s], 0, tx0 - 1, ty0 - 1, 0);
    else if (z >= g.nz && g.has_hi)
      tma_load_4d(stage(s), &thalo, &bar[s], 0, tx0 - 1, ty0 - 1, 1);
    else
      tma_load_4d(stage(s), &tin, &bar[s], 0, tx0 - 1, ty0 - 1, z);
  };

  if (tid == 0) {
    for (int q = 0; q < NST && q < nplanes; ++q) issue(q);
  }

  // Per-thread element bookkeeping: flat interior index e -> staged offset.
  const int rowlen = g.TX * g.ld;           // interior doubles per tile row
  const int ystride = (g.TX + 2) * g.ld;    // staged doubles per tile row
  int off[EPT];
  bool valid[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = tid + 256 * i;
    valid[i] = e < g.nelem;
    const int ty = valid[i] ? e / rowlen : 0;
    const int rem = valid[i] ? e - ty * rowlen : 0;
    off[i] = (ty + 1) * ystride + g.ld + rem;
  }

  double prev[EPT], cur[EPT];
  mbar_wait(&bar[0], 0);
#pragma unroll
  for (int i = 0; i < EPT; ++i) prev[i] = valid[i] ? stage(0)[off[i]] : 0.0;
  mbar_wait(&bar[1 % NST], (1 / NST) & 1);
#pragma unroll
  for (int i = 0; i < EPT; ++i) cur[i] = valid[i] ? stage(1 % NST)[off[i]] : 0.0;
  __syncthreads();
  if (tid == 0 && NST < nplanes) issue(NST);

  const double six = 6.0;
  const double sc = g.scale;
  for (int z = z0; z < z1; ++z) {
    const int q = z - z0 + 1;  // plane index of z
    const int sn = (q + 1) % NST;
    mbar_wait(&bar[sn], ((q + 1) / NST) & 1);
    const double* P = stage(q % NST);
    const double* N = stage(sn);
    double* O = (z & 1) ? outbuf1 : outbuf0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (valid[i]) {
        const int o = off[i];
        const double nx_ = N[o];
        double r = __dmul_rn(six, cur[i]);
        r = __dsub_rn(r, P[o - g.ld]);
        r = __dsub_rn(r, P[o + g.ld]);
        r = __dsub_rn(r, P[o - ystride]);
        r = __dsub_rn(r, P[o + ystride]);
        r = __dsub_rn(r, prev[i]);
        r = __dsub_rn(r, nx_);
        O[tid + 256 * i] = __dmul_rn(sc, r);
        prev[i] = cur[i];
        cur[i] = nx_;
      }
    }
    __syncthreads();
    if (tid == 0) {
      fence_async_smem();
      tma_store_4d(&tout, O, 0, tx0, ty0, z);
      bulk_commit();
      bulk_wait_read<1>();
      if (q + NST < nplanes) issue(q + NST);
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait<0>();
}

// ------------------------------------------------------------------ host

// z-chunk length for `tiles` xy tiles on `slots` resident CTAs.  A CTA pays a
// pipeline fill (two halo planes + the ring latency) per chunk, which
// measured costlier than a partly idle wave (C2, 128 tiles on 296 slots:
// chunks of 64 planes 138 us, 26 planes 148 us, 8 planes 161 us,
// tools/sweep_sgram.py), so: the longest chunks that still give every
// resident slot at most one CTA (one wave), chunks of >= 4 planes.
// More tiles than slots: enough z-chunks for about four waves (the last,
// partial wave then costs little), chunks of >= 64 planes (measured: C3
// 1024 tiles, 2 chunks of 128 planes 1.40 ms vs 1.54 ms unsplit; W1 464
// tiles, 3 chunks 0.44 ms vs 0.50 ms; C4 1740 tiles unsplit, flat).
int choose_zchunk(int tiles, int nz, int slots) {
  int zs;
  if (tiles >= slots) {
    zs = (4 * slots + tiles - 1) / tiles;
    const int cap = nz / 64 < 1 ? 1 : nz / 64;
    if (zs > cap) zs = cap;
  } else {
    zs = slots / tiles;
  }
  if (zs < 1) zs = 1;
  int c = (nz + zs - 1) / zs;
  if (c < 4) c = nz < 4 ? nz : 4;
  return c;
}

bool apply_zmode(StencilGeom& g, dim3& grid, int tiles, int mode, int slots) {
  g.zedge = 0;
  g.zbeg = 0;
  g.zend = g.nz;
  if (mode == Z_EDGE) {
    g.zedge = 1;
    g.zchunk = 1;
    grid = dim3(tiles, g.nz > 1 ? 2 : 1, 1);
    return true;
  }
  if (mode == Z_INTERIOR) {
    g.zbeg = 1;
    g.zend = g.nz - 1;
  }
  const int span = g.zend - g.zbeg;
  if (span <= 0) return false;
  g.zchunk = choose_zchunk(tiles, span, slots);
  grid = dim3(tiles, (span + g.zchunk - 1) / g.zchunk, 1);
  return true;
}

int plan_stencil(int nx, int ny, int nz, int ld, StencilPlan* p) {
  StencilGeom& g = p->g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.ld = ld;
  p->ept = (ld > 64) ? 16 : 8;
  const int maxe = 256 * p->ept;
  int TX = nx < 32 ? nx : 32;
  while (TX > 1 && TX * ld > maxe) TX = (TX + 1) / 2;
  int TY = maxe / (TX * ld);
  if (TY < 1) TY = 1;
  if (TY > ny) TY = ny;
  if (TY > 254) TY = 254;
  g.TX = TX;
  g.TY = TY;
  g.nelem = TX * TY * ld;
  g.tiles_x = (nx + TX - 1) / TX;
  const int tiles_y = (ny + TY - 1) / TY;
  const int tiles = g.tiles_x * tiles_y;
  g.stage_bytes = (uint32_t)((TX + 2) * (TY + 2) * ld * 8);
  g.stage_stride = (g.stage_bytes + 127u) & ~127u;
  g.out_stride = ((uint32_t)(TX * TY * ld * 8) + 127u) & ~127u;
  // Deepest ring that still lets two CTAs share an SM.
  p->nst = 4;
  size_t smem = (size_t)4 * g.stage_stride + 2 * g.out_stride + 64;
  if (smem > 113 * 1024) {
    p->nst = 3;
    smem = (size_t)3 * g.stage_stride + 2 * g.out_stride + 64;
  }
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL,
            "stencil tile does not fit in shared memory (ld too large)");
  p->smem = smem;
  apply_zmode(g, p->grid, tiles, Z_ALL, 2 * sm_count());
  return 0;
}

template <int EPT, int NST>
static int launch_stencil_t(const StencilPlan& p, const CUtensorMap& tin,
                            const CUtensorMap& thalo, const CUtensorMap& tout,
                            cudaStream_t st) {
  auto kern = stencil7_kernel<EPT, NST>;
  if (int rc = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem, 256, nullptr))
    return rc;
  kern<<<p.grid, 256, p.smem, st>>>(tin, thalo, tout, p.g);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}

int stencil7(const double* in, double* out, int nx, int ny, int nz, int ld,
             const double* halo, int has_lo, int has_hi, double scale,
             cudaStream_t st, int zmode) {
  B2L_CHECK(nx > 0 && ny > 0 && nz > 0, -B2L_EINVAL, "stencil: empty grid");
  B2L_CHECK(ld >= 2 && (ld % 2) == 0, -B2L_EINVAL,
            "stencil: ld must be even (16-B rows for TMA)");
  B2L_CHECK((reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(out) & 15) == 0,
            -B2L_EINVAL, "stencil: blocks must be 16-B aligned");
  B2L_CHECK(in != out, -B2L_EINVAL, "stencil: in-place apply not supported");
  B2L_CHECK(!(has_lo || has_hi) || halo != nullptr, -B2L_EINVAL,
            "stencil: halo flags set without a halo buffer");
  StencilPlan p;
  int rc = plan_stencil(nx, ny, nz, ld, &p);
  if (rc) return rc;
  p.g.has_lo = has_lo;
  p.g.has_hi = has_hi;
  p.g.scale = scale;
  if (zmode != Z_ALL) {
    const int tiles = p.grid.x;
    if (!apply_zmode(p.g, p.grid, tiles, zmode, 2 * sm_count())) return 0;
  }
  CUtensorMap tin, thalo, tout;
  const uint32_t TX = p.g.TX, TY = p.g.TY;
  rc = encode_tmap_4d(&tin, in, ld, nx, ny, nz, ld, TX + 2, TY + 2, 1);
  if (rc) return rc;
  rc = encode_tmap_4d(&tout, out, ld, nx, ny, nz, ld, TX, TY, 1);
  if (rc) return rc;
  if (halo) {
    rc = encode_tmap_4d(&thalo, halo, ld, nx, ny, 2, ld, TX + 2, TY + 2, 1);
    if (rc) return rc;
  } else {
    thalo = tin;
  }
  if (p.ept == 8 && p.nst == 4) return launch_stencil_t<8, 4>(p, tin, thalo, tout, st);
  if (p.ept == 8 && p.nst == 3) return launch_stencil_t<8, 3>(p, tin, thalo, tout, st);
  if (p.ept == 16 && p.nst == 4) return launch_stencil_t<16, 4>(p, tin, thalo, tout, st);
  return launch_stencil_t<16, 3>(p, tin, thalo, tout, st);
}

}  // namespace b2l
