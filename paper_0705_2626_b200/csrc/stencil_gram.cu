// K1+K5b: the z-streaming 7-point stencil fused with the Rayleigh-Ritz Gram
// blocks that involve A W (reference lobpcg.py:325 gram(w, aw) and :327
// gram(x, aw)):   AW = s L7 W   and   G = [X ; W]^T AW   ((m + kw) x kw).
//
// Same TMA plane ring as stencil.cu (4-D tile loads with a one-point xy halo,
// OOB zero fill = Dirichlet), plus one TMA box of X per plane.  Work is
// warp-local: a warp owns fixed groups of 8 points of the tile; for each
// plane it computes the stencil for all columns of its points (bitwise the
// reference's operation order) and immediately folds those 8-point rows into
// its own Gram accumulators on the fp64 tensor cores (DMMA) -- no hand-off
// between warps, one CTA barrier per plane (a 4-deep plane ring with double-
// buffered output tiles when two CTAs fit per SM, else 3 + 3; X boxes double
// buffered; the slot a plane writes is released by its TMA store's read
// before that barrier).  A W is never re-read from HBM.
#include <cstdlib>

#include "gram_tile.cuh"
#include "stencil.cuh"

// Shared-memory pitch (doubles per point) of the staged W planes, the A W
// tile and the X tile.  Rows of 16 doubles are 128 bytes: every point of a
// tile then starts on bank 0 and the four points of a Gram k-step meet on the
// same banks (8 wavefronts per fragment load instead of 2 -- two thirds of
// the C3 pass's shared-memory wavefronts, its data pipe at 83%).  The TMA
// boxes are therefore 20 wide there (columns 16..19 out of bounds: zero-
// filled on load, clipped on store), 160-byte rows.  (8-column rows, 64
// bytes, conflict 2-way; padding them to 96 bytes measured slower at W1,
// 0.49 -> 0.54 ms, and even at C4.)
#ifndef B2L_SGRAM_PAD16
#define B2L_SGRAM_PAD16 1
#endif
__host__ __device__ constexpr int sgram_pitch(int ld) {
  return (ld == 16 && B2L_SGRAM_PAD16) ? 20 : ld;
}
// Off by default: the other point order changes the Gram's rounding, and the
// golden 20^3 run (a chaotic degenerate-cluster endgame the tests hold to the
// reference's own 180..197 iteration band) then ends at 199.
#ifndef B2L_SGRAM_KSTRIDE
#define B2L_SGRAM_KSTRIDE 0
#endif

namespace b2l {

// LD = doubles per point of W / AW (template: it fixes the per-lane element
// count EPT = GPW*LD/4 and the Gram tile counts); GPW = 8-point groups per
// warp.  Every per-lane offset is precomputed once, so the plane loop is
// branch free: the stencil chains of a lane's EPT elements interleave and the
// Gram loads of all its rows issue ahead of the DMMAs.
// FULLB: the full block of the steady state (m = kw = ldx = LD) on a tile
// whose points fill every 8-point group and every lane's stencil elements
// (TX TY = 64 GPW, TX TY LD = 256 EPT): the Gram's shape, its lane-to-column
// maps and the X row stride are compile-time constants and no element or row
// predicate is needed (fewer address / predicate instructions per plane).
template <int LD, int GPW, int NST, int NOB, bool FULLB = false>
__global__ void __launch_bounds__(256, 2)
    stencil7_gram_kernel(const __grid_constant__ CUtensorMap tin,
                         const __grid_constant__ CUtensorMap thalo,
                         const __grid_constant__ CUtensorMap tout,
                         const __grid_constant__ CUtensorMap tx_map, StencilGeom g,
                         SGramGeom G) {
  constexpr int EPT = (GPW * LD + 3) / 4;
  constexpr int NI = (2 * LD + 7) / 8, NJ = (LD + 7) / 8;
  constexpr int NA = (NI * NJ >= 4) ? 1 : (NI * NJ >= 2 ? 2 : 4);
  constexpr int LDP = sgram_pitch(LD);   // pitch of the staged / output rows
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw;
  auto stage = [&](int s) -> double* {
    return reinterpret_cast<double*>(base + s * g.stage_stride);
  };
  auto outbuf = [&](int i) -> double* {
    return reinterpret_cast<double*>(base + NST * g.stage_stride + i * g.out_stride);
  };
  auto xbuf = [&](int i) -> double* {
    return reinterpret_cast<double*>(base + NST * g.stage_stride + NOB * g.out_stride +
                                     i * G.x_stride);
  };
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + NST * g.stage_stride + NOB * g.out_stride +
                                              2 * G.x_stride);
  uint64_t* xbar = bar + NST;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tx0 = (blockIdx.x % g.tiles_x) * g.TX;
  const int ty0 = (blockIdx.x / g.tiles_x) * g.TY;
  int z0, z1;
  stencil_zrange(g, z0, z1);
  const int ystride = (g.TX + 2) * LDP;
  auto staged_row = [&](int pt) { return (pt / g.TX + 1) * (g.TX + 2) + (pt % g.TX) + 1; };

  // stencil elements: the warp's groups (grp = warp + 8 gi) enumerated flat,
  // lane-contiguous (conflict-free smem).  Invalid slots read point 0.
  int off[EPT], oel[EPT];
  unsigned vmask = 0;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int idx = lane + 32 * i;
    const int gi = idx / (8 * LD), r = idx % (8 * LD);
    const int grp = warp + 8 * gi;
    const int e = grp * 8 * LD + r;
    const bool v = gi < GPW && grp < G.ngroups && e < g.nelem;
    const int p = v ? e / LD : 0;
    const int c = v ? e - p * LD : 0;
    off[i] = staged_row(p) * LDP + c;
    oel[i] = v ? p * LDP + c : 0;
    vmask |= (v ? 1u : 0u) << i;
  }
  // Gram rows: lane (q4 = lane & 3) holds point 8 grp + 4 ks + q4, or, where
  // that helps, 8 grp + 2 q4 + ks (the four points of a k-step two apart; any
  // fixed split of a group's 8 points over its two k-steps is a valid Gram).
  // At the 80-byte pitch of 10-column rows consecutive points put lanes of
  // one half-warp on the same banks (3-4 wavefronts per fragment load instead
  // of 2) and every other point does not (C2 pass 0.110 -> 0.107 ms); at 64-
  // or 128-byte pitches (m = 8, 16) the stride only makes it worse (W1 pass
  // 0.47 -> 0.58 ms), so it is taken only when 16 LD = 32 or 96 (mod 128).
  constexpr bool KS2 = B2L_SGRAM_KSTRIDE && ((16 * LD) % 128 == 32 || (16 * LD) % 128 == 96);
  const int q4 = lane & 3;
  const int Gm = FULLB ? LD : G.m, Gkw = FULLB ? LD : G.kw;
  const int Gldx = FULLB ? LDP : G.ldxp;   // pitch of the X tile
  const int Ga = Gm + Gkw, Gb = Gkw;
  int xo[GPW][2], po[GPW][2], oo[GPW][2];
  unsigned rmask = 0;
#pragma unroll
  for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int pt0 = 8 * (warp + 8 * gi) + (KS2 ? 2 * q4 + ks : 4 * ks + q4);
      const bool ok = pt0 < G.npts;
      const int pt = ok ? pt0 : 0;
      xo[gi][ks] = pt * Gldx;
      po[gi][ks] = staged_row(pt) * LDP;
      oo[gi][ks] = pt * LDP;
      rmask |= (ok ? 1u : 0u) << (2 * gi + ks);
    }
  // lane columns: L = [X (m) ; W (kw)], R = AW (kw)
  int acol[NI], bcol[NJ];
  bool aisx[NI], aok[NI], bok[NJ];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int ci = 8 * i + (lane >> 2);
    aok[i] = ci < Ga;
    aisx[i] = ci < Gm;
    acol[i] = !aok[i] ? 0 : (aisx[i] ? ci : ci - Gm);
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int cj = 8 * j + (lane >> 2);
    bok[j] = cj < Gb;
    bcol[j] = bok[j] ? cj : 0;
  }
  const int ni = (Ga + 7) / 8, nj = (Gb + 7) / 8;

  double gacc[NA][NI][NJ][2];
  // m = 10 full block: the Gram columns 8, 9 (AW's last two) on DFMA instead
  // of three 75%-empty DMMA column tiles; lane (row rl, point q4) keeps
  // sum over its points of L[row 8i + rl] * AW[8 + c] (reduced over q4 at the end)
  constexpr bool TAIL2 = FULLB && LD == 10 && NJ == 2;
  double tail[NI][2];
#pragma unroll
  for (int i = 0; i < NI; ++i) tail[i][0] = tail[i][1] = 0.0;
#pragma unroll
  for (int sa = 0; sa < NA; ++sa)
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) gacc[sa][i][j][0] = gacc[sa][i][j][1] = 0.0;

  if (z0 < z1) {
    const int nplanes = (z1 - z0) + 2;
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
      mbar_init(&xbar[0], 1);
      mbar_init(&xbar[1], 1);
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
    auto issue_x = [&](int z) {
      const int sl = (z - z0) & 1;
      mbar_expect_tx(&xbar[sl], G.x_bytes);
      tma_load_4d(xbuf(sl), &tx_map, &xbar[sl], 0, tx0, ty0, z);
    };
    const bool have_x = Gm > 0;   // m = 0: W^T AW only (PCG curvatures)
    if (tid == 0) {
      for (int q = 0; q < NST && q < nplanes; ++q) issue(q);
      if (have_x) {
        issue_x(z0);
        if (z0 + 1 < z1) issue_x(z0 + 1);
      }
    }
    double prev[EPT], cur[EPT];
    mbar_wait(&bar[0], 0);
#pragma unroll
    for (int i = 0; i < EPT; ++i) prev[i] = stage(0)[off[i]];
    mbar_wait(&bar[1 % NST], (1 / NST) & 1);
#pragma unroll
    for (int i = 0; i < EPT; ++i) cur[i] = stage(1 % NST)[off[i]];
    __syncthreads();
    if (tid == 0 && NST < nplanes) issue(NST);

    const double six = 6.0;
    const double sc = g.scale;
    for (int z = z0; z < z1; ++z) {
      const int q = z - z0 + 1;
      const int sn = (q + 1) % NST;
      mbar_wait(&bar[sn], ((q + 1) / NST) & 1);
      const double* P = stage(q % NST);
      const double* N = stage(sn);
      double* O = outbuf((z - z0) % NOB);
      // ---- stencil, reference operation order, no FMA contraction
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int o = off[i];
        const double nx_ = N[o];
        double r = __dmul_rn(six, cur[i]);
        r = __dsub_rn(r, P[o - LDP]);
        r = __dsub_rn(r, P[o + LDP]);
        r = __dsub_rn(r, P[o - ystride]);
        r = __dsub_rn(r, P[o + ystride]);
        r = __dsub_rn(r, prev[i]);
        r = __dsub_rn(r, nx_);
        if (FULLB || (vmask & (1u << i))) O[oel[i]] = __dmul_rn(sc, r);
        prev[i] = cur[i];
        cur[i] = nx_;
      }
      __syncwarp();
      // ---- Gram over this warp's rows (points); the lane reads only rows
      // its own warp wrote, so no CTA barrier is needed before it
      const int xs = (z - z0) & 1;
      if (have_x) mbar_wait(&xbar[xs], ((z - z0) >> 1) & 1);
      const double* Xb = xbuf(xs);
#pragma unroll
      for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          // Lanes past the Gram's rows (ci >= a) or columns (cj >= b) load a
          // finite in-tile value (column 0): it only reaches output entries
          // that are never written back, so no select is needed.  Points past
          // the tile (rok false, partial last groups) must contribute zero:
          // zeroing one operand (B) suffices.
          const bool rok = FULLB || (rmask & (1u << (2 * gi + ks)));
          double av[NI], bv[NJ];
#pragma unroll
          for (int i = 0; i < NI; ++i)
            av[i] = aisx[i] ? Xb[xo[gi][ks] + acol[i]] : P[po[gi][ks] + acol[i]];
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const double v = O[oo[gi][ks] + bcol[j]];
            bv[j] = rok ? v : 0.0;
          }
          const int sa = (2 * gi + ks) % NA;
          if constexpr (TAIL2) {
            const double aw8 = O[oo[gi][ks] + 8], aw9 = O[oo[gi][ks] + 9];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              dmma_8x8x4(gacc[0][i][0][0], gacc[0][i][0][1], av[i], bv[0]);
              tail[i][0] = fma(av[i], aw8, tail[i][0]);
              tail[i][1] = fma(av[i], aw9, tail[i][1]);
            }
          } else {
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j)
              if (i < ni && j < nj) {
#pragma unroll
                for (int t = 0; t < NA; ++t)
                  if (t == sa) dmma_8x8x4(gacc[t][i][j][0], gacc[t][i][j][1], av[i], bv[j]);
              }
          }
        }
      // The next plane writes output slot (z + 1) % NOB, last stored for
      // plane z + 1 - NOB: its TMA store must have read the slot before the
      // barrier releases the writers (a wait after the barrier would let the
      // other threads overwrite it while thread 0 still waits).
      if (tid == 0) bulk_wait_read<NOB - 2>();
      __syncthreads();
      if (tid == 0) {
        fence_async_smem();
        tma_store_4d(&tout, O, 0, tx0, ty0, z);
        bulk_commit();
        if (q + NST < nplanes) issue(q + NST);
        if (have_x && z + 2 < z1) issue_x(z + 2);
      }
    }
    if (tid == 0) bulk_wait<0>();
  }

  if constexpr (TAIL2) {
    // columns 8, 9: the sum over the lane's 4 point slots (q4), fixed order,
    // lands where the DMMA fragment layout keeps C[row][8 + e] (lane q4 = 0)
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double v01 = tail[i][e] + __shfl_xor_sync(0xffffffffu, tail[i][e], 1);
        const double v = v01 + __shfl_xor_sync(0xffffffffu, v01, 2);
        gacc[0][i][1][e] = q4 == 0 ? v : 0.0;
      }
  }
  // ---- CTA partial: fixed-order sum over the 8 warps (reuse stage memory)
  __syncthreads();
  double* red = reinterpret_cast<double*>(base);
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const size_t o = (((size_t)warp * NI * NJ + i * NJ + j) * 32 + lane) * 2;
      double v0 = gacc[0][i][j][0], v1 = gacc[0][i][j][1];
#pragma unroll
      for (int sa = 1; sa < NA; ++sa) {
        v0 += gacc[sa][i][j][0];
        v1 += gacc[sa][i][j][1];
      }
      red[o] = v0;
      red[o + 1] = v1;
    }
  __syncthreads();
  const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  double* outp = G.partial + cta * G.a * G.b;
  for (int e = tid; e < NI * NJ * 32; e += blockDim.x) {
    const int t = e / 32, ln = e & 31;
    double v0 = 0.0, v1 = 0.0;
    for (int w = 0; w < 8; ++w) {
      const size_t o = (((size_t)w * NI * NJ + t) * 32 + ln) * 2;
      v0 += red[o];
      v1 += red[o + 1];
    }
    const int row = 8 * (t / NJ) + (ln >> 2);
    const int col = 8 * (t % NJ) + 2 * (ln & 3);
    if (row < G.a) {
      if (col < G.b) outp[(size_t)row * G.b + col] = v0;
      if (col + 1 < G.b) outp[(size_t)row * G.b + col + 1] = v1;
    }
  }
}

int stencil7(const double* in, double* out, int nx, int ny, int nz, int ld, const double* halo,
             int has_lo, int has_hi, double scale, cudaStream_t st, int zmode = 0);
struct HostBlock {
  const double* p;
  int ld, cols;
};
int gram(int nrows, const HostBlock* L, int nl, const HostBlock* R, int nr, unsigned rw_mask,
         const double* d, const unsigned char* pair_mode, double* out, cudaStream_t st);

template <int LD, int GPW>
static int launch_sgram_t(const StencilPlan& p, size_t smem, const CUtensorMap& tin,
                          const CUtensorMap& thalo, const CUtensorMap& tout,
                          const CUtensorMap& txm, const SGramGeom& G, cudaStream_t st) {
  // a 4-deep plane ring with double-buffered outputs when it fits two CTAs
  // per SM (more loads in flight), else 3 + 3; the compile-time full block
  // for the block sizes of the BASELINE configs (m = 8, 10, 16)
  constexpr bool FB_OK = LD == 8 || LD == 10 || LD == 16;
  constexpr int EPT = (GPW * LD + 3) / 4;
  const bool full = FB_OK && G.m == LD && G.kw == LD && G.ldx == LD && G.npts == 64 * GPW &&
                    p.g.nelem == 256 * EPT;
  auto kern = p.nst == 4 ? (full ? stencil7_gram_kernel<LD, GPW, 4, 2, FB_OK>
                                 : stencil7_gram_kernel<LD, GPW, 4, 2, false>)
              : p.nob == 3 ? (full ? stencil7_gram_kernel<LD, GPW, 3, 3, FB_OK>
                                   : stencil7_gram_kernel<LD, GPW, 3, 3, false>)
                           : (full ? stencil7_gram_kernel<LD, GPW, 3, 2, FB_OK>
                                   : stencil7_gram_kernel<LD, GPW, 3, 2, false>);
  if (int rc = prepare_kernel(reinterpret_cast<const void*>(kern), smem, 256, nullptr)) return rc;
  kern<<<p.grid, 256, smem, st>>>(tin, thalo, tout, txm, p.g, G);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}

template <int LD>
static int launch_sgram_ld(int gpw, const StencilPlan& p, size_t smem, const CUtensorMap& tin,
                           const CUtensorMap& thalo, const CUtensorMap& tout,
                           const CUtensorMap& txm, const SGramGeom& G, cudaStream_t st) {
  switch (gpw) {
    case 1: return launch_sgram_t<LD, 1>(p, smem, tin, thalo, tout, txm, G, st);
    case 2: return launch_sgram_t<LD, 2>(p, smem, tin, thalo, tout, txm, G, st);
    case 3: return launch_sgram_t<LD, 3>(p, smem, tin, thalo, tout, txm, G, st);
    default: return launch_sgram_t<LD, 4>(p, smem, tin, thalo, tout, txm, G, st);
  }
}

int sgram_plan(const double* in, double* out, int nx, int ny, int nz, int ld, const double* halo,
               int has_lo, int has_hi, double scale, const double* x, int ldx, int m, int kw,
               int zmode, SGramPlan* P) {
  B2L_CHECK(nx > 0 && ny > 0 && nz > 0, -B2L_EINVAL, "stencil: empty grid");
  B2L_CHECK(ld >= 2 && (ld % 2) == 0 && (m == 0 || (ldx >= 2 && (ldx % 2) == 0)), -B2L_EINVAL,
            "stencil: ld and ldx must be even (16-B rows for TMA)");
  B2L_CHECK(kw >= 1 && kw <= ld && m >= 0 && m <= ldx && (m == 0 || x), -B2L_EINVAL,
            "stencil: bad m / kw");
  B2L_CHECK(in != out, -B2L_EINVAL, "stencil: in-place apply not supported");
  B2L_CHECK(!(has_lo || has_hi) || halo != nullptr, -B2L_EINVAL,
            "stencil: halo flags set without a halo buffer");
  *P = SGramPlan{};
  P->in = in;
  P->out = out;
  P->x = x;
  P->nx = nx;
  P->ny = ny;
  P->nz = nz;
  P->ld = ld;
  P->ldx = ldx;
  P->halo = halo;
  P->has_lo = has_lo;
  P->has_hi = has_hi;
  P->scale = scale;
  P->zmode = zmode;
  SGramGeom& G = P->G;
  G.m = m;
  G.ldx = ldx;
  G.kw = kw;
  G.a = m + kw;
  G.b = kw;
  if (ld > 16 || m > ld) {
    // outside the fused kernel's templates: the two-pass form (K1, then K5)
    P->twopass = 1;
    P->nparts = 0;
    return 0;
  }
  StencilPlan& p = P->p;
  int rc = plan_stencil(nx, ny, nz, ld, &p);
  if (rc) return rc;
  StencilGeom& g = p.g;
  const int TX = g.TX;
  // shared-memory pitches (sgram_pitch): the boxes of the tensor maps below
  const int ldp = sgram_pitch(ld), ldxp = m ? sgram_pitch(ldx) : ldx;
  G.ldxp = ldxp;
  auto need = [&](int ty) {
    const size_t stg = (((size_t)(TX + 2) * (ty + 2) * ldp * 8) + 127) & ~(size_t)127;
    const size_t ob = (((size_t)TX * ty * ldp * 8) + 127) & ~(size_t)127;
    const size_t xb = m ? ((((size_t)TX * ty * ldxp * 8) + 127) & ~(size_t)127) : 0;
    return 3 * stg + 3 * ob + 2 * xb + 128;
  };
  auto need4 = [&](int ty) {
    const size_t stg = (((size_t)(TX + 2) * (ty + 2) * ldp * 8) + 127) & ~(size_t)127;
    const size_t ob = (((size_t)TX * ty * ldp * 8) + 127) & ~(size_t)127;
    const size_t xb = m ? ((((size_t)TX * ty * ldxp * 8) + 127) & ~(size_t)127) : 0;
    return 4 * stg + 2 * ob + 2 * xb + 128;
  };
  auto need32 = [&](int ty) {   // the smallest ring: 3 planes, 2 output tiles
    const size_t stg = (((size_t)(TX + 2) * (ty + 2) * ldp * 8) + 127) & ~(size_t)127;
    const size_t ob = (((size_t)TX * ty * ldp * 8) + 127) & ~(size_t)127;
    const size_t xb = m ? ((((size_t)TX * ty * ldxp * 8) + 127) & ~(size_t)127) : 0;
    return 3 * stg + 2 * ob + 2 * xb + 128;
  };
  // 8 warps x GPW groups of 8 points per tile; the largest tile that keeps
  // two CTAs resident per SM (<= ~110 KB shared memory) wins
  int gpw = 0, TY = 1;
  for (int cand = 4; cand >= 1; --cand) {
    if ((cand * ld + 3) / 4 > 16) continue;
    int ty = (64 * cand) / TX;
    if (ty < 1) ty = 1;
    if (ty > ny) ty = ny;
    if (ty > 254) ty = 254;
    if (TX * ty > 64 * cand) continue;
    if (need32(ty) > 110 * 1024) continue;
    gpw = cand;
    TY = ty;
    break;
  }
  B2L_CHECK(gpw > 0, -B2L_EINVAL, "stencil_gram: no tile fits shared memory");
  // shrink the group count to what the tile actually holds
  while (gpw > 1 && 64 * (gpw - 1) >= TX * TY) --gpw;
  g.TY = TY;
  g.nelem = TX * TY * ld;
  G.npts = TX * TY;
  G.ngroups = (G.npts + 7) / 8;
  const int tiles_y = (ny + TY - 1) / TY;
  const int tiles = g.tiles_x * tiles_y;
  g.stage_bytes = (uint32_t)((TX + 2) * (TY + 2) * ldp * 8);
  g.stage_stride = (g.stage_bytes + 127u) & ~127u;
  g.out_stride = ((uint32_t)(TX * TY * ldp * 8) + 127u) & ~127u;
  G.x_bytes = m ? (uint32_t)(TX * TY * ldxp * 8) : 0u;
  G.x_stride = (G.x_bytes + 127u) & ~127u;
  size_t smem = need32(TY);
  p.nst = 3;
  p.nob = 2;
  if (need4(TY) <= 110 * 1024) {
    p.nst = 4;
    smem = need4(TY);
  } else if (need(TY) <= 110 * 1024) {
    p.nob = 3;
    smem = need(TY);
  }
  const int NI = (2 * ld + 7) / 8, NJ = (ld + 7) / 8;
  const size_t red = (size_t)8 * NI * NJ * 64 * 8;
  if (red > smem) smem = red + 128;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "stencil_gram: tile does not fit");
  P->smem = smem;
  P->gpw = gpw;
  if (!apply_zmode(g, p.grid, tiles, zmode, 2 * sm_count())) {
    P->nparts = 0;   // no plane in this mode
    return 0;
  }
  if (zmode == Z_ALL) {
    if (const char* zc = getenv("B2L_SGRAM_ZCHUNK")) {     // tuning override
      const int v = atoi(zc);
      if (v >= 1) {
        g.zchunk = v < nz ? v : nz;
        p.grid.y = (nz + g.zchunk - 1) / g.zchunk;
      }
    }
  }
  g.has_lo = has_lo;
  g.has_hi = has_hi;
  g.scale = scale;
  P->nparts = (int)(p.grid.x * p.grid.y);
  rc = encode_tmap_4d(&P->tin, in, ld, nx, ny, nz, ldp, TX + 2, TY + 2, 1);
  if (rc) return rc;
  rc = encode_tmap_4d(&P->tout, out, ld, nx, ny, nz, ldp, TX, TY, 1);
  if (rc) return rc;
  if (m) {
    rc = encode_tmap_4d(&P->txm, x, ldx, nx, ny, nz, ldxp, TX, TY, 1);
    if (rc) return rc;
  } else {
    P->txm = P->tout;   // never loaded
  }
  if (halo) {
    rc = encode_tmap_4d(&P->thalo, halo, ld, nx, ny, 2, ldp, TX + 2, TY + 2, 1);
    if (rc) return rc;
  } else {
    P->thalo = P->tin;
  }
  return 0;
}

int sgram_launch(SGramPlan& P, double* partial, cudaStream_t st) {
  if (P.twopass)
    return stencil7(P.in, P.out, P.nx, P.ny, P.nz, P.ld, P.halo, P.has_lo, P.has_hi, P.scale, st,
                    P.zmode);
  if (P.nparts == 0) return 0;
  P.G.partial = partial;
  const StencilPlan& p = P.p;
  const int gpw = P.gpw;
  const size_t smem = P.smem;
  const SGramGeom& G = P.G;
  switch (P.ld) {
    case 2: return launch_sgram_ld<2>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 4: return launch_sgram_ld<4>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 6: return launch_sgram_ld<6>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 8: return launch_sgram_ld<8>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 10: return launch_sgram_ld<10>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 12: return launch_sgram_ld<12>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    case 14: return launch_sgram_ld<14>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
    default: return launch_sgram_ld<16>(gpw, p, smem, P.tin, P.thalo, P.tout, P.txm, G, st);
  }
}

// The Gram of a two-pass plan (after its stencil launches), or the sum of
// the CTA partials of fused launches.
int sgram_finish(const SGramPlan& P, const double* partial, int nparts, double* gram_out,
                 cudaStream_t st) {
  const SGramGeom& G = P.G;
  if (P.twopass) {
    const HostBlock L[2] = {{P.x, P.ldx, G.m}, {P.in, P.ld, G.kw}};
    const HostBlock R[1] = {{P.out, P.ld, G.kw}};
    const int rows = P.nx * P.ny * P.nz;
    if (G.m == 0) return gram(rows, L + 1, 1, R, 1, 0u, nullptr, nullptr, gram_out, st);
    return gram(rows, L, 2, R, 1, 0u, nullptr, nullptr, gram_out, st);
  }
  return sum_parts(partial, nparts, G.a * G.b, gram_out, st);
}

int stencil7_gram(const double* in, double* out, int nx, int ny, int nz, int ld,
                  const double* halo, int has_lo, int has_hi, double scale,
                  const double* x, int ldx, int m, int kw, double* gram_out,
                  cudaStream_t st) {
  SGramPlan P;
  int rc = sgram_plan(in, out, nx, ny, nz, ld, halo, has_lo, has_hi, scale, x, ldx, m, kw, Z_ALL,
                      &P);
  if (rc) return rc;
  double* part = nullptr;
  if (!P.twopass) {
    int werr = 0;
    part = static_cast<double*>(
        workspace((size_t)P.nparts * P.G.a * P.G.b * sizeof(double), &werr));
    if (werr) return werr;
  }
  rc = sgram_launch(P, part, st);
  if (rc) return rc;
  return sgram_finish(P, part, P.nparts, gram_out, st);
}

// Interior planes (no halo needed), then the two edge planes (halo), one
// partial buffer, one second-stage sum: the z-slab overlap form
// (b2l_slab_stencil7_gram runs the halo exchange between the two launches;
// this single-stream variant serves tests and halo-less callers).
int stencil7_gram_split(const double* in, double* out, int nx, int ny, int nz, int ld,
                        const double* halo, int has_lo, int has_hi, double scale,
                        const double* x, int ldx, int m, int kw, double* gram_out,
                        cudaStream_t st, double** part_buf, size_t* part_cap,
                        cudaEvent_t before_edges) {
  SGramPlan Pi, Pe;
  int rc = sgram_plan(in, out, nx, ny, nz, ld, halo, has_lo, has_hi, scale, x, ldx, m, kw,
                      Z_INTERIOR, &Pi);
  if (rc) return rc;
  rc = sgram_plan(in, out, nx, ny, nz, ld, halo, has_lo, has_hi, scale, x, ldx, m, kw, Z_EDGE,
                  &Pe);
  if (rc) return rc;
  const size_t len = (size_t)Pi.G.a * Pi.G.b;
  const size_t need = ((size_t)Pi.nparts + Pe.nparts) * len;
  double* part = nullptr;
  if (!Pi.twopass) {
    if (part_buf) {
      if (*part_cap < need) {
        if (*part_buf) B2L_CUDA(cudaFree(*part_buf));
        *part_buf = nullptr;
        *part_cap = 0;
        B2L_CUDA(cudaMalloc(part_buf, need * sizeof(double)));
        *part_cap = need;
      }
      part = *part_buf;
    } else {
      int werr = 0;
      part = static_cast<double*>(workspace(need * sizeof(double), &werr));
      if (werr) return werr;
    }
  }
  rc = sgram_launch(Pi, part, st);
  if (rc) return rc;
  if (before_edges) B2L_CUDA(cudaStreamWaitEvent(st, before_edges, 0));
  rc = sgram_launch(Pe, part ? part + (size_t)Pi.nparts * len : nullptr, st);
  if (rc) return rc;
  return sgram_finish(Pi, part, Pi.nparts + Pe.nparts, gram_out, st);
}

}  // namespace b2l
