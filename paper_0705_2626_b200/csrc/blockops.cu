// Tall-skinny block kernels for the LOBPCG iteration (sm_100a).
//
//   K5  gram      : L^T diag(w) R over several (n, ld) blocks at once
//                   (reference multivec.py:58-71, 11 calls per iteration at
//                   lobpcg.py:419, :176, :325-338 collapsed into one pass)
//   K4+K2 resid   : W = T (AX - BX Lambda) for the active columns, plus the
//                   squared column norms of every residual
//                   (lobpcg.py:429-430, :466-467; operators.py:297-298)
//   K6  update    : P' = W Cw + P_J Cp ; X' = X Cx + P' and the A-side twins
//                   (lobpcg.py:520-540; multivec.py:74-86), with the Cholesky
//                   factors of W and P folded into Cw/Cp on the host so W and P
//                   are never rewritten (replaces tri_solve_right,
//                   multivec.py:125-146): one thread per row for m <= 16,
//                   DMMA with resident coefficients for 16 < m <= 64, a scalar
//                   fallback otherwise
//   K5 for wide / large Grams (gram_big): 4x4 tile blocks per warp, padded
//                   TMA rows, producer warp (the m = 64 pencil of C5)
//
// Every reduction is deterministic: CTA partials in a fixed row assignment,
// then a fixed-order second stage over CTAs.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "gram_tile.cuh"

namespace b2l {

// =========================================================================
// K5: multi-block Gram on fp64 tensor cores (DMMA), TMA-staged row chunks
// =========================================================================
constexpr int GRAM_THREADS = 256;
constexpr int GRAM_MAXU = 8;
constexpr int GRAM_MAXL = 4;
constexpr int GRAM_MAXR = 8;
constexpr int GT_TI = 2;      // 8x8 tiles per warp tile block (rows)
constexpr int GT_TJ = 4;      //                               (cols)

struct GramArgs {
  int nrows;
  int rc;  // rows per chunk (power of 2, >= 4*rs)
  int nu;
  const double* up[GRAM_MAXU];
  int uld[GRAM_MAXU];
  int ubase[GRAM_MAXU];  // offset (doubles) of block u inside a stage
  int a, b;              // total left / right columns
  int nl, nr;
  int lu[GRAM_MAXL], lcum[GRAM_MAXL + 1];
  int ru[GRAM_MAXR], rcum[GRAM_MAXR + 1];
  unsigned rw_mask;
  const double* d;
  int dbase;
  int stage_doubles;
  int nst;
  int NI, NJ, tsI, tsJ;  // 8x8 tile grid, TIxTJ tile-block grid
  int ts_per_cta, rs;    // tile blocks per CTA, row slices per chunk
  unsigned tmask[32];    // needed-tile bitmap, bit (i*NJ + j)
  double* partial;       // [gridDim.x][a*b]
};


__device__ __forceinline__ void gram_issue(const GramArgs& A, double* st, uint64_t* bar, int c) {
  const int r0 = c * A.rc;
  const int nvalid = min(A.rc, A.nrows - r0);
  const int nv4 = (nvalid + 3) & ~3;
  // zero the rows that complete the last 4-row group of a tail chunk
  for (int u = 0; u < A.nu; ++u)
    for (int e = nvalid * A.uld[u]; e < nv4 * A.uld[u]; ++e) st[A.ubase[u] + e] = 0.0;
  uint32_t tx = 0;
  for (int u = 0; u < A.nu; ++u) tx += (uint32_t)nvalid * A.uld[u] * 8u;
  const bool d_bulk = A.d && (nvalid % 2 == 0);
  if (A.d) {
    if (d_bulk) {
      tx += (uint32_t)nvalid * 8u;
      for (int e = nvalid; e < nv4; ++e) st[A.dbase + e] = 0.0;
    } else {
      for (int e = 0; e < nv4; ++e) st[A.dbase + e] = e < nvalid ? A.d[r0 + e] : 0.0;
    }
  }
  fence_async_smem();
  mbar_expect_tx(bar, tx);
  for (int u = 0; u < A.nu; ++u)
    bulk_load(st + A.ubase[u], A.up[u] + (size_t)r0 * A.uld[u],
              (uint32_t)nvalid * A.uld[u] * 8u, bar);
  if (d_bulk) bulk_load(st + A.dbase, A.d + r0, (uint32_t)nvalid * 8u, bar);
}

__global__ void __launch_bounds__(GRAM_THREADS) gram_kernel(GramArgs A) {
  extern __shared__ __align__(128) unsigned char gsm_raw[];
  double* stages = reinterpret_cast<double*>(gsm_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(gsm_raw + (size_t)A.nst * A.stage_doubles * 8);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  const int tsl = warp % A.ts_per_cta;
  const int slice = warp / A.ts_per_cta;
  const int ts = blockIdx.y * A.ts_per_cta + tsl;
  const bool wactive = slice < A.rs && ts < A.tsI * A.tsJ;
  const int ti0 = wactive ? (ts / A.tsJ) * GT_TI : 0;
  const int tj0 = wactive ? (ts % A.tsJ) * GT_TJ : 0;

  LaneCol la[GT_TI], lb[GT_TJ];
#pragma unroll
  for (int i = 0; i < GT_TI; ++i) {
    const int ci = 8 * (ti0 + i) + (lane >> 2);
    la[i] = LaneCol{0, 0, false, false};
    if (ci < A.a) {
      int l = 0;
      while (l + 1 < A.nl && A.lcum[l + 1] <= ci) ++l;
      la[i] = LaneCol{A.ubase[A.lu[l]] + (ci - A.lcum[l]), A.uld[A.lu[l]], true, false};
    }
  }
#pragma unroll
  for (int j = 0; j < GT_TJ; ++j) {
    const int cj = 8 * (tj0 + j) + (lane >> 2);
    lb[j] = LaneCol{0, 0, false, false};
    if (cj < A.b) {
      int r = 0;
      while (r + 1 < A.nr && A.rcum[r + 1] <= cj) ++r;
      lb[j] = LaneCol{A.ubase[A.ru[r]] + (cj - A.rcum[r]), A.uld[A.ru[r]], true,
                      ((A.rw_mask >> r) & 1u) != 0};
    }
  }
  unsigned mask = 0;
#pragma unroll
  for (int i = 0; i < GT_TI; ++i)
#pragma unroll
    for (int j = 0; j < GT_TJ; ++j) {
      const int ti = ti0 + i, tj = tj0 + j;
      if (wactive && ti < A.NI && tj < A.NJ) {
        const int t = ti * A.NJ + tj;
        if ((A.tmask[t >> 5] >> (t & 31)) & 1u) mask |= 1u << (i * GT_TJ + j);
      }
    }

  WarpGram<GT_TI, GT_TJ> g;
  g.zero();

  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      const int c = blockIdx.x + s * gridDim.x;
      if (c < nchunks) gram_issue(A, stages + (size_t)s * A.stage_doubles, &bar[s], c);
    }
  }
  const int rows_per_slice = A.rc / A.rs;
  int it = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int s = it % A.nst;
    double* st = stages + (size_t)s * A.stage_doubles;
    mbar_wait(&bar[s], (it / A.nst) & 1);
    const int nvalid = min(A.rc, A.nrows - c * A.rc);
    const int nv4 = (nvalid + 3) & ~3;
    if (wactive && mask) {
      const int lo = slice * rows_per_slice;
      const int hi = min(lo + rows_per_slice, nv4);
      g.run(st, la, lb, A.d ? st + A.dbase : nullptr, lo, hi, mask, DenseRows());
    }
    __syncthreads();
    if (tid == 0) {
      const int cn = c + A.nst * gridDim.x;
      if (cn < nchunks) gram_issue(A, st, &bar[s], cn);
    }
  }
  __syncthreads();

  // fixed-order reduction of the row slices, then the CTA partial
  double* red = stages;
  const int nt = GT_TI * GT_TJ;
  if (wactive && slice > 0) {
#pragma unroll
    for (int i = 0; i < GT_TI; ++i)
#pragma unroll
      for (int j = 0; j < GT_TJ; ++j) {
        const size_t o = ((((size_t)(slice - 1) * A.ts_per_cta + tsl) * nt + i * GT_TJ + j) * 32 + lane) * 2;
        red[o] = g.acc[i][j][0];
        red[o + 1] = g.acc[i][j][1];
      }
  }
  __syncthreads();
  if (wactive && slice == 0) {
    double* out = A.partial + (size_t)blockIdx.x * A.a * A.b;
#pragma unroll
    for (int i = 0; i < GT_TI; ++i)
#pragma unroll
      for (int j = 0; j < GT_TJ; ++j) {
        double v0 = g.acc[i][j][0], v1 = g.acc[i][j][1];
        for (int sl = 1; sl < A.rs; ++sl) {
          const size_t o = ((((size_t)(sl - 1) * A.ts_per_cta + tsl) * nt + i * GT_TJ + j) * 32 + lane) * 2;
          v0 += red[o];
          v1 += red[o + 1];
        }
        const int row = 8 * (ti0 + i) + (lane >> 2);
        const int col = 8 * (tj0 + j) + 2 * (lane & 3);
        if (row < A.a) {
          if (col < A.b) out[(size_t)row * A.b + col] = v0;
          if (col + 1 < A.b) out[(size_t)row * A.b + col + 1] = v1;
        }
      }
  }
}


struct HostBlock {
  const double* p;
  int ld, cols;
};


// -------------------------------------------------------------------------
// K5 for large Grams (the m = 64 pencil of C5: [X W P]^T [BX BW BP AP] is
// 24 x 32 tiles of 8x8, ~490 needed): every warp owns a 4x4 block of needed
// tiles (16 DMMA per 8 fragment loads, accumulators in registers for the
// whole pass), the needed tile blocks are split over gridDim.y CTA groups,
// row chunks of every block stream through a TMA ring (2-D tile loads with
// padded shared rows -> conflict-free fragment loads) filled by one producer
// warp with full / empty mbarriers, no CTA-wide barrier in the loop.  CTAs
// of one row range but different tile groups run side by side, so the
// re-reads of a chunk hit L2.  Deterministic like K5: per-CTA partials,
// fixed-order second stage.
constexpr int GB_TI = 4, GB_TJ = 4, GB_MAXW = 12, GB_MAXBLK = 64;

struct GbArgs {
  int nrows, rc, nst;
  int nu;
  int ubase[GRAM_MAXU];        // stage offsets (doubles)
  int ustr[GRAM_MAXU];         // shared row strides
  int a, b, nl, nr;
  int lu[GRAM_MAXL], lcum[GRAM_MAXL + 1];
  int ru[GRAM_MAXR], rcum[GRAM_MAXR + 1];
  unsigned rw_mask;
  const double* d;
  int dbase;
  int stage_doubles;
  uint32_t stage_tx;
  int wpc, nblk, nzero;
  int ks, nwc;                       // row (k) slices per chunk; compute warps = wpc * ks
  unsigned short blk[GB_MAXBLK];     // (ti0 << 8) | tj0 of needed 4x4 tile blocks
  unsigned short bmask[GB_MAXBLK];   // needed tiles inside the block, bit i*4+j
  unsigned short zblk[GB_MAXBLK];    // tile blocks nobody computes (zeroed)
  double* partial;                   // [gridDim.x][ks][a*b]
};
struct GbMaps {
  CUtensorMap u[GRAM_MAXU];
};

template <int KS>
__global__ void __launch_bounds__(32 * (GB_MAXW + 1), 1)
    gram_big_kernel(const __grid_constant__ GbMaps M, const __grid_constant__ GbArgs A) {
  extern __shared__ __align__(128) unsigned char gb_raw[];
  double* stages = reinterpret_cast<double*>(gb_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(gb_raw + (size_t)A.nst * A.stage_doubles * 8);
  uint64_t* empty = full + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], A.nwc);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int ksl = KS == 1 ? 0 : warp / A.wpc;   // this warp's row slice of every chunk
  double* out = A.partial + ((size_t)blockIdx.x * KS + (warp < A.nwc ? ksl : 0)) * A.a * A.b;

  if (warp == A.nwc) {
    // ---- producer
    if (lane == 0)
      for (int it = 0; it < nloc; ++it) {
        const int s = it % A.nst;
        if (it >= A.nst) mbar_wait(&empty[s], (it / A.nst - 1) & 1);
        double* st = stages + (size_t)s * A.stage_doubles;
        const int r0 = (blockIdx.x + it * gridDim.x) * A.rc;
        const int nvalid = min(A.rc, A.nrows - r0);
        uint32_t tx = A.stage_tx;
        bool dbulk = false;
        if (A.d) {
          dbulk = (nvalid % 2) == 0;
          if (dbulk) tx += (uint32_t)nvalid * 8u;
          else
            for (int e = 0; e < nvalid; ++e) st[A.dbase + e] = A.d[r0 + e];
          for (int e = nvalid; e < A.rc; ++e) st[A.dbase + e] = 0.0;
          fence_async_smem();
        }
        mbar_expect_tx(&full[s], tx);
        for (int u = 0; u < A.nu; ++u) tma_load_2d(st + A.ubase[u], &M.u[u], &full[s], 0, r0);
        if (dbulk) bulk_load(st + A.dbase, A.d + r0, (uint32_t)nvalid * 8u, &full[s]);
      }
  } else if (warp < A.nwc) {
    const int bi = blockIdx.y * A.wpc + (KS == 1 ? warp : warp % A.wpc);
    const bool act = bi < A.nblk;
    const int ti0 = act ? (A.blk[bi] >> 8) : 0, tj0 = act ? (A.blk[bi] & 255) : 0;
    const unsigned mask = act ? A.bmask[bi] : 0u;
    LaneCol la[GB_TI], lb[GB_TJ];
#pragma unroll
    for (int i = 0; i < GB_TI; ++i) {
      const int ci = 8 * (ti0 + i) + (lane >> 2);
      la[i] = LaneCol{0, 0, false, false};
      if (act && ci < A.a) {
        int l = 0;
        while (l + 1 < A.nl && A.lcum[l + 1] <= ci) ++l;
        la[i] = LaneCol{A.ubase[A.lu[l]] + (ci - A.lcum[l]), A.ustr[A.lu[l]], true, false};
      }
    }
#pragma unroll
    for (int j = 0; j < GB_TJ; ++j) {
      const int cj = 8 * (tj0 + j) + (lane >> 2);
      lb[j] = LaneCol{0, 0, false, false};
      if (act && cj < A.b) {
        int r = 0;
        while (r + 1 < A.nr && A.rcum[r + 1] <= cj) ++r;
        lb[j] = LaneCol{A.ubase[A.ru[r]] + (cj - A.rcum[r]), A.ustr[A.ru[r]], true,
                        ((A.rw_mask >> r) & 1u) != 0};
      }
    }
    WarpGram<GB_TI, GB_TJ> g;
    g.zero();
    // Branch-free inner loop: all 16 tiles of the block are accumulated (the
    // few unneeded ones are never read), lanes whose column lies beyond the
    // Gram read a valid smem column instead (their products land only in
    // accumulator rows / columns the output loop skips), and the loads walk
    // fixed per-lane offsets -- no predicated mma (no WARPSYNC per DMMA).
    const int q = lane & 3;
    int aoff[GB_TI], astr[GB_TI], boff[GB_TJ], bstr[GB_TJ];
    bool bw[GB_TJ];
#pragma unroll
    for (int i = 0; i < GB_TI; ++i) {
      aoff[i] = la[i].ok ? la[i].off + q * la[i].str : A.ubase[0];
      astr[i] = la[i].ok ? 4 * la[i].str : 0;
    }
#pragma unroll
    for (int j = 0; j < GB_TJ; ++j) {
      boff[j] = lb[j].ok ? lb[j].off + q * lb[j].str : A.ubase[0];
      bstr[j] = lb[j].ok ? 4 * lb[j].str : 0;
      bw[j] = lb[j].ok && lb[j].weighted;
    }
    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst;
      mbar_wait(&full[s], (it / A.nst) & 1);
      const double* st = stages + (size_t)s * A.stage_doubles;
      if (mask) {
        const double* dw = A.d ? st + A.dbase + q : nullptr;
#pragma unroll 2
        for (int r = 4 * ksl; r < A.rc; r += 4 * KS) {
          const int k4 = r >> 2;
          double av[GB_TI], bv[GB_TJ];
#pragma unroll
          for (int i = 0; i < GB_TI; ++i) av[i] = st[aoff[i] + k4 * astr[i]];
          const double w = dw ? dw[r] : 1.0;
#pragma unroll
          for (int j = 0; j < GB_TJ; ++j) {
            const double v = st[boff[j] + k4 * bstr[j]];
            bv[j] = bw[j] ? __dmul_rn(w, v) : v;
          }
#pragma unroll
          for (int i = 0; i < GB_TI; ++i)
#pragma unroll
            for (int j = 0; j < GB_TJ; ++j) dmma_8x8x4(g.acc[i][j][0], g.acc[i][j][1], av[i], bv[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }
    if (act) {
#pragma unroll
      for (int i = 0; i < GB_TI; ++i)
#pragma unroll
        for (int j = 0; j < GB_TJ; ++j) {
          const int row = 8 * (ti0 + i) + (lane >> 2);
          const int col = 8 * (tj0 + j) + 2 * (lane & 3);
          if (row < A.a) {
            if (col < A.b) out[(size_t)row * A.b + col] = g.acc[i][j][0];
            if (col + 1 < A.b) out[(size_t)row * A.b + col + 1] = g.acc[i][j][1];
          }
        }
    }
  }
  // tile blocks nobody computes: defined zeros (group 0 of every row range)
  if (blockIdx.y == 0)
    for (int e = tid; e < KS * A.nzero * 256; e += blockDim.x) {
      const int kz = e / (A.nzero * 256), ez = e % (A.nzero * 256);
      const int zb = ez >> 8, t = ez & 255;
      const int row = 8 * (A.zblk[zb] >> 8) + (t >> 4);
      const int col = 8 * (A.zblk[zb] & 255) + (t & 15) * 2;
      double* o = A.partial + ((size_t)blockIdx.x * KS + kz) * A.a * A.b;
      for (int c = col; c < col + 2; ++c)
        if (row < A.a && c < A.b) o[(size_t)row * A.b + c] = 0.0;
    }
}

// The large-Gram path of gram(): returns 1 when the shapes do not qualify.
static int gram_big(int nrows, const HostBlock* L, int nl, const HostBlock* R, int nr,
                    unsigned rw_mask, const double* d, const GramArgs& G, double* out,
                    cudaStream_t st) {
  GbArgs A{};
  A.nrows = nrows;
  A.nu = G.nu;
  A.a = G.a;
  A.b = G.b;
  A.nl = nl;
  A.nr = nr;
  for (int l = 0; l < nl; ++l) A.lu[l] = G.lu[l];
  for (int l = 0; l <= nl; ++l) A.lcum[l] = G.lcum[l];
  for (int r = 0; r < nr; ++r) A.ru[r] = G.ru[r];
  for (int r = 0; r <= nr; ++r) A.rcum[r] = G.rcum[r];
  A.rw_mask = rw_mask;
  A.d = rw_mask ? d : nullptr;
  // needed 4x4 tile blocks
  const int bI = (G.NI + GB_TI - 1) / GB_TI, bJ = (G.NJ + GB_TJ - 1) / GB_TJ;
  for (int bi = 0; bi < bI; ++bi)
    for (int bj = 0; bj < bJ; ++bj) {
      unsigned msk = 0;
      for (int i = 0; i < GB_TI; ++i)
        for (int j = 0; j < GB_TJ; ++j) {
          const int ti = GB_TI * bi + i, tj = GB_TJ * bj + j;
          if (ti < G.NI && tj < G.NJ) {
            const int t = ti * G.NJ + tj;
            if ((G.tmask[t >> 5] >> (t & 31)) & 1u) msk |= 1u << (i * GB_TJ + j);
          }
        }
      const unsigned short code = (unsigned short)(((GB_TI * bi) << 8) | (GB_TJ * bj));
      if (msk) {
        if (A.nblk >= GB_MAXBLK) return 1;
        A.blk[A.nblk] = code;
        A.bmask[A.nblk++] = (unsigned short)msk;
      } else {
        if (A.nzero >= GB_MAXBLK) return 1;
        A.zblk[A.nzero++] = code;
      }
    }
  // CTA groups: a warp's DMMAs issue on its SM sub-partition, so an SM's
  // pass over one row chunk takes ceil(wpc / 4) warp-rounds; choose the
  // split that minimises rounds x chunks per CTA (e.g. 30 tile blocks: 4
  // groups of 8 warps, not 3 of 10)
  const int nchunks_est = (nrows + 31) / 32;
  int gy = (A.nblk + GB_MAXW - 1) / GB_MAXW;
  {
    long best = -1;
    for (int g = gy; g <= A.nblk && g <= sm_count(); ++g) {
      const int w = (A.nblk + g - 1) / g;
      const int gxg = sm_count() / g;
      const long cost = (long)((w + 3) / 4) * ((nchunks_est + gxg - 1) / gxg);
      if (best < 0 || cost * 50 < best * 49) {   // more groups = more L2 re-reads: need 2%
        best = cost;
        gy = g;
      }
    }
  }
  A.wpc = (A.nblk + gy - 1) / gy;
  // few tile blocks per group (e.g. the drift Gram X^T B X: 3): split each
  // chunk's rows over ks warps per block so every sub-partition has DMMA
  // work; the ks partials are summed by the fixed-order second stage
  A.ks = A.wpc * 4 <= GB_MAXW ? 4 : 1;
  if (const char* e = getenv("B2L_GB_KS")) {
    const int v = atoi(e);
    if ((v == 1 || v == 4) && A.wpc * v <= GB_MAXW) A.ks = v;
  }
  A.nwc = A.wpc * A.ks;
  // stage: padded rows of every distinct block (+ the weights)
  int width = 0;
  for (int u = 0; u < A.nu; ++u) {
    A.ustr[u] = smem_stride(G.uld[u]);
    width += A.ustr[u];
  }
  // the longest row chunk whose 3-stage ring fits in shared memory (longer
  // chunks = fewer ring hand-offs per DMMA; B2L_GB_RC overrides for sweeps)
  constexpr size_t kRing = 222 * 1024;
  A.rc = 64;
  while (A.rc > 8 && (size_t)A.rc * (width + 16) * 8 * 3 > kRing) A.rc >>= 1;
  if (const char* e = getenv("B2L_GB_RC")) {
    const int v = atoi(e);
    if (v == 8 || v == 16 || v == 32 || v == 64) A.rc = v;
  }
  int off = 0;
  A.stage_tx = 0;
  for (int u = 0; u < A.nu; ++u) {
    A.ubase[u] = off;
    off += (A.rc * A.ustr[u] + 15) & ~15;
    A.stage_tx += (uint32_t)(A.rc * A.ustr[u] * 8);
  }
  A.dbase = off;
  off += A.d ? ((A.rc + 15) & ~15) : 0;
  A.stage_doubles = off;
  A.nst = (size_t)off * 8 * 3 <= kRing ? 3 : 2;
  const size_t smem = (size_t)A.nst * off * 8 + 128;
  if (smem > 227 * 1024) return 1;
  GbMaps Mp;
  for (int u = 0; u < A.nu; ++u)
    if (int rc = encode_tmap_2d(&Mp.u[u], G.up[u], G.uld[u], nrows, A.ustr[u], A.rc)) return rc;
  const int threads = 32 * (A.nwc + 1);
  int per_sm = 1;
  const void* kfn = A.ks == 4 ? reinterpret_cast<const void*>(gram_big_kernel<4>)
                               : reinterpret_cast<const void*>(gram_big_kernel<1>);
  if (int rc = prepare_kernel(kfn, smem, threads,
                              &per_sm))
    return rc;
  const int nchunks = (nrows + A.rc - 1) / A.rc;
  int gx = (sm_count() * per_sm) / gy;
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  int werr = 0;
  double* part =
      static_cast<double*>(workspace((size_t)gx * A.ks * A.a * A.b * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  if (A.ks == 4)
    gram_big_kernel<4><<<dim3(gx, gy), threads, smem, st>>>(Mp, A);
  else
    gram_big_kernel<1><<<dim3(gx, gy), threads, smem, st>>>(Mp, A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return sum_parts(part, gx * A.ks, A.a * A.b, out, st);
}

// pair_mode[l*nr + r]: 0 = block pair not needed, 1 = full, 2 = upper
// triangle only (a symmetric diagonal pair).  nullptr = all full.
int gram(int nrows, const HostBlock* L, int nl, const HostBlock* R, int nr,
         unsigned rw_mask, const double* d, const unsigned char* pair_mode,
         double* out, cudaStream_t st) {
  B2L_CHECK(nl >= 1 && nl <= GRAM_MAXL && nr >= 1 && nr <= GRAM_MAXR, -B2L_EINVAL,
            "gram: 1..4 left and 1..8 right blocks");
  B2L_CHECK(nrows >= 0, -B2L_EINVAL, "gram: negative row count");
  B2L_CHECK(!rw_mask || d != nullptr, -B2L_EINVAL, "gram: weight mask without weights");
  GramArgs A{};
  A.nrows = nrows;
  A.nl = nl;
  A.nr = nr;
  auto uid = [&](const HostBlock& b) -> int {
    for (int u = 0; u < A.nu; ++u)
      if (A.up[u] == b.p && A.uld[u] == b.ld) return u;
    if (A.nu >= GRAM_MAXU) return -1;
    A.up[A.nu] = b.p;
    A.uld[A.nu] = b.ld;
    return A.nu++;
  };
  A.lcum[0] = 0;
  for (int l = 0; l < nl; ++l) {
    B2L_CHECK(L[l].ld >= 2 && (L[l].ld & 1) == 0 && L[l].cols <= L[l].ld && L[l].cols >= 0,
              -B2L_EINVAL, "gram: left block needs even ld >= cols");
    B2L_CHECK((reinterpret_cast<uintptr_t>(L[l].p) & 15) == 0, -B2L_EINVAL,
              "gram: blocks must be 16-B aligned");
    const int u = uid(L[l]);
    B2L_CHECK(u >= 0, -B2L_EINVAL, "gram: too many distinct blocks");
    A.lu[l] = u;
    A.lcum[l + 1] = A.lcum[l] + L[l].cols;
  }
  A.rcum[0] = 0;
  for (int r = 0; r < nr; ++r) {
    B2L_CHECK(R[r].ld >= 2 && (R[r].ld & 1) == 0 && R[r].cols <= R[r].ld && R[r].cols >= 0,
              -B2L_EINVAL, "gram: right block needs even ld >= cols");
    B2L_CHECK((reinterpret_cast<uintptr_t>(R[r].p) & 15) == 0, -B2L_EINVAL,
              "gram: blocks must be 16-B aligned");
    const int u = uid(R[r]);
    B2L_CHECK(u >= 0, -B2L_EINVAL, "gram: too many distinct blocks");
    A.ru[r] = u;
    A.rcum[r + 1] = A.rcum[r] + R[r].cols;
  }
  A.a = A.lcum[nl];
  A.b = A.rcum[nr];
  A.rw_mask = rw_mask;
  A.d = rw_mask ? d : nullptr;
  if (A.a * A.b == 0) return 0;
  A.NI = (A.a + 7) / 8;
  A.NJ = (A.b + 7) / 8;
  B2L_CHECK(A.NI * A.NJ <= 32 * 32, -B2L_EINVAL, "gram: output too large (max 1024 8x8 tiles)");
  // needed tiles from the block-pair modes
  for (int ti = 0; ti < A.NI; ++ti)
    for (int tj = 0; tj < A.NJ; ++tj) {
      bool need = false;
      for (int l = 0; l < nl && !need; ++l)
        for (int r = 0; r < nr && !need; ++r) {
          const int mode = pair_mode ? pair_mode[l * nr + r] : 1;
          if (!mode) continue;
          const int i0 = max(8 * ti, A.lcum[l]), i1 = min(8 * ti + 8, A.lcum[l + 1]);
          const int j0 = max(8 * tj, A.rcum[r]), j1 = min(8 * tj + 8, A.rcum[r + 1]);
          if (i0 >= i1 || j0 >= j1) continue;
          if (mode == 2) {
            // upper triangle of the pair: local row <= local col somewhere
            const int li0 = i0 - A.lcum[l];
            const int lj1 = j1 - A.rcum[r];
            if (li0 > lj1 - 1) continue;
          }
          need = true;
        }
      if (need) {
        const int t = ti * A.NJ + tj;
        A.tmask[t >> 5] |= 1u << (t & 31);
      }
    }
  // large Grams (> 96 needed 8x8 tiles, e.g. the m = 64 pencil): 4x4 tile
  // blocks per warp, TMA ring, producer warp (gram_big)
  {
    int need = 0;
    for (int t = 0; t < A.NI * A.NJ; ++t) need += (A.tmask[t >> 5] >> (t & 31)) & 1u;
    static const bool small_only = [] {
      const char* v = getenv("B2L_GRAM_SMALL");
      return v && v[0] == '1';
    }();
    // ... and any Gram over wide blocks (ld >= 32): the small kernel stages
    // dense rows, whose 8-B fragment loads then fall on a few banks
    int maxld = 0;
    for (int u = 0; u < A.nu; ++u) maxld = A.uld[u] > maxld ? A.uld[u] : maxld;
    if ((need > 96 || maxld >= 32) && nrows > 0 && !small_only) {
      const int rc = gram_big(nrows, L, nl, R, nr, rw_mask, d, A, out, st);
      if (rc != 1) return rc;
    }
  }
  A.tsI = (A.NI + GT_TI - 1) / GT_TI;
  A.tsJ = (A.NJ + GT_TJ - 1) / GT_TJ;
  const int TS = A.tsI * A.tsJ;
  const int warps = GRAM_THREADS / 32;
  if (TS <= warps) {
    A.ts_per_cta = TS;
    A.rs = 1;
    while (A.rs * 2 * TS <= warps) A.rs *= 2;
  } else {
    A.ts_per_cta = warps;
    A.rs = 1;
  }
  const int gy = (TS + A.ts_per_cta - 1) / A.ts_per_cta;
  // rows per chunk: the largest power of two whose stage stays <= ~24 KB, so
  // a 3-deep ring leaves room for the two CTAs per SM the grid assumes
  int width = A.d ? 1 : 0;
  for (int u = 0; u < A.nu; ++u) width += A.uld[u];
  A.rc = 256;
  while (A.rc > 16 && (size_t)A.rc * width * 8 > 24 * 1024) A.rc >>= 1;
  while (A.rs > 1 && A.rc / A.rs < 4) A.rs >>= 1;
  int off = 0;
  for (int u = 0; u < A.nu; ++u) {
    A.ubase[u] = off;
    off += A.rc * A.uld[u];
  }
  A.dbase = off;
  off += A.d ? A.rc : 0;
  A.stage_doubles = (off + 15) & ~15;
  const size_t stage_bytes = (size_t)A.stage_doubles * 8;
  A.nst = stage_bytes * 3 <= 150 * 1024 ? 3 : 2;
  B2L_CHECK(stage_bytes * A.nst <= 200 * 1024, -B2L_EINVAL, "gram: blocks too wide");
  const size_t red_bytes = (size_t)(A.rs > 1 ? A.rs - 1 : 0) * A.ts_per_cta * GT_TI * GT_TJ * 64 * 8;
  size_t smem = stage_bytes * A.nst;
  if (red_bytes > smem) smem = red_bytes;
  smem += 64;  // barriers
  const int nchunks = (nrows + A.rc - 1) / A.rc;
  int gx = (2 * sm_count() + gy - 1) / gy;
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  int werr = 0;
  double* part = static_cast<double*>(workspace((size_t)gx * A.a * A.b * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  if (nrows == 0) {
    B2L_CUDA(cudaMemsetAsync(out, 0, (size_t)A.a * A.b * sizeof(double), st));
    return 0;
  }
  // the barrier block sits right after the stages / reduction area
  // (kernel indexes it from nst*stage_doubles; keep the reduction inside)
  if (red_bytes > stage_bytes * A.nst) {
    A.stage_doubles = (int)((red_bytes / 8 + A.nst - 1) / A.nst + 15) & ~15;
    smem = (size_t)A.stage_doubles * 8 * A.nst + 64;
  }
  B2L_CUDA(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  gram_kernel<<<dim3(gx, gy), GRAM_THREADS, smem, st>>>(A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  const int tot = A.a * A.b;
  return sum_parts(part, gx, tot, out, st);
}

// =========================================================================
// K4+K2: residual, preconditioner, column norms
// =========================================================================
struct ResidArgs {
  int nrows, m, rp;        // rp = rows per pass = blockDim / m
  const double* x;
  const double* ax;
  int ldx;
  const double* d;         // diag(B) or null
  const double* lam;       // (m)
  int tmode;               // 0 none, 1 scalar, 2 vector
  double tinv;
  const double* tvec;
  const int* pos;          // (m) column -> W column or -1
  int kw;
  double* w;
  int ldw;
  int want_ax;
  double* partial;         // [grid][2m]
};

__global__ void __launch_bounds__(256) resid_kernel(ResidArgs A) {
  extern __shared__ double rsm[];
  const int tid = threadIdx.x;
  const int rr = tid / A.m;
  const int j = tid - rr * A.m;
  const bool on = rr < A.rp;
  double s_w = 0.0, s_a = 0.0;
  if (on) {
    const double lam = A.lam[j];
    const int p = A.pos ? A.pos[j] : -1;
    const bool padw = (p == A.kw - 1) && (A.ldw > A.kw);
    // four rows per thread in flight: all loads of a group are issued before
    // its W stores (which may alias nothing, but the compiler cannot know);
    // the norm chains still run over the rows in the original order
    constexpr int U = 4;
    const int stride = gridDim.x * A.rp;
    for (int r0 = blockIdx.x * A.rp + rr; r0 < A.nrows; r0 += U * stride) {
      double xv[U], av[U], dv[U], tvv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * stride;
        const bool ok = r < A.nrows;
        xv[u] = ok ? A.x[(size_t)r * A.ldx + j] : 0.0;
        av[u] = ok ? A.ax[(size_t)r * A.ldx + j] : 0.0;
        dv[u] = (ok && A.d) ? A.d[r] : 1.0;
        tvv[u] = (ok && A.tmode == 2) ? A.tvec[r] : 1.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * stride;
        if (r >= A.nrows) break;
        const double bx = A.d ? __dmul_rn(dv[u], xv[u]) : xv[u];
        const double wf = __dsub_rn(av[u], __dmul_rn(bx, lam));
        s_w = fma(wf, wf, s_w);
        if (A.want_ax) s_a = fma(av[u], av[u], s_a);
        if (p >= 0) {
          double tv = wf;
          if (A.tmode == 1) tv = __dmul_rn(A.tinv, wf);
          else if (A.tmode == 2) tv = __dmul_rn(tvv[u], wf);
          A.w[(size_t)r * A.ldw + p] = tv;
          if (padw) A.w[(size_t)r * A.ldw + A.kw] = 0.0;
        }
      }
    }
  }
  // fixed-order CTA reduction over the rp row lanes of each column
  if (on) {
    rsm[rr * A.m + j] = s_w;
    rsm[(A.rp + rr) * A.m + j] = s_a;
  }
  __syncthreads();
  if (tid < A.m) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < A.rp; ++q) {
      a += rsm[q * A.m + tid];
      b += rsm[(A.rp + q) * A.m + tid];
    }
    A.partial[(size_t)blockIdx.x * 2 * A.m + tid] = a;
    A.partial[(size_t)blockIdx.x * 2 * A.m + A.m + tid] = b;
  }
}

// out[e] = sum_c partial[c][e].  A 32 x 32 block per 32 outputs: column
// lane x, part slice y (parts y, y+32, ...; four independent chains), then a
// fixed-order sum of the 32 slices -- deterministic, and latency bound on
// nparts/128 dependent loads instead of nparts.
__global__ void __launch_bounds__(1024) sum_parts_kernel(const double* partial, int nparts,
                                                         int len, double* out) {
  __shared__ double red[32][33];
  const int e = blockIdx.x * 32 + threadIdx.x;
  const int y = threadIdx.y;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (e < len) {
    int c = y;
    for (; c + 96 < nparts; c += 128) {
      s0 += partial[(size_t)c * len + e];
      s1 += partial[(size_t)(c + 32) * len + e];
      s2 += partial[(size_t)(c + 64) * len + e];
      s3 += partial[(size_t)(c + 96) * len + e];
    }
    for (; c < nparts; c += 32) s0 += partial[(size_t)c * len + e];
  }
  red[y][threadIdx.x] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (y == 0 && e < len) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += red[k][threadIdx.x];
    out[e] = s;
  }
}

int sum_parts(const double* partial, int nparts, int len, double* out, cudaStream_t st) {
  if (len <= 0) return 0;
  sum_parts_kernel<<<(len + 31) / 32, dim3(32, 32), 0, st>>>(partial, nparts, len, out);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}

int residual(int nrows, int m, const double* x, const double* ax, int ldx,
             const double* d, const double* lam, int tmode, double tinv,
             const double* tvec, const int* pos, int kw, double* w, int ldw,
             int want_ax, double* sums_out, cudaStream_t st) {
  B2L_CHECK(m >= 1 && m <= 256, -B2L_EINVAL, "residual: 1 <= m <= 256");
  B2L_CHECK(ldx >= m, -B2L_EINVAL, "residual: ldx < m");
  B2L_CHECK(kw == 0 || (w != nullptr && ldw >= kw), -B2L_EINVAL, "residual: bad W");
  ResidArgs A{};
  A.nrows = nrows;
  A.m = m;
  A.rp = 256 / m;
  A.x = x;
  A.ax = ax;
  A.ldx = ldx;
  A.d = d;
  A.lam = lam;
  A.tmode = tmode;
  A.tinv = tinv;
  A.tvec = tvec;
  A.pos = pos;
  A.kw = kw;
  A.w = w;
  A.ldw = ldw;
  A.want_ax = want_ax;
  int blocks = (nrows + A.rp - 1) / A.rp;
  const int cap = 4 * sm_count();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  int werr = 0;
  double* part = static_cast<double*>(workspace((size_t)blocks * 2 * m * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  const size_t smem = (size_t)2 * A.rp * m * sizeof(double);
  resid_kernel<<<blocks, 256, smem, st>>>(A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return sum_parts(part, blocks, 2 * m, sums_out, st);
}

// =========================================================================
// K6: block update  P' = W Cw + P_J Cp ; X' = X Cx (+ P') ; A-side twins
// =========================================================================
struct UpdArgs {
  int nrows, m, rp;
  const double* x;
  const double* ax;
  int ldx;
  const double* w;
  const double* aw;
  int ldw, kw;
  const double* p;
  const double* ap;
  int ldp, kp;
  const double* cx;  // m x m
  const double* cw;  // kw x m
  const double* cp;  // kp x m
  const int* pcols;  // kp
  double* xo;
  double* axo;
  int ldo;
  double* po;
  double* apo;
  int ldpo;
  int x_plus_p;
};

__global__ void __launch_bounds__(256) update_kernel(UpdArgs A) {
  extern __shared__ double usm[];
  double* scx = usm;
  double* scw = scx + A.m * A.m;
  double* scp = scw + A.kw * A.m;
  int* spc = reinterpret_cast<int*>(scp + A.kp * A.m);
  const int tid = threadIdx.x;
  if (A.x)
    for (int i = tid; i < A.m * A.m; i += blockDim.x) scx[i] = A.cx[i];
  for (int i = tid; i < A.kw * A.m; i += blockDim.x) scw[i] = A.cw[i];
  for (int i = tid; i < A.kp * A.m; i += blockDim.x) scp[i] = A.cp[i];
  for (int i = tid; i < A.kp; i += blockDim.x) spc[i] = A.pcols[i];
  __syncthreads();
  const int rr = tid / A.m;
  const int c = tid - rr * A.m;
  if (rr >= A.rp) return;
  const bool haveP = (A.kw + A.kp) > 0;
  const bool padx = (c == A.m - 1) && (A.ldo > A.m);
  const bool padp = (c == A.m - 1) && (A.ldpo > A.m);
  for (int r = blockIdx.x * A.rp + rr; r < A.nrows; r += gridDim.x * A.rp) {
    // ---- B/X side
    double pn = 0.0;
    if (haveP) {
      double pw = 0.0, pp = 0.0;
      const double* wr = A.w + (size_t)r * A.ldw;
      for (int i = 0; i < A.kw; ++i) pw = fma(wr[i], scw[i * A.m + c], pw);
      const double* prow = A.p + (size_t)r * A.ldp;
      for (int q = 0; q < A.kp; ++q) pp = fma(prow[spc[q]], scp[q * A.m + c], pp);
      pn = (A.kw && A.kp) ? __dadd_rn(pw, pp) : (A.kw ? pw : pp);
      if (A.po) {
        A.po[(size_t)r * A.ldpo + c] = pn;
        if (padp)
          for (int e = A.m; e < A.ldpo; ++e) A.po[(size_t)r * A.ldpo + e] = 0.0;
      }
    }
    {
      double xs = 0.0;
      if (A.x) {
        const double* xr = A.x + (size_t)r * A.ldx;
        for (int i = 0; i < A.m; ++i) xs = fma(xr[i], scx[i * A.m + c], xs);
        if (A.x_plus_p) xs = __dadd_rn(xs, pn);
      } else {
        xs = pn;   // no X term: X' = P'
      }
      A.xo[(size_t)r * A.ldo + c] = xs;
      if (padx)
        for (int e = A.m; e < A.ldo; ++e) A.xo[(size_t)r * A.ldo + e] = 0.0;
    }
    // ---- A side
    if (A.ax) {
      double apn = 0.0;
      if (haveP) {
        double pw = 0.0, pp = 0.0;
        const double* wr = A.aw + (size_t)r * A.ldw;
        for (int i = 0; i < A.kw; ++i) pw = fma(wr[i], scw[i * A.m + c], pw);
        const double* prow = A.ap + (size_t)r * A.ldp;
        for (int q = 0; q < A.kp; ++q) pp = fma(prow[spc[q]], scp[q * A.m + c], pp);
        apn = (A.kw && A.kp) ? __dadd_rn(pw, pp) : (A.kw ? pw : pp);
        if (A.apo) {
          A.apo[(size_t)r * A.ldpo + c] = apn;
          if (padp)
            for (int e = A.m; e < A.ldpo; ++e) A.apo[(size_t)r * A.ldpo + e] = 0.0;
        }
      }
      double xs = 0.0;
      const double* xr = A.ax + (size_t)r * A.ldx;
      for (int i = 0; i < A.m; ++i) xs = fma(xr[i], scx[i * A.m + c], xs);
      if (A.x_plus_p) xs = __dadd_rn(xs, apn);
      A.axo[(size_t)r * A.ldo + c] = xs;
      if (padx)
        for (int e = A.m; e < A.ldo; ++e) A.axo[(size_t)r * A.ldo + e] = 0.0;
    }
  }
}


// -------------------------------------------------------------------------
// K6 for large blocks (16 < m <= 64): the same products on the fp64 tensor
// cores.  Out (rows x m) = In (rows x K) C (K x m) is a tall-skinny GEMM
// whose C is tiny and shared by every row: the coefficients sit in shared
// memory for the whole kernel, row chunks of the six input blocks stream
// through a TMA double buffer (one producer warp), and compute warp j owns
// output columns 8j..8j+7 of every chunk (DMMA m8n8k4: A = 8 data rows x 4,
// B = 4 coefficient rows x 8).  P_J Cp is formed as P Cp^ with Cp^ the m x m
// scatter of Cp's rows to the pcols positions (zero rows elsewhere), so the
// column gather needs no data movement.  Shared rows are padded to
// smem_stride(ld) (TMA out-of-bounds columns read as zero): conflict-free
// fragment loads.  Reference: lobpcg.py:520-540, multivec.multiply :74-86.
constexpr int UM_R = 16;                     // rows per chunk (two 8-row tiles)
constexpr int UM_NW = 8;                     // compute warps = 64 / 8 column tiles
constexpr int UM_THREADS = 32 * (UM_NW + 1);
constexpr int UM_NST = 2;
constexpr int UM_CS = 68;                    // coefficient row stride (smem_stride(64))

struct UmArgs {
  int nrows, m, kw, kp;
  int kx4, kw4, kp4;                         // K extents rounded up to 4
  int sx, sw, sp;                            // shared row strides of X-, W-, P-like blocks
  int ldo, ldpo;
  int x_plus_p, has_x, has_ax, has_p_out, has_ap_out;
  int in_off[6];                             // X AX W AW P AP, doubles within a stage
  int stage_doubles;
  uint32_t stage_tx;
  int coef_off;                              // Cx | Cw | Cp^ (doubles)
  int bar_off;
  const double* cx;
  const double* cw;
  const double* cp;
  const int* pcols;
  double* xo;
  double* axo;
  double* po;
  double* apo;
};
struct UmMaps {
  CUtensorMap in[6];
};

__global__ void __launch_bounds__(UM_THREADS, 1)
    update_mma_kernel(const __grid_constant__ UmMaps M, const __grid_constant__ UmArgs A) {
  extern __shared__ __align__(128) unsigned char um_raw[];
  double* sm = reinterpret_cast<double*>(um_raw);
  double* Cx = sm + A.coef_off;
  double* Cw = Cx + A.kx4 * UM_CS;
  double* Cp = Cw + A.kw4 * UM_CS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + A.bar_off);
  uint64_t* empty = full + UM_NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = A.m;
  for (int i = tid; i < A.kx4 * UM_CS; i += blockDim.x) {
    const int k = i / UM_CS, c = i - k * UM_CS;
    Cx[i] = (A.has_x && k < m && c < m) ? A.cx[k * m + c] : 0.0;
  }
  for (int i = tid; i < A.kw4 * UM_CS; i += blockDim.x) {
    const int k = i / UM_CS, c = i - k * UM_CS;
    Cw[i] = (k < A.kw && c < m) ? A.cw[k * m + c] : 0.0;
  }
  for (int i = tid; i < A.kp4 * UM_CS; i += blockDim.x) {
    const int k = i / UM_CS, c = i - k * UM_CS;
    double v = 0.0;
    if (c < m)
      for (int q = 0; q < A.kp; ++q)
        if (A.pcols[q] == k) v = A.cp[q * m + c];
    Cp[i] = v;
  }
  if (tid == 0) {
    for (int s = 0; s < UM_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], UM_NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = (A.nrows + UM_R - 1) / UM_R;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool on[6] = {A.has_x != 0, A.has_ax != 0, A.kw > 0, A.kw > 0 && A.has_ax != 0,
                      A.kp > 0, A.kp > 0 && A.has_ax != 0};

  if (warp == UM_NW) {
    // ---- producer
    if (lane == 0)
      for (int it = 0; it < nloc; ++it) {
        const int s = it % UM_NST;
        if (it >= UM_NST) mbar_wait(&empty[s], (it / UM_NST - 1) & 1);
        double* st = sm + (size_t)s * A.stage_doubles;
        const int r0 = (blockIdx.x + it * gridDim.x) * UM_R;
        mbar_expect_tx(&full[s], A.stage_tx);
        for (int b = 0; b < 6; ++b)
          if (on[b]) tma_load_2d(st + A.in_off[b], &M.in[b], &full[s], 0, r0);
      }
    return;
  }

  // ---- compute warp: output column tile j = warp
  const int j = warp;
  const int ra = lane >> 2, qa = lane & 3;        // A fragment: row, k
  const int bk = lane & 3, bn = lane >> 2;        // B fragment: k, column
  const double* cxl = Cx + bk * UM_CS + 8 * j + bn;
  const double* cwl = Cw + bk * UM_CS + 8 * j + bn;
  const double* cpl = Cp + bk * UM_CS + 8 * j + bn;
  const int col = 8 * j + 2 * qa;                 // accumulator columns col, col + 1
  const bool have_pw = A.kw > 0 || A.kp > 0;
  for (int it = 0; it < nloc; ++it) {
    const int s = it % UM_NST;
    mbar_wait(&full[s], (it / UM_NST) & 1);
    const double* st = sm + (size_t)s * A.stage_doubles;
    const double* X = st + A.in_off[0] + ra * A.sx + qa;
    const double* AX = st + A.in_off[1] + ra * A.sx + qa;
    const double* W = st + A.in_off[2] + ra * A.sw + qa;
    const double* AW = st + A.in_off[3] + ra * A.sw + qa;
    const double* P = st + A.in_off[4] + ra * A.sp + qa;
    const double* AP = st + A.in_off[5] + ra * A.sp + qa;
    double pacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, apacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double xacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, axacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const bool hax = A.has_ax != 0;
    for (int k = 0; k < A.kw4; k += 4) {
      const double b = cwl[k * UM_CS];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        dmma_8x8x4(pacc[rt][0], pacc[rt][1], W[8 * rt * A.sw + k], b);
        if (hax) dmma_8x8x4(apacc[rt][0], apacc[rt][1], AW[8 * rt * A.sw + k], b);
      }
    }
    for (int k = 0; k < A.kp4 && A.kp > 0; k += 4) {
      const double b = cpl[k * UM_CS];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        dmma_8x8x4(pacc[rt][0], pacc[rt][1], P[8 * rt * A.sp + k], b);
        if (hax) dmma_8x8x4(apacc[rt][0], apacc[rt][1], AP[8 * rt * A.sp + k], b);
      }
    }
    if (A.has_x)
      for (int k = 0; k < A.kx4; k += 4) {
        const double b = cxl[k * UM_CS];
#pragma unroll
        for (int rt = 0; rt < 2; ++rt) {
          dmma_8x8x4(xacc[rt][0], xacc[rt][1], X[8 * rt * A.sx + k], b);
          if (hax) dmma_8x8x4(axacc[rt][0], axacc[rt][1], AX[8 * rt * A.sx + k], b);
        }
      }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty[s]);
    const int r0 = (blockIdx.x + it * gridDim.x) * UM_R;
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) {
      const int row = r0 + 8 * rt + ra;
      if (row >= A.nrows) continue;
      double xv[2], av[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        xv[e] = !A.has_x ? pacc[rt][e]
                         : (A.x_plus_p && have_pw ? __dadd_rn(xacc[rt][e], pacc[rt][e])
                                                  : xacc[rt][e]);
        av[e] = A.x_plus_p && have_pw ? __dadd_rn(axacc[rt][e], apacc[rt][e]) : axacc[rt][e];
      }
      if (col < A.ldo) {
        *reinterpret_cast<double2*>(A.xo + (size_t)row * A.ldo + col) = make_double2(xv[0], xv[1]);
        if (hax && A.axo)
          *reinterpret_cast<double2*>(A.axo + (size_t)row * A.ldo + col) =
              make_double2(av[0], av[1]);
      }
      if (col < A.ldpo) {
        if (A.has_p_out)
          *reinterpret_cast<double2*>(A.po + (size_t)row * A.ldpo + col) =
              make_double2(pacc[rt][0], pacc[rt][1]);
        if (A.has_ap_out)
          *reinterpret_cast<double2*>(A.apo + (size_t)row * A.ldpo + col) =
              make_double2(apacc[rt][0], apacc[rt][1]);
      }
    }
  }
}


// -------------------------------------------------------------------------
// K6 for small blocks (m <= 16): one thread per row, the row's outputs in
// registers (MT >= m columns), inputs read element by element (L1-cached:
// a warp's 32 rows are contiguous), coefficients broadcast from shared
// memory.  The scalar update_kernel kept one thread per (row, column) and
// re-read the row m times; this is the memory-bound form (repairs, the
// initial block, the exit refresh and the unfused paths at m <= 16).
template <int MT>
__global__ void __launch_bounds__(256) update_row_kernel(UpdArgs A) {
  extern __shared__ double usm[];
  double* scx = usm;
  double* scw = scx + MT * MT;
  double* scp = scw + MT * MT;
  const int tid = threadIdx.x;
  const int m = A.m;
  // zero-padded MT x MT coefficient blocks; Cp rows scattered to pcols
  for (int i = tid; i < 3 * MT * MT; i += blockDim.x) usm[i] = 0.0;
  __syncthreads();
  if (A.x)
    for (int i = tid; i < m * m; i += blockDim.x) scx[(i / m) * MT + i % m] = A.cx[i];
  for (int i = tid; i < A.kw * m; i += blockDim.x) scw[(i / m) * MT + i % m] = A.cw[i];
  for (int i = tid; i < A.kp * m; i += blockDim.x) scp[A.pcols[i / m] * MT + i % m] = A.cp[i];
  __syncthreads();
  const bool haveP = (A.kw + A.kp) > 0;
  for (int r = blockIdx.x * blockDim.x + tid; r < A.nrows; r += gridDim.x * blockDim.x) {
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
      const bool aside = side == 1;
      if (aside && !A.ax) break;
      double pn[MT], xs[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c) pn[c] = xs[c] = 0.0;
      if (haveP) {
        const double* wr = (aside ? A.aw : A.w) + (size_t)r * A.ldw;
        for (int k = 0; k < A.kw; ++k) {
          const double v = wr[k];
#pragma unroll
          for (int c = 0; c < MT; ++c) pn[c] = fma(v, scw[k * MT + c], pn[c]);
        }
        if (A.kp) {
          double pp[MT];
#pragma unroll
          for (int c = 0; c < MT; ++c) pp[c] = 0.0;
          const double* pr = (aside ? A.ap : A.p) + (size_t)r * A.ldp;
          for (int k = 0; k < m; ++k) {
            const double v = pr[k];
#pragma unroll
            for (int c = 0; c < MT; ++c) pp[c] = fma(v, scp[k * MT + c], pp[c]);
          }
#pragma unroll
          for (int c = 0; c < MT; ++c) pn[c] = A.kw ? __dadd_rn(pn[c], pp[c]) : pp[c];
        }
      }
      if (A.x) {
        const double* xr = (aside ? A.ax : A.x) + (size_t)r * A.ldx;
        for (int k = 0; k < m; ++k) {
          const double v = xr[k];
#pragma unroll
          for (int c = 0; c < MT; ++c) xs[c] = fma(v, scx[k * MT + c], xs[c]);
        }
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (A.x_plus_p && haveP) xs[c] = __dadd_rn(xs[c], pn[c]);
      } else {
#pragma unroll
        for (int c = 0; c < MT; ++c) xs[c] = pn[c];
      }
      double* xo = (aside ? A.axo : A.xo) + (size_t)r * A.ldo;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < A.ldo) xo[c] = c < m ? xs[c] : 0.0;
      double* po = aside ? A.apo : A.po;
      if (haveP && po) {
        po += (size_t)r * A.ldpo;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < A.ldpo) po[c] = c < m ? pn[c] : 0.0;
      }
    }
  }
}

static int update_mma(int nrows, int m, const double* x, const double* ax, int ldx,
                      const double* cx, const double* w, const double* aw, int ldw, int kw,
                      const double* cw, const double* p, const double* ap, int ldp,
                      const int* pcols, int kp, const double* cp, double* xo, double* axo,
                      int ldo, double* po, double* apo, int ldpo, int x_plus_p,
                      cudaStream_t st) {
  UmArgs A{};
  A.nrows = nrows;
  A.m = m;
  A.kw = kw;
  A.kp = kp;
  auto r4 = [](int v) { return (v + 3) & ~3; };
  A.kx4 = r4(m);
  A.kw4 = r4(kw);
  A.kp4 = kp ? r4(m) : 0;
  A.sx = smem_stride(ldx > 0 ? ldx : 2);
  A.sw = smem_stride(kw ? ldw : 2);
  A.sp = smem_stride(kp ? ldp : 2);
  A.ldo = ldo;
  A.ldpo = ldpo;
  A.x_plus_p = x_plus_p;
  A.has_x = x != nullptr;
  A.has_ax = ax != nullptr;
  A.has_p_out = po != nullptr;
  A.has_ap_out = apo != nullptr && ax != nullptr;
  A.cx = cx;
  A.cw = cw;
  A.cp = cp;
  A.pcols = pcols;
  A.xo = xo;
  A.axo = axo;
  A.po = po;
  A.apo = apo;
  const int sin_[6] = {A.sx, A.sx, A.sw, A.sw, A.sp, A.sp};
  const bool on[6] = {x != nullptr, ax != nullptr, kw > 0, kw > 0 && ax != nullptr, kp > 0,
                      kp > 0 && ax != nullptr};
  int off = 0;
  A.stage_tx = 0;
  for (int b = 0; b < 6; ++b) {
    A.in_off[b] = off;
    if (on[b]) {
      off += ((UM_R * sin_[b]) + 15) & ~15;
      A.stage_tx += (uint32_t)(UM_R * sin_[b] * 8);
    }
  }
  A.stage_doubles = off;
  off *= UM_NST;
  A.coef_off = off;
  off += (A.kx4 + A.kw4 + A.kp4) * UM_CS;
  off = (off + 15) & ~15;
  A.bar_off = off;
  off += 2 * UM_NST;
  const size_t smem = (size_t)off * 8 + 64;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "update: block too large for the MMA kernel");
  UmMaps M;
  const double* ins[6] = {x, ax, w, aw, p, ap};
  const int lds[6] = {ldx, ldx, ldw, ldw, ldp, ldp};
  for (int b = 0; b < 6; ++b) {
    if (!on[b]) {
      M.in[b] = M.in[0];
      continue;
    }
    if (int rc = encode_tmap_2d(&M.in[b], ins[b], lds[b], nrows, sin_[b], UM_R)) return rc;
  }
  if (int rc = prepare_kernel(reinterpret_cast<const void*>(update_mma_kernel), smem, UM_THREADS,
                              nullptr))
    return rc;
  const int nchunks = (nrows + UM_R - 1) / UM_R;
  int grid = sm_count();
  if (grid > nchunks) grid = nchunks;
  update_mma_kernel<<<grid, UM_THREADS, smem, st>>>(M, A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}

int update(int nrows, int m, const double* x, const double* ax, int ldx,
           const double* cx, const double* w, const double* aw, int ldw, int kw,
           const double* cw, const double* p, const double* ap, int ldp,
           const int* pcols, int kp, const double* cp, double* xo, double* axo,
           int ldo, double* po, double* apo, int ldpo, int x_plus_p,
           cudaStream_t st) {
  B2L_CHECK(m >= 1 && m <= 256, -B2L_EINVAL, "update: 1 <= m <= 256");
  B2L_CHECK((!x || ldx >= m) && ldo >= m, -B2L_EINVAL, "update: ld < m");
  B2L_CHECK(kw >= 0 && kp >= 0, -B2L_EINVAL, "update: negative block width");
  B2L_CHECK(!ax || axo, -B2L_EINVAL, "update: A-side input without output");
  B2L_CHECK(x != xo && (!ax || ax != axo), -B2L_EINVAL, "update: in-place not supported");
  B2L_CHECK(x || (!ax && kw + kp > 0), -B2L_EINVAL,
            "update: without x, only X' = W Cw + P Cp (no A side) is defined");
  B2L_CHECK(!x || cx, -B2L_EINVAL, "update: x without cx");
  // 16 < m <= 64 with TMA-compatible (even) leading dimensions: fp64 tensor cores
  static const bool scalar_only = [] {
    const char* v = getenv("B2L_UPDATE_SCALAR");
    return v && v[0] == '1';
  }();
  if (!scalar_only && m > 16 && m <= 64 && (!x || (ldx % 2) == 0) && (kw == 0 || (ldw % 2) == 0) &&
      (kp == 0 || (ldp % 2) == 0) && (ldo % 2) == 0 && (!po || (ldpo % 2) == 0) &&
      (x || !ax))
    return update_mma(nrows, m, x, ax, ldx, cx, w, aw, ldw, kw, cw, p, ap, ldp, pcols, kp, cp, xo,
                      axo, ldo, po, apo, ldpo, x_plus_p, st);
  UpdArgs A{};
  A.nrows = nrows;
  A.m = m;
  A.rp = 256 / m;
  A.x = x;
  A.ax = ax;
  A.ldx = ldx;
  A.w = w;
  A.aw = aw;
  A.ldw = ldw;
  A.kw = kw;
  A.p = p;
  A.ap = ap;
  A.ldp = ldp;
  A.kp = kp;
  A.cx = cx;
  A.cw = cw;
  A.cp = cp;
  A.pcols = pcols;
  A.xo = xo;
  A.axo = axo;
  A.ldo = ldo;
  A.po = po;
  A.apo = apo;
  A.ldpo = ldpo;
  A.x_plus_p = x_plus_p;
  // the row kernel keeps its coefficient blocks as MT x MT tiles: MT must
  // cover the W block's width too (a constraint projection passes kw = the
  // number of constraints, which can exceed m: with m = 2 and six constraints
  // the Cw rows used to run past the 4 x 4 tile and the shared-memory block)
  const int mk = m > kw ? m : kw;
  const int mt_r = mk <= 4 ? 4 : (mk <= 8 ? 8 : (mk <= 10 ? 10 : 16));
  if (mk <= 16 && !scalar_only && ldo <= mt_r && (!po || ldpo <= mt_r)) {
    // one thread per row (memory-bound form); MT = the next of 4 / 8 / 10 / 16
    const int blocks_r = (int)(((size_t)nrows + 255) / 256);
    int grid_r = blocks_r < 8 * sm_count() ? blocks_r : 8 * sm_count();
    if (grid_r < 1) grid_r = 1;
    auto launch = [&](auto mt) {
      constexpr int MT = decltype(mt)::value;
      update_row_kernel<MT><<<grid_r, 256, 3 * MT * MT * sizeof(double), st>>>(A);
      count_launch();
    };
    if (mt_r == 4) launch(std::integral_constant<int, 4>{});
    else if (mt_r == 8) launch(std::integral_constant<int, 8>{});
    else if (mt_r == 10) launch(std::integral_constant<int, 10>{});
    else launch(std::integral_constant<int, 16>{});
    B2L_CUDA(cudaGetLastError());
    return 0;
  }
  const size_t smem = (size_t)(m * m + kw * m + kp * m) * sizeof(double) + kp * sizeof(int) + 16;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "update: coefficients too large");
  int blocks = (nrows + A.rp - 1) / A.rp;
  const int cap = 8 * sm_count();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  B2L_CUDA(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  update_kernel<<<blocks, 256, smem, st>>>(A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace b2l
