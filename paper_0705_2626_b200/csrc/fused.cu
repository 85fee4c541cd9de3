// F1: one fused pass per LOBPCG iteration over the tall blocks (sm_100a).
//
// For a chunk of rows, staged in shared memory by 2-D TMA tile loads:
//   (1) Ritz update (reference lobpcg.py:520-540, multivec.multiply :74-86)
//         P'  = W Cw + P[:, J] Cp        AP' = AW Cw + AP[:, J] Cp
//         X'  = X Cx + P'                AX' = AX Cx + AP'
//       on the fp64 tensor cores (DMMA), with the Cholesky-QR factors of W and
//       P already folded into Cw/Cp (replaces tri_solve_right,
//       multivec.py:125-146);
//   (2) the NEXT iteration's residual block and lock norms
//       (lobpcg.py:429-430, :466-467): W'_J = T (AX' - BX' Lambda'),
//       sum of squares of every residual column (and of AX' for relative tol);
//   (3) every Gram product of the next Rayleigh-Ritz step that does not
//       involve A W' (lobpcg.py:419 drift, :176 W/P orthonormalisation,
//       :328-338 pencil blocks): [X' W' P']^T B [X' W' P'] (upper) and
//       [X' W' P']^T AP', on DMMA.
// X', AX', P', AP', W' are written back with TMA tile stores.  Each row is read
// once and written once per iteration; the only other pass is the stencil
// (stencil.cu), which also produces [X' W']^T A W'.
//
// Three warp-specialised variants (persistent grid, one CTA per SM):
//   step_pair_kernel  (m = 9..10; C2): loader warp (TMA loads into a 4-deep
//       ring; a stage comes back as soon as the update has read it), 7 warp
//       pairs, storer warp (TMA stores of triple-buffered outputs).  Warp 0 of
//       a pair forms columns 0-7 on DMMA, warp 1 the two tail columns on DFMA;
//       after a pair barrier each folds the 8 rows into half the needed Gram
//       tiles.  Output buffers come back through an mbarrier the storer
//       arrives on (compute warps never meet at a CTA-wide barrier).  The
//       full block (every column active) is a compile-time specialisation.
//   step_local_kernel (m <= 8; C1, C4): loader, 8 compute warps (one 8-row
//       tile each: update, residual and the whole Gram in registers), storer;
//       mbarrier hand-offs.
//   step_kernel       (11 <= m <= 16; C3): one producer/storer warp, 4 update
//       warps, 6 Gram warps folding the finished output buffer while the next
//       chunk is updated; named barriers for the double-buffered outputs.
// Input stages: mbarriers full[s] (TMA) / empty[s] (consumers).

// Shared-memory rows are padded to smem_stride(ld) doubles (4 or 12 mod 16):
// the TMA box is wider than the block's row, the extra columns are zero-filled
// on load and clipped on store, and the DMMA fragment loads are free of bank
// conflicts.  Out-of-range rows of the last chunk are zero-filled by the TMA.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "gram_tile.cuh"

#ifndef B2L_STORE_SWZ8   // conflict-free output stores of the m = 8 full-block local kernel
#define B2L_STORE_SWZ8 1
#endif

namespace b2l {

#ifndef B2L_STEP_NU
#define B2L_STEP_NU 4
#endif
#ifndef B2L_STEP_NG
#define B2L_STEP_NG 6
#endif
// 4 update + 6 Gram warps: at m = 16 the Gram (~40 needed 8x8 tiles, 80
// DMMA per 8 rows) outweighs the update (48 DMMA per 8 rows); 8 + 3 left the
// Gram warps 4x more loaded (C3 step 10.2 -> 8.7 ms; 6 + 5, 5 + 6 slower)
constexpr int STEP_NU = B2L_STEP_NU;                        // update warps
constexpr int STEP_NG = B2L_STEP_NG;                        // Gram warps
constexpr int STEP_GI = 2;                                  // Gram items per Gram warp
// (the loader / storer split of the other F1 variants measured slower here:
// C3 step 9.1 ms vs 8.7 ms with one producer warp doing both)
constexpr int STEP_THREADS = 32 * (1 + STEP_NU + STEP_NG);  // 352
constexpr int NB_OFULL = 1;                                 // named barriers 1,2
constexpr int NB_OEMPTY = 3;                                // named barriers 3,4

struct StepMaps {
  CUtensorMap in[6];   // X AX W AW P AP          box (stride, rc)
  CUtensorMap out[5];  // X' AX' P' AP' W'        box (stride, rc)
};

struct StepArgs {
  int nrows, m, ldx;
  int kw, kp, kwn;
  int sx, sw, swn;      // shared-memory row strides (X-like, W, W')
  int ldwn;             // W' leading dimension in HBM (its columns kwn..ldwn-1 are zeroed)
  const double* d;      // diag(B) or null
  const double* tvec;
  const double* coef;   // [Cx m*m | Cw kw*m | Cp kp*m]
  const int* pcols;     // kp
  const int* wpos;      // m
  const double* lam;    // m
  int tmode;
  double tinv;
  int want_ax;
  int xpp;              // 1: X' = X Cx + P' (the update); 0: X' = X Cx (drift repair)
  int rc, nst;
  uint32_t stage_tx;    // TMA bytes per stage (full boxes)
  // shared-memory layout, in doubles
  int in_off[6];
  int d_off, t_off;
  int stage_doubles;
  int out_off[5];       // buffer 0
  int out_stride;       // doubles between the two output buffers
  int coef_off, lam_off, int_off, zero_off;
  int tail_off;         // m = 10 full block: tail-column coefficient table (72 doubles)
  int bar_off, red_off, gred_off;
  // Gram of the next step
  int a, b;
  int lcum[4], rcum[5];
  int NI, NJ, tsI, tsJ, TS, rs;
  unsigned tmask[32];
  double* partial;      // [gridDim.x][2m + a*b]
};

// Coefficients passed by value in the launch (kernel parameter space) instead
// of through an H2D copy: the steady-state driver (b2l_fast_iteration) hands
// its host-side Rayleigh-Ritz output straight to the launch.  Used when
// StepArgs::coef is null.
struct StepCoef {
  double c[3 * 16 * 16];   // [Cx m*m | Cw kw*m | Cp kp*m]
  double lam[16];
  int pcols[16], wpos[16];
};

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void step_issue(const StepMaps& M, const StepArgs& A, double* st,
                                           uint64_t* bar, int c) {
  const int r0 = c * A.rc;
  const int nvalid = min(A.rc, A.nrows - r0);
  const bool on[6] = {true, true, A.kw > 0, A.kw > 0, A.kp > 0, A.kp > 0};
  uint32_t tx = A.stage_tx;
  const bool even = (nvalid % 2) == 0;
  if (A.d) {
    if (even) tx += (uint32_t)nvalid * 8u;
    else
      for (int e = 0; e < nvalid; ++e) st[A.d_off + e] = A.d[r0 + e];
    for (int e = nvalid; e < A.rc; ++e) st[A.d_off + e] = 0.0;  // tail rows feed the Gram
  }
  if (A.tmode == 2) {
    if (even) tx += (uint32_t)nvalid * 8u;
    else
      for (int e = 0; e < nvalid; ++e) st[A.t_off + e] = A.tvec[r0 + e];
    for (int e = nvalid; e < A.rc; ++e) st[A.t_off + e] = 0.0;
  }
  fence_async_smem();
  mbar_expect_tx(bar, tx);
  for (int b = 0; b < 6; ++b)
    if (on[b]) tma_load_2d(st + A.in_off[b], &M.in[b], bar, 0, r0);
  if (A.d && even) bulk_load(st + A.d_off, A.d + r0, (uint32_t)nvalid * 8u, bar);
  if (A.tmode == 2 && even) bulk_load(st + A.t_off, A.tvec + r0, (uint32_t)nvalid * 8u, bar);
}

// NT = ceil(m/8) output column tiles, KS = ceil(m/4) k-steps (kw, kp <= m),
// WGT: B = diag(d) weights the B-Gram blocks.
template <int NT, int KS, bool WGT>
__global__ void __launch_bounds__(STEP_THREADS, 1)
    step_kernel(const __grid_constant__ StepMaps M, const __grid_constant__ StepArgs Ain,
                    const __grid_constant__ StepCoef Cf) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  // The parameters (1.7 KB with the tensor maps) overflow the constant cache
  // when the hot loops re-read fields: keep a shared copy.
  __shared__ StepArgs sA;
  if (threadIdx.x == 0) sA = Ain;
  __syncthreads();
  const StepArgs& A = sA;
  double* sm = reinterpret_cast<double*>(sm_raw);
  const uint32_t sm_base = smem_u32(sm_raw);
  double* stages = sm;
  double* coef = sm + A.coef_off;
  double* slam = sm + A.lam_off;
  int* spc = reinterpret_cast<int*>(sm + A.int_off);
  int* swp = spc + A.kp;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + A.bar_off);
  uint64_t* empty = full + 4;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int m = A.m;
  const int sx = A.sx, sw = A.sw, swn = A.swn;
  const int ncoef = m * m + A.kw * m + A.kp * m;
  const bool inl = A.coef == nullptr;
  for (int i = tid; i < ncoef; i += blockDim.x) coef[i] = inl ? Cf.c[i] : A.coef[i];
  for (int i = tid; i < m; i += blockDim.x) {
    slam[i] = inl ? Cf.lam[i] : A.lam[i];
    swp[i] = inl ? Cf.wpos[i] : A.wpos[i];
  }
  for (int i = tid; i < A.kp; i += blockDim.x) spc[i] = inl ? Cf.pcols[i] : A.pcols[i];
  for (int i = tid; i < 16; i += blockDim.x) sm[A.zero_off + i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], STEP_NU + STEP_NG);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk_of = [&](int it) { return blockIdx.x + it * gridDim.x; };

  double s_w0 = 0.0, s_w1 = 0.0, s_a0 = 0.0, s_a1 = 0.0;  // update warps: norm partials
  double gacc[STEP_GI][2][4][2];                           // Gram warps
#pragma unroll
  for (int u = 0; u < STEP_GI; ++u)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) gacc[u][i][j][0] = gacc[u][i][j][1] = 0.0;
  const int gw = warp - 1 - STEP_NU;

  if (warp == 0) {
    // ================= producer / storer =================
    if (lane == 0)
      for (int j = 0; j < A.nst && j < nloc; ++j)
        step_issue(M, A, stages + (size_t)j * A.stage_doubles, &full[j], chunk_of(j));
    for (int it = 0; it < nloc; ++it) {
      const int b = it & 1;
      nbar_sync(NB_OFULL + b, STEP_THREADS);
      if (lane == 0) {
        const int r0 = chunk_of(it) * A.rc;
        const int ob = b * A.out_stride;
        for (int k = 0; k < 5; ++k) {
          if (k == 4 && A.kwn == 0) continue;
          tma_store_2d(&M.out[k], sm + A.out_off[k] + ob, 0, r0);
        }
        bulk_commit();
        bulk_wait_read<0>();           // release the buffer once read
      }
      __syncwarp();
      nbar_arrive(NB_OEMPTY + b, STEP_THREADS);
      const int jn = it + A.nst;       // refill the stage chunk `it` used
      if (lane == 0 && jn < nloc) {
        const int s = it % A.nst;
        mbar_wait(&empty[s], (it / A.nst) & 1);
        step_issue(M, A, stages + (size_t)s * A.stage_doubles, &full[s], chunk_of(jn));
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();
  } else if (warp <= STEP_NU) {
    // ================= update + residual =================
    const int wu = warp - 1;
    const int q = lane & 3, rl = lane >> 2;
    // coefficient B-fragments for the whole kernel: C[k][cb], k = 4 ks + q
    double cW[NT][KS], cP[NT][KS], cX[NT][KS];
    int pcol[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + q;
      pcol[ks] = k < A.kp ? spc[k] : 0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int cb = 8 * nt + rl;
        const bool cv = cb < m;
        cW[nt][ks] = (cv && k < A.kw) ? coef[m * m + k * m + cb] : 0.0;
        cP[nt][ks] = (cv && k < A.kp) ? coef[m * m + A.kw * m + k * m + cb] : 0.0;
        cX[nt][ks] = (cv && k < m) ? coef[k * m + cb] : 0.0;
      }
    }
    const int RP = m <= 32 ? 32 / m : 1;
    const int rsub = m <= 32 ? lane / m : 0;
    const int j0 = m <= 32 ? lane % m : lane;
    const bool on0 = rsub < RP && j0 < m;
    const bool on1 = m > 32 && lane + 32 < m;
    const double lam0 = on0 ? slam[j0] : 0.0;
    const double lam1 = on1 ? slam[lane + 32] : 0.0;
    const int jpos0 = on0 ? swp[j0] : -1;
    const int jpos1 = on1 ? swp[lane + 32] : -1;
    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst, b = it & 1;
      const int r0 = chunk_of(it) * A.rc;
      const int nvalid = min(A.rc, A.nrows - r0);
      if (it >= 2) nbar_sync(NB_OEMPTY + b, STEP_THREADS);
      mbar_wait(&full[s], (it / A.nst) & 1);
      const double* st = stages + (size_t)s * A.stage_doubles;
      const double* X = st + A.in_off[0];
      const double* AX = st + A.in_off[1];
      const double* W = st + A.in_off[2];
      const double* AW = st + A.in_off[3];
      const double* P = st + A.in_off[4];
      const double* AP = st + A.in_off[5];
      double* O0 = sm + A.out_off[0] + b * A.out_stride;
      double* O1 = sm + A.out_off[1] + b * A.out_stride;
      double* O2 = sm + A.out_off[2] + b * A.out_stride;
      double* O3 = sm + A.out_off[3] + b * A.out_stride;
      double* O4 = sm + A.out_off[4] + b * A.out_stride;
      for (int mt = wu; mt < (A.rc >> 3); mt += STEP_NU) {
        const int r = 8 * mt + rl;
        // six chains x NT column tiles; the A operands of a k-step are
        // loaded once and shared by the column tiles
        double acc[NT][6][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 6; ++c) acc[nt][c][0] = acc[nt][c][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int k = 4 * ks + q;
          const bool kw_ok = k < A.kw, kp_ok = k < A.kp, km_ok = k < m;
          const double wv = kw_ok ? W[r * sw + k] : 0.0;
          const double awv = kw_ok ? AW[r * sw + k] : 0.0;
          const double pv = kp_ok ? P[r * sx + pcol[ks]] : 0.0;
          const double apv = kp_ok ? AP[r * sx + pcol[ks]] : 0.0;
          const double xv = km_ok ? X[r * sx + k] : 0.0;
          const double axv = km_ok ? AX[r * sx + k] : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            dmma_8x8x4(acc[nt][0][0], acc[nt][0][1], wv, cW[nt][ks]);
            dmma_8x8x4(acc[nt][1][0], acc[nt][1][1], awv, cW[nt][ks]);
            dmma_8x8x4(acc[nt][2][0], acc[nt][2][1], pv, cP[nt][ks]);
            dmma_8x8x4(acc[nt][3][0], acc[nt][3][1], apv, cP[nt][ks]);
            dmma_8x8x4(acc[nt][4][0], acc[nt][4][1], xv, cX[nt][ks]);
            dmma_8x8x4(acc[nt][5][0], acc[nt][5][1], axv, cX[nt][ks]);
          }
        }
        const bool bw = A.kw > 0, bp = A.kp > 0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int co = 8 * nt + 2 * q;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // (W Cw) + (P Cp), then (X Cx) + P', as the reference sums them
            const double pn = (bw && bp) ? __dadd_rn(acc[nt][0][e], acc[nt][2][e])
                                         : (bw ? acc[nt][0][e] : acc[nt][2][e]);
            const double apn = (bw && bp) ? __dadd_rn(acc[nt][1][e], acc[nt][3][e])
                                          : (bw ? acc[nt][1][e] : acc[nt][3][e]);
            if (co + e < A.ldx) {
              O0[r * sx + co + e] = A.xpp ? __dadd_rn(acc[nt][4][e], pn) : acc[nt][4][e];
              O1[r * sx + co + e] = A.xpp ? __dadd_rn(acc[nt][5][e], apn) : acc[nt][5][e];
              O2[r * sx + co + e] = pn;
              O3[r * sx + co + e] = apn;
            }
          }
        }
        __syncwarp();
        // residual of the 8 rows: m <= 32 -> lane = (rsub, j), RP rows per
        // instruction; m > 32 -> lane owns columns j, j+32.  A lane's columns
        // are fixed for the whole kernel: its norm partials stay in registers.
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool on = h == 0 ? on0 : on1;
          if (!on) continue;
          const int j = h == 0 ? j0 : lane + 32;
          const double lam = h == 0 ? lam0 : lam1;
          const int jpos = h == 0 ? jpos0 : jpos1;
          double sw_ = 0.0, sa_ = 0.0;
          for (int rr = rsub; rr < 8; rr += RP) {
            const int row = 8 * mt + rr;
            double wv = 0.0;
            if (row < nvalid) {
              const double xv = O0[row * sx + j];
              const double av = O1[row * sx + j];
              const double bx = A.d ? __dmul_rn(st[A.d_off + row], xv) : xv;
              const double wf = __dsub_rn(av, __dmul_rn(bx, lam));
              sw_ = fma(wf, wf, sw_);
              if (A.want_ax) sa_ = fma(av, av, sa_);
              wv = wf;
              if (A.tmode == 1) wv = __dmul_rn(A.tinv, wf);
              else if (A.tmode == 2) wv = __dmul_rn(st[A.t_off + row], wf);
            }
            if (jpos >= 0) O4[row * swn + jpos] = wv;
          }
          if (h == 0) {
            s_w0 += sw_;
            s_a0 += sa_;
          } else {
            s_w1 += sw_;
            s_a1 += sa_;
          }
        }
        // zero W' pad columns kwn..swn-1 of the 8 rows
        const int npad = A.ldwn - A.kwn;
        for (int e = lane; e < 8 * npad; e += 32)
          O4[(8 * mt + e / npad) * swn + A.kwn + e % npad] = 0.0;
      }
      fence_async_smem();   // generic writes -> the TMA store (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      nbar_arrive(NB_OFULL + b, STEP_THREADS);
    }
    // balance the output-buffer barrier: consume the last two phases
    for (int it = (nloc > 2 ? nloc : 2); it < nloc + 2; ++it)
      nbar_sync(NB_OEMPTY + (it & 1), STEP_THREADS);
  } else {
    // ================= Gram of the finished output buffers =================
    // item = (tile block ts, row slice sl); warp gw owns items gw, gw + NG.
    const int Lblk[3] = {0, 4, 2};        // X', W', P' (indices into out_off)
    const int Rblk[4] = {0, 4, 2, 3};     // X', W', P', AP'
    uint32_t aadr[STEP_GI][2], bsadr[STEP_GI][4];  // lane column byte addresses (buffer 0)
    uint32_t astr[STEP_GI][2], bstr[STEP_GI][4];   // byte stride per row
    bool bwt[STEP_GI][4];
    unsigned mask[STEP_GI];
    int lo[STEP_GI], hi_[STEP_GI];
    const int rps = A.rc / A.rs;
    const uint32_t zero_adr = sm_base + (uint32_t)A.zero_off * 8u;
#pragma unroll
    for (int u = 0; u < STEP_GI; ++u) {
      const int item = gw + u * STEP_NG;
      const int ts = item % A.TS, sl = item / A.TS;
      const bool act = sl < A.rs;
      const int ti0 = (ts / A.tsJ) * 2, tj0 = (ts % A.tsJ) * 4;
      lo[u] = sl * rps;
      hi_[u] = lo[u] + rps;
      mask[u] = 0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int ci = 8 * (ti0 + i) + (lane >> 2);
        aadr[u][i] = zero_adr;
        astr[u][i] = 0;
        if (act && ci < A.a) {
          int l = 0;
          while (l + 1 < 3 && A.lcum[l + 1] <= ci) ++l;
          aadr[u][i] = sm_base + 8u * (A.out_off[Lblk[l]] + (ci - A.lcum[l]));
          astr[u][i] = 8u * (l == 1 ? swn : sx);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cj = 8 * (tj0 + j) + (lane >> 2);
        bsadr[u][j] = zero_adr;
        bstr[u][j] = 0;
        bwt[u][j] = false;
        if (act && cj < A.b) {
          int r = 0;
          while (r + 1 < 4 && A.rcum[r + 1] <= cj) ++r;
          bsadr[u][j] = sm_base + 8u * (A.out_off[Rblk[r]] + (cj - A.rcum[r]));
          bstr[u][j] = 8u * (r == 1 ? swn : sx);
          bwt[u][j] = r < 3;
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ti = ti0 + i, tj = tj0 + j;
          if (act && ti < A.NI && tj < A.NJ) {
            const int t = ti * A.NJ + tj;
            if ((A.tmask[t >> 5] >> (t & 31)) & 1u) mask[u] |= 1u << (i * 4 + j);
          }
        }
    }
    const int q = lane & 3;
    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst, b = it & 1;
      const int r0 = chunk_of(it) * A.rc;
      const int nvalid = min(A.rc, A.nrows - r0);
      const int nv4 = (nvalid + 3) & ~3;
      nbar_sync(NB_OFULL + b, STEP_THREADS);
      const uint32_t boff = 8u * (uint32_t)(b * A.out_stride);
      const double* dst_ = stages + (size_t)s * A.stage_doubles + A.d_off;
#pragma unroll
      for (int u = 0; u < STEP_GI; ++u) {
        if (!mask[u]) continue;
        const int h = min(hi_[u], nv4);
        for (int r = lo[u]; r < h; r += 4) {
          const uint32_t row = (uint32_t)(r + q);
          double av[2], bv[4];
#pragma unroll
          for (int i = 0; i < 2; ++i)
            av[i] = lds64(aadr[u][i] + (astr[u][i] ? boff : 0u) + row * astr[u][i]);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            bv[j] = lds64(bsadr[u][j] + (bstr[u][j] ? boff : 0u) + row * bstr[u][j]);
          if (WGT) {
            const double w = dst_[r + q];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (bwt[u][j]) bv[j] = __dmul_rn(w, bv[j]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (mask[u] & (1u << (i * 4 + j)))
                dmma_8x8x4(gacc[u][i][j][0], gacc[u][i][j][1], av[i], bv[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      nbar_arrive(NB_OEMPTY + b, STEP_THREADS);
    }
  }
  __syncthreads();

  // ---- CTA reduction: residual sums, fixed order over (update warp, lane)
  double* red = sm + A.red_off;
  const int NL = STEP_NU * 32;
  if (warp >= 1 && warp <= STEP_NU) {
    const int o = (warp - 1) * 32 + lane;
    red[o] = s_w0;
    red[NL + o] = s_a0;
    red[2 * NL + o] = s_w1;
    red[3 * NL + o] = s_a1;
  }
  __syncthreads();
  double* out = A.partial + (size_t)blockIdx.x * (2 * m + A.a * A.b);
  if (tid < m) {
    double a = 0.0, bb = 0.0;
    const int RP = m <= 32 ? 32 / m : 1;
    for (int qq = 0; qq < STEP_NU; ++qq) {
      if (m <= 32) {
        for (int r_ = 0; r_ < RP; ++r_) {
          a += red[qq * 32 + r_ * m + tid];
          bb += red[NL + qq * 32 + r_ * m + tid];
        }
      } else {
        const int h = tid >= 32;
        a += red[2 * h * NL + qq * 32 + (tid & 31)];
        bb += red[(2 * h + 1) * NL + qq * 32 + (tid & 31)];
      }
    }
    out[tid] = a;
    out[m + tid] = bb;
  }
  __syncthreads();
  // ---- Gram: per item, fixed-order sum over row slices
  double* gred = sm + A.gred_off;  // [item][8 tiles][32 lanes][2]
  if (gw >= 0) {
#pragma unroll
    for (int u = 0; u < STEP_GI; ++u) {
      const int item = gw + u * STEP_NG;
      if (item >= A.TS * A.rs) continue;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        gred[((size_t)item * 8 + t) * 64 + lane * 2] = gacc[u][t >> 2][t & 3][0];
        gred[((size_t)item * 8 + t) * 64 + lane * 2 + 1] = gacc[u][t >> 2][t & 3][1];
      }
    }
  }
  __syncthreads();
  // thread per (tile block, tile, lane): sum the row slices in order
  double* go = out + 2 * m;
  for (int e = tid; e < A.TS * 8 * 32; e += blockDim.x) {
    const int ts = e / 256, t = (e / 32) & 7, ln = e & 31;
    double v0 = 0.0, v1 = 0.0;
    for (int sl = 0; sl < A.rs; ++sl) {
      const int item = sl * A.TS + ts;
      v0 += gred[((size_t)item * 8 + t) * 64 + ln * 2];
      v1 += gred[((size_t)item * 8 + t) * 64 + ln * 2 + 1];
    }
    const int ti0 = (ts / A.tsJ) * 2, tj0 = (ts % A.tsJ) * 4;
    const int row = 8 * (ti0 + (t >> 2)) + (ln >> 2);
    const int col = 8 * (tj0 + (t & 3)) + 2 * (ln & 3);
    if (row < A.a && ti0 + (t >> 2) < A.NI && tj0 + (t & 3) < A.NJ) {
      if (col < A.b) go[(size_t)row * A.b + col] = v0;
      if (col + 1 < A.b) go[(size_t)row * A.b + col + 1] = v1;
    }
  }
}


// Needed 8x8 tiles of a Gram with column segments lcum/rcum and block-pair
// modes (0 skip, 1 full, 2 upper triangle).
void tile_mask(int NI, int NJ, const int* lcum, int nl, const int* rcum, int nr,
               const unsigned char* modes, unsigned* tmask) {
  for (int t = 0; t < 32; ++t) tmask[t] = 0;
  for (int ti = 0; ti < NI; ++ti)
    for (int tj = 0; tj < NJ; ++tj) {
      bool need = false;
      for (int l = 0; l < nl && !need; ++l)
        for (int r = 0; r < nr && !need; ++r) {
          const int mode = modes[l * nr + r];
          if (!mode) continue;
          const int i0 = max(8 * ti, lcum[l]), i1 = min(8 * ti + 8, lcum[l + 1]);
          const int j0 = max(8 * tj, rcum[r]), j1 = min(8 * tj + 8, rcum[r + 1]);
          if (i0 >= i1 || j0 >= j1) continue;
          if (mode == 2 && (i0 - lcum[l]) > (j1 - rcum[r]) - 1) continue;
          need = true;
        }
      if (need) {
        const int t = ti * NJ + tj;
        tmask[t >> 5] |= 1u << (t & 31);
      }
    }
}

// The Gram tiles one warp of a pair owns, as a compile-time list.
// MFIX = 0: the tile block of half h (all NI x NJ tiles split along i when NI
// is even, else along j).  MFIX = m > 0: only the tiles the next step needs
// when kw_next = m (the pair modes {2,1,1,1; 0,2,1,1; 0,0,2,1} of
// b2l_lobpcg_step), split evenly between the halves in row-major order.
struct PairTiles {
  int n;
  int ti[32], tj[32];
  unsigned imask, jmask;          // tile rows / columns used
  unsigned need[2];               // all needed tiles (bit t = i*NJ + j)
};

__host__ __device__ constexpr bool pair_tile_needed(int m, int ti, int tj) {
  const int lcum[4] = {0, m, 2 * m, 3 * m};
  const int rcum[5] = {0, m, 2 * m, 3 * m, 4 * m};
  const int modes[12] = {2, 1, 1, 1, 0, 2, 1, 1, 0, 0, 2, 1};
  for (int l = 0; l < 3; ++l)
    for (int r = 0; r < 4; ++r) {
      const int md = modes[l * 4 + r];
      if (!md) continue;
      const int i0 = (8 * ti > lcum[l]) ? 8 * ti : lcum[l];
      const int i1 = (8 * ti + 8 < lcum[l + 1]) ? 8 * ti + 8 : lcum[l + 1];
      const int j0 = (8 * tj > rcum[r]) ? 8 * tj : rcum[r];
      const int j1 = (8 * tj + 8 < rcum[r + 1]) ? 8 * tj + 8 : rcum[r + 1];
      if (i0 >= i1 || j0 >= j1) continue;
      if (md == 2 && (i0 - lcum[l]) > (j1 - rcum[r]) - 1) continue;
      return true;
    }
  return false;
}

__host__ __device__ constexpr PairTiles pair_tiles(int NI, int NJ, int mfix, int h, int nh = 2,
                                                   int first_h0 = -1) {
  PairTiles T{};
  if (mfix == 0 && nh == 1) {
    for (int i = 0; i < NI; ++i)
      for (int j = 0; j < NJ; ++j) {
        T.ti[T.n] = i;
        T.tj[T.n] = j;
        ++T.n;
      }
  } else if (mfix == 0) {
    const bool split_i = (NI % 2) == 0;
    const int gi = split_i ? NI / 2 : NI, gj = split_i ? NJ : (NJ + 1) / 2;
    const int i0 = split_i ? h * gi : 0, j0 = split_i ? 0 : h * gj;
    for (int i = i0; i < i0 + gi && i < NI; ++i)
      for (int j = j0; j < j0 + gj && j < NJ; ++j) {
        T.ti[T.n] = i;
        T.tj[T.n] = j;
        ++T.n;
      }
  } else {
    int tot = 0;
    for (int i = 0; i < NI; ++i)
      for (int j = 0; j < NJ; ++j)
        if (pair_tile_needed(mfix, i, j)) {
          const int t = i * NJ + j;
          T.need[t >> 5] |= 1u << (t & 31);
          ++tot;
        }
    const int first = nh == 1 ? tot : (first_h0 >= 0 ? first_h0 : (tot + 1) / 2);
    int k = 0;
    for (int i = 0; i < NI; ++i)
      for (int j = 0; j < NJ; ++j)
        if (pair_tile_needed(mfix, i, j)) {
          if ((h == 0 && k < first) || (h == 1 && k >= first)) {
            T.ti[T.n] = i;
            T.tj[T.n] = j;
            ++T.n;
          }
          ++k;
        }
  }
  for (int t = 0; t < T.n; ++t) {
    T.imask |= 1u << T.ti[t];
    T.jmask |= 1u << T.tj[t];
  }
  return T;
}

// ---------------------------------------------------------------------------
// F1, warp-local variant (m <= 10): every compute warp owns 8 rows of a chunk
// and does everything for them -- update, residual, and the Gram over those 8
// rows for all needed tiles, with the whole Gram accumulator (NI x NJ 8x8
// tiles) in its registers.  No hand-off between compute warps at all: the only
// synchronisation is TMA -> warp (full), warp -> producer (empty / buffer
// full) and producer -> warp (buffer empty).  8 warps keep the fp64 tensor
// pipe busy without the load imbalance of a separate Gram warp group.
constexpr int LOC_NW = 8;                        // compute warps (8 x 8 = 64 rows)
constexpr int LOC_THREADS = 32 * (2 + LOC_NW);   // 320: loader + 8 compute + storer

template <int NT, int KS, int NI, int NJ, int MFIX, bool WGT>
__global__ void __launch_bounds__(LOC_THREADS, 1)
    step_local_kernel(const __grid_constant__ StepMaps M, const __grid_constant__ StepArgs Ain,
                    const __grid_constant__ StepCoef Cf) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  __shared__ StepArgs sA;
  if (threadIdx.x == 0) sA = Ain;
  __syncthreads();
  const StepArgs& A = sA;
  double* sm = reinterpret_cast<double*>(sm_raw);
  const uint32_t sm_base = smem_u32(sm_raw);
  double* stages = sm;
  double* coef = sm + A.coef_off;
  double* slam = sm + A.lam_off;
  int* spc = reinterpret_cast<int*>(sm + A.int_off);
  int* swp = spc + A.kp;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + A.bar_off);
  uint64_t* empty = full + 4;
  uint64_t* ofull = full + 8;    // output buffer b written (compute warps arrive)
  uint64_t* oempty = full + 10;  // output buffer b read by its TMA store (storer arrives)

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int m = A.m;
  const int sx = A.sx, sw = A.sw, swn = A.swn;
  // MFIX > 0: the full block (kw = kp = kw_next = m = MFIX, ld = MFIX): every
  // output block has the row stride SF
  constexpr bool FIX = MFIX > 0;
  constexpr int SF = FIX ? smem_stride(MFIX) : 4;
  const int ncoef = m * m + A.kw * m + A.kp * m;
  const bool inl = A.coef == nullptr;
  for (int i = tid; i < ncoef; i += blockDim.x) coef[i] = inl ? Cf.c[i] : A.coef[i];
  for (int i = tid; i < m; i += blockDim.x) {
    slam[i] = inl ? Cf.lam[i] : A.lam[i];
    swp[i] = inl ? Cf.wpos[i] : A.wpos[i];
  }
  for (int i = tid; i < A.kp; i += blockDim.x) spc[i] = inl ? Cf.pcols[i] : A.pcols[i];
  for (int i = tid; i < 16; i += blockDim.x) sm[A.zero_off + i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], LOC_NW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ofull[b], LOC_NW);
      mbar_init(&oempty[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk_of = [&](int it) { return blockIdx.x + it * gridDim.x; };

  double s_w[NT][2], s_a[NT][2];   // per-lane residual-norm partials (columns 8nt + 2q + e)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) s_w[nt][0] = s_w[nt][1] = s_a[nt][0] = s_a[nt][1] = 0.0;
  constexpr PairTiles TL = pair_tiles(NI, NJ, MFIX, 0, 1);
  double gacc[TL.n][2];
#pragma unroll
  for (int t = 0; t < TL.n; ++t) gacc[t][0] = gacc[t][1] = 0.0;

  if (warp == 0) {
    // ================= loader: refills a stage as soon as it is released
    if (lane == 0)
      for (int j = 0; j < nloc; ++j) {
        const int s = j % A.nst;
        if (j >= A.nst) mbar_wait(&empty[s], (j / A.nst - 1) & 1);
        step_issue(M, A, stages + (size_t)s * A.stage_doubles, &full[s], chunk_of(j));
      }
  } else if (warp == LOC_NW + 1) {
    // ================= storer (mbarrier hand-offs: no CTA-wide barrier)
    if (lane == 0) {
      for (int it = 0; it < nloc; ++it) {
        const int b = it & 1;
        mbar_wait(&ofull[b], (it >> 1) & 1);
        const int r0 = chunk_of(it) * A.rc;
        const int ob = b * A.out_stride;
        for (int k = 0; k < 5; ++k) {
          if (k == 4 && A.kwn == 0) continue;
          tma_store_2d(&M.out[k], sm + A.out_off[k] + ob, 0, r0);
        }
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&oempty[b]);
      }
      bulk_wait<0>();
    }
  } else {
    const int mt = warp - 1;                   // this warp's 8-row tile
    const int q = lane & 3, rl = lane >> 2;
    // update coefficients (B fragments) for the whole kernel
    double cW[NT][KS], cP[NT][KS], cX[NT][KS];
    int pcol[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + q;
      pcol[ks] = k < A.kp ? spc[k] : 0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int cb = 8 * nt + rl;
        const bool cv = cb < m;
        cW[nt][ks] = (cv && k < A.kw) ? coef[m * m + k * m + cb] : 0.0;
        cP[nt][ks] = (cv && k < A.kp) ? coef[m * m + A.kw * m + k * m + cb] : 0.0;
        cX[nt][ks] = (cv && k < m) ? coef[k * m + cb] : 0.0;
      }
    }
    // residual columns of this lane: c = 8 nt + 2q + e (fragment layout of C)
    double lamc[NT][2];
    int wposc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * nt + 2 * q + e;
        lamc[nt][e] = c < m ? slam[c] : 0.0;
        wposc[nt][e] = c < m ? swp[c] : -1;
      }
    const bool weighted = A.d != nullptr, want_ax = A.want_ax != 0;
    const int tmode = A.tmode;
    const double tinv = A.tinv;
    const int npad = A.ldwn - A.kwn;
    // Gram lane columns: L = [X' W' P'] (a cols), R = [X' W' P' AP'] (b cols)
    const uint32_t zero_adr = sm_base + (uint32_t)A.zero_off * 8u;
    uint32_t la_[NI], ls_[NI], rb_[NJ], rs_[NJ];
    bool rw_[NJ];
    const int Lblk[3] = {0, 4, 2};
    const int Rblk[4] = {0, 4, 2, 3};
    if constexpr (FIX) {
      // full block: a = 3m rows, b = 4m columns, every block at row stride
      // SF -- compile-time strides; lanes past the last row / column read a
      // valid in-tile address (their entries are never written back)
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int ci0 = 8 * i + (lane >> 2);
        const int ci = ci0 < 3 * MFIX ? ci0 : 0;
        const int l = ci / MFIX;
        la_[i] = sm_base + 8u * (uint32_t)(A.out_off[Lblk[l]] + (ci - l * MFIX));
        ls_[i] = 8u * SF;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int cj0 = 8 * j + (lane >> 2);
        const int cj = cj0 < 4 * MFIX ? cj0 : 0;
        const int r = cj / MFIX;
        rb_[j] = sm_base + 8u * (uint32_t)(A.out_off[Rblk[r]] + (cj - r * MFIX));
        rs_[j] = 8u * SF;
        rw_[j] = r < 3 && cj0 < 4 * MFIX;
      }
    } else {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int ci = 8 * i + (lane >> 2);
      la_[i] = zero_adr;
      ls_[i] = 0;
      if (ci < A.a) {
        int l = 0;
        while (l + 1 < 3 && A.lcum[l + 1] <= ci) ++l;
        la_[i] = sm_base + 8u * (A.out_off[Lblk[l]] + (ci - A.lcum[l]));
        ls_[i] = 8u * (l == 1 ? swn : sx);
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int cj = 8 * j + (lane >> 2);
      rb_[j] = zero_adr;
      rs_[j] = 0;
      rw_[j] = false;
      if (cj < A.b) {
        int r = 0;
        while (r + 1 < 4 && A.rcum[r + 1] <= cj) ++r;
        rb_[j] = sm_base + 8u * (A.out_off[Rblk[r]] + (cj - A.rcum[r]));
        rs_[j] = 8u * (r == 1 ? swn : sx);
        rw_[j] = r < 3;
      }
    }
    }
    unsigned tm[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      tm[i] = 0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int t = i * A.NJ + j;
        if (i < A.NI && j < A.NJ && ((A.tmask[t >> 5] >> (t & 31)) & 1u)) tm[i] |= 1u << j;
      }
    }

    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst, b = it & 1;
      const int r0 = chunk_of(it) * A.rc;
      const int nvalid = min(A.rc, A.nrows - r0);
      if (it >= 2) mbar_wait(&oempty[b], ((it >> 1) - 1) & 1);
      mbar_wait(&full[s], (it / A.nst) & 1);
      const double* st = stages + (size_t)s * A.stage_doubles;
      const double* X = st + A.in_off[0];
      const double* AX = st + A.in_off[1];
      const double* W = st + A.in_off[2];
      const double* AW = st + A.in_off[3];
      const double* P = st + A.in_off[4];
      const double* AP = st + A.in_off[5];
      const int ob = b * A.out_stride;
      double* O0 = sm + A.out_off[0] + ob;
      double* O1 = sm + A.out_off[1] + ob;
      double* O2 = sm + A.out_off[2] + ob;
      double* O3 = sm + A.out_off[3] + ob;
      double* O4 = sm + A.out_off[4] + ob;
      const int r = 8 * mt + rl;
      {
        // ---- (1) update of the 8 rows, all column tiles
        double acc[NT][6][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 6; ++c) acc[nt][c][0] = acc[nt][c][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int k = 4 * ks + q;
          const bool kw_ok = k < A.kw, kp_ok = k < A.kp, km_ok = k < m;
          const double wv = kw_ok ? W[r * sw + k] : 0.0;
          const double awv = kw_ok ? AW[r * sw + k] : 0.0;
          const double pv = kp_ok ? P[r * sx + pcol[ks]] : 0.0;
          const double apv = kp_ok ? AP[r * sx + pcol[ks]] : 0.0;
          const double xv = km_ok ? X[r * sx + k] : 0.0;
          const double axv = km_ok ? AX[r * sx + k] : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            dmma_8x8x4(acc[nt][0][0], acc[nt][0][1], wv, cW[nt][ks]);
            dmma_8x8x4(acc[nt][1][0], acc[nt][1][1], awv, cW[nt][ks]);
            dmma_8x8x4(acc[nt][2][0], acc[nt][2][1], pv, cP[nt][ks]);
            dmma_8x8x4(acc[nt][3][0], acc[nt][3][1], apv, cP[nt][ks]);
            dmma_8x8x4(acc[nt][4][0], acc[nt][4][1], xv, cX[nt][ks]);
            dmma_8x8x4(acc[nt][5][0], acc[nt][5][1], axv, cX[nt][ks]);
          }
        }
        const bool bw = A.kw > 0, bp = A.kp > 0;
        const double dr = weighted ? st[A.d_off + r] : 1.0;
        const double tr = tmode == 2 ? st[A.t_off + r] : tinv;
        // m = 8 full block: the odd rows store their second column first (the
        // conflict-free store order of the pair kernel, see there)
        constexpr bool SWZ = FIX && MFIX == 8 && NT == 1 && B2L_STORE_SWZ8;
        if constexpr (SWZ) {
          double xn_[2], axn_[2], pn_[2], apn_[2], wv_[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            pn_[e] = __dadd_rn(acc[0][0][e], acc[0][2][e]);
            apn_[e] = __dadd_rn(acc[0][1][e], acc[0][3][e]);
            xn_[e] = A.xpp ? __dadd_rn(acc[0][4][e], pn_[e]) : acc[0][4][e];
            axn_[e] = A.xpp ? __dadd_rn(acc[0][5][e], apn_[e]) : acc[0][5][e];
            const double bx = weighted ? __dmul_rn(dr, xn_[e]) : xn_[e];
            const double wf = __dsub_rn(axn_[e], __dmul_rn(bx, lamc[0][e]));
            s_w[0][e] = fma(wf, wf, s_w[0][e]);
            if (want_ax) s_a[0][e] = fma(axn_[e], axn_[e], s_a[0][e]);
            wv_[e] = tmode == 0 ? wf : __dmul_rn(tr, wf);
          }
          const bool odd = rl & 1;
          const int a0 = r * SF + 2 * q + (odd ? 1 : 0), a1 = r * SF + 2 * q + (odd ? 0 : 1);
          O0[a0] = odd ? xn_[1] : xn_[0];
          O1[a0] = odd ? axn_[1] : axn_[0];
          O2[a0] = odd ? pn_[1] : pn_[0];
          O3[a0] = odd ? apn_[1] : apn_[0];
          O4[a0] = odd ? wv_[1] : wv_[0];
          O0[a1] = odd ? xn_[0] : xn_[1];
          O1[a1] = odd ? axn_[0] : axn_[1];
          O2[a1] = odd ? pn_[0] : pn_[1];
          O3[a1] = odd ? apn_[0] : apn_[1];
          O4[a1] = odd ? wv_[0] : wv_[1];
        } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int co = 8 * nt + 2 * q;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double pn = (bw && bp) ? __dadd_rn(acc[nt][0][e], acc[nt][2][e])
                                         : (bw ? acc[nt][0][e] : acc[nt][2][e]);
            const double apn = (bw && bp) ? __dadd_rn(acc[nt][1][e], acc[nt][3][e])
                                          : (bw ? acc[nt][1][e] : acc[nt][3][e]);
            const double xn = A.xpp ? __dadd_rn(acc[nt][4][e], pn) : acc[nt][4][e];
            const double axn = A.xpp ? __dadd_rn(acc[nt][5][e], apn) : acc[nt][5][e];
            if (co + e < A.ldx) {
              O0[r * sx + co + e] = xn;
              O1[r * sx + co + e] = axn;
              O2[r * sx + co + e] = pn;
              O3[r * sx + co + e] = apn;
            }
            if (co + e < m) {
              // ---- (2) W'_j = T (AX'_j - BX'_j lam_j) from the accumulators
              const double bx = weighted ? __dmul_rn(dr, xn) : xn;
              const double wf = __dsub_rn(axn, __dmul_rn(bx, lamc[nt][e]));
              s_w[nt][e] = fma(wf, wf, s_w[nt][e]);
              if (want_ax) s_a[nt][e] = fma(axn, axn, s_a[nt][e]);
              const double wv = tmode == 0 ? wf : __dmul_rn(tr, wf);
              if (wposc[nt][e] >= 0) O4[r * swn + wposc[nt][e]] = wv;
            }
          }
        }
        }
      }
      for (int e = lane; e < 8 * npad; e += 32) {
        const int rr = e / npad;
        O4[(8 * mt + rr) * swn + A.kwn + (e - rr * npad)] = 0.0;
      }
      __syncwarp();
      // ---- (3) Gram over the 8 rows, every needed tile
      const uint32_t boff = 8u * (uint32_t)ob;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t row = (uint32_t)(8 * mt + 4 * ks + q);
        double av[NI], bv[NJ];
#pragma unroll
        for (int i = 0; i < NI; ++i) av[i] = lds64(la_[i] + (ls_[i] ? boff : 0u) + row * ls_[i]);
#pragma unroll
        for (int j = 0; j < NJ; ++j) bv[j] = lds64(rb_[j] + (rs_[j] ? boff : 0u) + row * rs_[j]);
        if (WGT) {
          const double w = st[A.d_off + row];
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (rw_[j]) bv[j] = __dmul_rn(w, bv[j]);
        }
        // compile-time tile list: all tiles, or (MFIX) only the needed ones
#pragma unroll
        for (int t = 0; t < TL.n; ++t)
          dmma_8x8x4(gacc[t][0], gacc[t][1], av[TL.ti[t]], bv[TL.tj[t]]);
      }
      fence_async_smem();   // generic writes -> the TMA store (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        mbar_arrive(&ofull[b]);
      }
    }
  }
  __syncthreads();

  // ---- CTA reductions (fixed order over compute warps / rows)
  double* red = sm + A.red_off;
  const int NL = LOC_NW * 32 * 2 * NT;    // [warp][lane][nt][e]
  if (warp >= 1 && warp <= LOC_NW) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int o = (((warp - 1) * 32 + lane) * NT + nt) * 2 + e;
        red[o] = s_w[nt][e];
        red[NL + o] = s_a[nt][e];
      }
  }
  __syncthreads();
  double* out = A.partial + (size_t)blockIdx.x * (2 * m + A.a * A.b);
  if (tid < m) {
    const int nt = tid >> 3, qq = (tid & 7) >> 1, e = tid & 1;
    double a = 0.0, bb = 0.0;
    for (int w = 0; w < LOC_NW; ++w)
      for (int g = 0; g < 8; ++g) {
        const int o = (((w * 32) + 4 * g + qq) * NT + nt) * 2 + e;
        a += red[o];
        bb += red[NL + o];
      }
    out[tid] = a;
    out[m + tid] = bb;
  }
  double* gred = sm + A.gred_off;   // [warp][NI*NJ tiles][32][2]
  if (warp >= 1 && warp <= LOC_NW) {
#pragma unroll
    for (int t = 0; t < TL.n; ++t) {
      const size_t o =
          (((size_t)(warp - 1) * NI * NJ + TL.ti[t] * NJ + TL.tj[t]) * 32 + lane) * 2;
      gred[o] = gacc[t][0];
      gred[o + 1] = gacc[t][1];
    }
    if (MFIX)
      for (int t = 0; t < NI * NJ; ++t)
        if (!((TL.need[t >> 5] >> (t & 31)) & 1u)) {
          const size_t o = (((size_t)(warp - 1) * NI * NJ + t) * 32 + lane) * 2;
          gred[o] = 0.0;
          gred[o + 1] = 0.0;
        }
  }
  __syncthreads();
  double* go = out + 2 * m;
  for (int e = tid; e < NI * NJ * 32; e += blockDim.x) {
    const int t = e / 32, ln = e & 31;
    const int i = t / NJ, j = t % NJ;
    double v0 = 0.0, v1 = 0.0;
    for (int w = 0; w < LOC_NW; ++w) {
      const size_t o = (((size_t)w * NI * NJ + t) * 32 + ln) * 2;
      v0 += gred[o];
      v1 += gred[o + 1];
    }
    const int row = 8 * i + (ln >> 2);
    const int col = 8 * j + 2 * (ln & 3);
    if (row < A.a) {
      if (col < A.b) go[(size_t)row * A.b + col] = v0;
      if (col + 1 < A.b) go[(size_t)row * A.b + col + 1] = v1;
    }
  }
}

// full-block tail columns (8, 9 at m = 10) on DFMA.  0: DMMA (a 75%-empty
// column tile); 1: lane = (row, side, column), every lane sums k = 0..9 (each
// 16-byte load serves two lanes: 8 shared-memory wavefronts per load, 150 per
// warp-chunk with the coefficient loads); 2: lane = (row, side, k-half), 32
// distinct conflict-free 16-byte loads per instruction and three shuffles
// (72 wavefronts per warp-chunk).  The pass is bound by the shared-memory
// data pipe (ncu: l1tex__data_pipe_lsu_wavefronts at 81% of peak with form 1).
#ifndef B2L_TAIL_DFMA
#define B2L_TAIL_DFMA 2
#endif
#ifndef B2L_STORE_SWZ   // conflict-free output stores of the full-block pair kernels
#define B2L_STORE_SWZ 1
#endif
#ifndef B2L_PAIR_NW
#define B2L_PAIR_NW 14
#endif
constexpr int PAIR_NW = B2L_PAIR_NW;               // compute warps (7 pairs, 56-row chunks)
// m = 16 full block: 6 pairs, 48-row chunks -- three compute warps on every SM
// sub-partition (14 = 4 + 4 + 3 + 3 leaves the pace to the fuller ones); the
// DMMA-bound pass gains 3-6% (C3 F1 5.37 -> 5.18 ms), the m = 10 pass nothing
#ifndef B2L_PAIR16_NW
#define B2L_PAIR16_NW 12
#endif
constexpr int PAIR16_NW = B2L_PAIR16_NW;
#ifndef B2L_PAIR16_NOB
#define B2L_PAIR16_NOB 2
#endif
constexpr int PAIR16_NOB = B2L_PAIR16_NOB;         // its output buffers
constexpr int PAIR_THREADS = 32 * (2 + PAIR_NW);   // 512: loader + 14 compute + storer warps
constexpr int PAIR_BAR = 32 * (1 + PAIR_NW);       // output-buffer barriers: compute + storer
#ifndef B2L_PAIR_NOB
#define B2L_PAIR_NOB 3
#endif
constexpr int PAIR_NOB = B2L_PAIR_NOB;             // output buffers
constexpr int NB_POFULL = 1;                       // named barriers 1..3
constexpr int NB_PAIR = 5;                         // named barriers 5..11
constexpr int NB_POEMPTY = 12;                     // named barriers 12..14
constexpr int NB_PAIR_DONE = 15;
constexpr int NB_GRND = 4;                         // compute warps, Gram rounds

// Which half of its pair compute warp cw is.  A warp issues on SM
// sub-partition (warp index) % 4, and at m = 10 half 0 carries ~1.8x the fp64
// pipe time of half 1 (18 + 14 DMMA against the DFMA tail + 14 DMMA per
// chunk): with H = cw & 1 every half-0 warp lands on sub-partitions 1 and 3.
// Flipping every other pair of pairs gives each sub-partition both kinds.
// timing ablations of the pair kernel (wrong results; tools/time_f1.py only):
// 1 no Gram phase, 2 no update math, 4 no TMA stores, 8 no pair barrier,
// 16 no output stores to shared memory
#ifndef B2L_ABLATE
#define B2L_ABLATE 0
#endif
// -DB2L_TRACE: phase time stamps (clock64) of CTA 0's compute warps for its
// first 48 chunks (tools/trace_f1.py reads them through b2l_debug_trace)
#ifdef B2L_TRACE
__device__ long long g_trace[16 * 48 * 8];
#define TRACE(slot)                                                          \
  do {                                                                       \
    if (blockIdx.x == 0 && lane == 0 && it < 48)                             \
      g_trace[((warp - 1) * 48 + it) * 8 + (slot)] = clock64();              \
  } while (0)
#else
#define TRACE(slot) ((void)0)
#endif
#ifndef B2L_PAIR_BALANCE
#define B2L_PAIR_BALANCE 1
#endif
__device__ __forceinline__ int pair_half(int cw) {
  return B2L_PAIR_BALANCE ? ((cw & 1) ^ ((cw >> 2) & 1)) : (cw & 1);
}

// ---------------------------------------------------------------------------
// F1, warp-pair variant (m = 9..10): 14 compute warps, two per 8-row tile.
// Of a pair, warp h = 0 forms P' and X', warp h = 1 forms AP' and AX' (the
// same coefficients on the A-side blocks); after a pair barrier the 64
// threads form the residual of the 8 rows, and after a second one each warp
// folds the 8 rows into its share of the Gram tiles (a compile-time tile
// list: with MFIX the tiles the next step never reads are not computed).
// Halving every warp's accumulators keeps 4 warps per SM sub-partition
// resident (vs 2 in the one-warp-per-tile layout), which is what keeps the
// DMMA pipe fed.
// NOB output buffers (3; 2 at m = 16, whose 56-row buffers are 45 KB each);
// GRND: the CTA's Gram partials are summed pair by pair into one tile set
// (rounds) instead of stashed per pair -- the per-pair stash of m = 16 (48
// tiles x 7 pairs) would not fit the idle stage ring.  Same summation order.
template <int NT, int KS, int NI, int NJ, int MFIX, bool WGT, int NOB = PAIR_NOB,
          bool GRND = false, int NW = PAIR_NW>
__global__ void __launch_bounds__(32 * (2 + NW), 1)
    step_pair_kernel(const __grid_constant__ StepMaps M, const __grid_constant__ StepArgs Ain,
                    const __grid_constant__ StepCoef Cf) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  __shared__ StepArgs sA;
  if (threadIdx.x == 0) sA = Ain;
  __syncthreads();
  const StepArgs& A = sA;
  double* sm = reinterpret_cast<double*>(sm_raw);
  const uint32_t sm_base = smem_u32(sm_raw);
  double* stages = sm;
  double* coef = sm + A.coef_off;
  double* slam = sm + A.lam_off;
  int* spc = reinterpret_cast<int*>(sm + A.int_off);
  int* swp = spc + A.kp;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + A.bar_off);
  uint64_t* empty = full + 4;
  // output buffer b free again: the storer's arrival after its TMA store has
  // read the buffer (an mbarrier, so compute warps wait individually instead
  // of meeting at a CTA-wide named barrier every chunk)
  uint64_t* oempty = full + 8;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // MFIX > 0: the full-block step (kw = kp = kw_next = m = MFIX, every column
  // active, so P and W' columns are the identity maps): every size, stride
  // and predicate below is a compile-time constant
  constexpr bool FIX = MFIX > 0;
  constexpr bool CSM = MFIX == 16;   // coefficient fragments from shared memory
  constexpr int SF = FIX ? smem_stride(MFIX) : 4;
  const int m = FIX ? MFIX : A.m;
  const int kw = FIX ? MFIX : A.kw, kp = FIX ? MFIX : A.kp;
  const int sx = FIX ? SF : A.sx, sw = FIX ? SF : A.sw, swn = FIX ? SF : A.swn;
  const int ncoef = m * m + kw * m + kp * m;
  const bool inl = A.coef == nullptr;
  // m = 16 full block: the coefficient rows at the padded stride of the tiles
  // (20 doubles) -- a fragment load takes rows k = 4 ks + q of one column
  // octet, and at a 128-byte pitch its four q lanes meet on one bank
  // (8 wavefronts instead of 2: 29% of the pass's shared-memory wavefronts)
  constexpr int CPITCH = CSM ? SF : 0;
  for (int i = tid; i < ncoef; i += blockDim.x)
    coef[CSM ? (i / MFIX) * CPITCH + (i % MFIX) : i] = inl ? Cf.c[i] : A.coef[i];
  for (int i = tid; i < m; i += blockDim.x) {
    slam[i] = inl ? Cf.lam[i] : A.lam[i];
    swp[i] = inl ? Cf.wpos[i] : A.wpos[i];
  }
  for (int i = tid; i < kp; i += blockDim.x) spc[i] = inl ? Cf.pcols[i] : A.pcols[i];
  for (int i = tid; i < 16; i += blockDim.x) sm[A.zero_off + i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int b = 0; b < NOB; ++b) mbar_init(&oempty[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (FIX && MFIX == 10 && B2L_TAIL_DFMA == 2) {
    // tail table: entry ((kh*3 + j)*2 + e)*3 + blk = rows k of (Cw, Cp, Cx),
    // columns 8 and 9, k = 4j + 2kh + e (j < 2), k = 8 + e (j = 2, kh = 0);
    // (j = 2, kh = 1) re-reads k = 8, 9 against zeros
    if (tid < 36) {
      const int blk = tid % 3, e = (tid / 3) & 1, j = (tid / 6) % 3, kh = tid / 18;
      const int k = j == 2 ? 8 + e : 4 * j + 2 * kh + e;
      const bool z = j == 2 && kh == 1;
      const double* cb = coef + (blk == 0 ? MFIX * MFIX : blk == 1 ? 2 * MFIX * MFIX : 0) + k * MFIX;
      sm[A.tail_off + 2 * tid] = z ? 0.0 : cb[8];
      sm[A.tail_off + 2 * tid + 1] = z ? 0.0 : cb[9];
    }
    __syncthreads();
  }

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk_of = [&](int it) { return blockIdx.x + it * gridDim.x; };
  double* gred = sm + A.gred_off;   // [pair][NI*NJ tiles][32][2]
  double s_w0 = 0.0, s_a0 = 0.0, s_w1 = 0.0, s_a1 = 0.0;   // per-lane column partials

  // compute warps: one instantiation per half, so each owns exactly its
  // accumulators (the register allocator never sees the other half's)
  auto run_half = [&](auto hc) {
    constexpr int H = decltype(hc)::value;
    // even split of the Gram tiles: the pair barrier makes the chunk's path
    // max(update) + max(Gram), so moving tiles to the lighter half 1 (DFMA
    // tail update) does not pay (measured: 4/10 and 5/9 splits slower)
    constexpr PairTiles TL = pair_tiles(NI, NJ, MFIX, H);
    const int cw = warp - 1;
    const int mt = cw >> 1;                    // 8-row tile
    const int pbar = NB_PAIR + mt;
    const int q = lane & 3, rl = lane >> 2;
    // this warp's output column tile: nt = H (columns 8H .. 8H+7)
    static_assert(NT == 2, "the warp pair splits the update by column tile");
    double cW[KS], cP[KS], cX[KS];
    int pcol[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + q;
      if ((FIX && MFIX == 10 && H == 1 && B2L_TAIL_DFMA) || CSM) {   // tail on DFMA / m = 16
        cW[ks] = cP[ks] = cX[ks] = 0.0;
        pcol[ks] = FIX ? k : 0;
        continue;
      }
      pcol[ks] = FIX ? k : (k < kp ? spc[k] : 0);
      const int cb = 8 * H + rl;
      const bool cv = cb < m;
      cW[ks] = (cv && k < kw) ? coef[m * m + k * m + cb] : 0.0;
      cP[ks] = (cv && k < kp) ? coef[m * m + kw * m + k * m + cb] : 0.0;
      cX[ks] = (cv && k < m) ? coef[k * m + cb] : 0.0;
    }
    // residual columns of this lane: c = 8H + 2q + e (fragment layout of C)
    double lamc[2];
    int wposc[2];
    bool colok[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 8 * H + 2 * q + e;
      colok[e] = c < m;
      lamc[e] = colok[e] ? slam[c] : 0.0;
      wposc[e] = colok[e] ? (FIX ? c : swp[c]) : -1;
    }
    // (a compile-time `weighted = WGT` measured 1.5% slower at C2: ptxas orders the
    // epilogue differently)
    const bool weighted = A.d != nullptr, want_ax = A.want_ax != 0;
    const int tmode = A.tmode;
    const double tinv = A.tinv;
    const int npad = FIX ? 0 : A.ldwn - A.kwn;
    const int ldx = FIX ? MFIX : A.ldx;
    double s_w[2] = {0.0, 0.0}, s_a[2] = {0.0, 0.0};
    // lane columns of the tile rows / columns this warp uses
    const uint32_t zero_adr = sm_base + (uint32_t)A.zero_off * 8u;
    uint32_t la_[NI], ls_[NI], rb_[NJ], rs_[NJ];
    bool rw_[NJ];
    const int Lblk[3] = {0, 4, 2};
    const int Rblk[4] = {0, 4, 2, 3};
    const uint32_t obase_lane = sm_base + 8u * (uint32_t)(A.out_off[0] + (lane >> 2));
    if constexpr (FIX && !CSM) {
      // full block: a = 3m rows, b = 4m columns, every block at row stride
      // SF -- compile-time strides; lanes past the last row / column read a
      // valid in-tile address (their entries are never written back)
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int ci0 = 8 * i + (lane >> 2);
        const int ci = ci0 < 3 * MFIX ? ci0 : 0;
        const int l = ci / MFIX;
        la_[i] = sm_base + 8u * (uint32_t)(A.out_off[Lblk[l]] + (ci - l * MFIX));
        ls_[i] = 8u * SF;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int cj0 = 8 * j + (lane >> 2);
        const int cj = cj0 < 4 * MFIX ? cj0 : 0;
        const int r = cj / MFIX;
        rb_[j] = sm_base + 8u * (uint32_t)(A.out_off[Rblk[r]] + (cj - r * MFIX));
        rs_[j] = 8u * SF;
        rw_[j] = r < 3 && cj0 < 4 * MFIX;
      }
    } else {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (CSM) break;
      la_[i] = zero_adr;
      ls_[i] = 0;
      if (!((TL.imask >> i) & 1u)) continue;
      const int ci = 8 * i + (lane >> 2);
      if (ci < A.a) {
        int l = 0;
        while (l + 1 < 3 && A.lcum[l + 1] <= ci) ++l;
        la_[i] = sm_base + 8u * (A.out_off[Lblk[l]] + (ci - A.lcum[l]));
        ls_[i] = 8u * (l == 1 ? swn : sx);
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (CSM) break;
      rb_[j] = zero_adr;
      rs_[j] = 0;
      rw_[j] = false;
      if (!((TL.jmask >> j) & 1u)) continue;
      const int cj = 8 * j + (lane >> 2);
      if (cj < A.b) {
        int r = 0;
        while (r + 1 < 4 && A.rcum[r + 1] <= cj) ++r;
        rb_[j] = sm_base + 8u * (A.out_off[Rblk[r]] + (cj - A.rcum[r]));
        rs_[j] = 8u * (r == 1 ? swn : sx);
        rw_[j] = r < 3;
      }
    }
    }
    double gacc[TL.n > 0 ? TL.n : 1][2];
#pragma unroll
    for (int t = 0; t < TL.n; ++t) gacc[t][0] = gacc[t][1] = 0.0;

    int s = 0, b = 0;
    uint32_t phase = 0, ophase = 0;
    for (int it = 0; it < nloc; ++it) {
      TRACE(0);
      if (it >= NOB) mbar_wait(&oempty[b], ophase);
      TRACE(1);
      mbar_wait(&full[s], phase);
      TRACE(2);
      const double* st = stages + (size_t)s * A.stage_doubles;
      const int ob = b * A.out_stride;
      const int r = 8 * mt + rl;
      if constexpr (!(B2L_ABLATE & 2)) {
        // ---- (1) update of this warp's column tile, all six products, and
        // (2) the next residual straight from the accumulators
        const double* W = st + A.in_off[2];
        const double* AW = st + A.in_off[3];
        const double* P = st + A.in_off[4];
        const double* AP = st + A.in_off[5];
        const double* X = st + A.in_off[0];
        const double* AX = st + A.in_off[1];
        // per lane: the two columns co, co+1 of P', AP', X', AX'
        double pn_[2], apn_[2], xn_[2], axn_[2];
        const bool bw = kw > 0, bp = kp > 0;
        if constexpr (FIX && MFIX == 10 && H == 1 && B2L_TAIL_DFMA == 2) {
          // full block, columns 8, 9 on DFMA, k split over lane pairs: lane =
          // (kh = lane & 1, row = 4 (lane >> 4) + ((lane >> 1) & 3), side =
          // (lane >> 3) & 1).  An 8-lane phase of a 16-byte load covers 4 rows
          // x 2 k-halves of one block: rows 96 B apart, halves 16 B apart --
          // eight distinct 16-byte bank groups.
          const int kh = lane & 1;
          const int tr_ = 8 * mt + 4 * (lane >> 4) + ((lane >> 1) & 3);
          const bool aside = (lane >> 3) & 1;
          const double* D1 = (aside ? AW : W) + tr_ * SF;
          const double* D2 = (aside ? AP : P) + tr_ * SF;
          const double* D3 = (aside ? AX : X) + tr_ * SF;
          const double2* T2 = reinterpret_cast<const double2*>(sm + A.tail_off) + 18 * kh;
          double sw0 = 0.0, sw1 = 0.0, sp0 = 0.0, sp1 = 0.0, sx0 = 0.0, sx1 = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int kk = j == 2 ? 8 : 4 * j + 2 * kh;
            const double2 w2 = *reinterpret_cast<const double2*>(D1 + kk);
            const double2 p2 = *reinterpret_cast<const double2*>(D2 + kk);
            const double2 x2 = *reinterpret_cast<const double2*>(D3 + kk);
            const double2 cwa = T2[(2 * j) * 3], cpa = T2[(2 * j) * 3 + 1], cxa = T2[(2 * j) * 3 + 2];
            const double2 cwb = T2[(2 * j + 1) * 3], cpb = T2[(2 * j + 1) * 3 + 1],
                          cxb = T2[(2 * j + 1) * 3 + 2];
            sw0 = fma(w2.x, cwa.x, sw0);
            sw1 = fma(w2.x, cwa.y, sw1);
            sp0 = fma(p2.x, cpa.x, sp0);
            sp1 = fma(p2.x, cpa.y, sp1);
            sx0 = fma(x2.x, cxa.x, sx0);
            sx1 = fma(x2.x, cxa.y, sx1);
            sw0 = fma(w2.y, cwb.x, sw0);
            sw1 = fma(w2.y, cwb.y, sw1);
            sp0 = fma(p2.y, cpb.x, sp0);
            sp1 = fma(p2.y, cpb.y, sp1);
            sx0 = fma(x2.y, cxb.x, sx0);
            sx1 = fma(x2.y, cxb.y, sx1);
          }
          // lane kh keeps column 8 + kh: it sends its partial of the other
          // column and adds the partner's partial of its own
          const double t0 = __dadd_rn(sw0, sp0), t1 = __dadd_rn(sw1, sp1);
          const double pv = __dadd_rn(kh ? t1 : t0, __shfl_xor_sync(0xffffffffu, kh ? t0 : t1, 1));
          const double sxv =
              __dadd_rn(kh ? sx1 : sx0, __shfl_xor_sync(0xffffffffu, kh ? sx0 : sx1, 1));
          const double xv = A.xpp ? __dadd_rn(sxv, pv) : sxv;   // X' / AX' entry
          const double ov = __shfl_xor_sync(0xffffffffu, xv, 8);   // the other side's
          const int oc = tr_ * SF + 8 + kh;
          (sm + A.out_off[aside ? 1 : 0] + ob)[oc] = xv;
          (sm + A.out_off[aside ? 3 : 2] + ob)[oc] = pv;
          if (!aside) {
            const double dr = weighted ? st[A.d_off + tr_] : 1.0;
            const double bx = weighted ? __dmul_rn(dr, xv) : xv;
            const double wf = __dsub_rn(ov, __dmul_rn(bx, slam[8 + kh]));
            s_w[0] = fma(wf, wf, s_w[0]);
            const double trw = tmode == 2 ? st[A.t_off + tr_] : tinv;
            (sm + A.out_off[4] + ob)[oc] = tmode == 0 ? wf : __dmul_rn(trw, wf);
          } else if (want_ax) {
            s_a[0] = fma(xv, xv, s_a[0]);
          }
        } else {
        if constexpr (FIX && MFIX == 10 && H == 1 && B2L_TAIL_DFMA) {
          // full block, columns 8..MFIX-1 (2 at MFIX = 10): DFMA instead of a
          // 75%-empty DMMA column tile.  Lane (row rl, q) forms column
          // 8 + (q & 1) of the P side (q < 2: W, P, X) or the A side (q >= 2:
          // AW, AP, AX); the four values of a row are then gathered in its
          // q = 0 lane, the lane the DMMA layout gives columns 8, 9.
          const int c = 8 + (q & 1);
          const bool aside = q >= 2;
          const double* D1 = (aside ? AW : W) + r * SF;
          const double* D2 = (aside ? AP : P) + r * SF;
          const double* D3 = (aside ? AX : X) + r * SF;
          const double* cw = coef + MFIX * MFIX + c;
          const double* cp = coef + 2 * MFIX * MFIX + c;
          const double* cx = coef + c;
          double sw_ = 0.0, sp_ = 0.0, sx_ = 0.0;
#pragma unroll
          for (int k = 0; k < MFIX; k += 2) {
            const double2 w2 = *reinterpret_cast<const double2*>(D1 + k);
            const double2 p2 = *reinterpret_cast<const double2*>(D2 + k);
            const double2 x2 = *reinterpret_cast<const double2*>(D3 + k);
            sw_ = fma(w2.x, cw[k * MFIX], sw_);
            sp_ = fma(p2.x, cp[k * MFIX], sp_);
            sx_ = fma(x2.x, cx[k * MFIX], sx_);
            sw_ = fma(w2.y, cw[(k + 1) * MFIX], sw_);
            sp_ = fma(p2.y, cp[(k + 1) * MFIX], sp_);
            sx_ = fma(x2.y, cx[(k + 1) * MFIX], sx_);
          }
          const double pv = __dadd_rn(sw_, sp_);
          const double xv = A.xpp ? __dadd_rn(sx_, pv) : sx_;
          pn_[0] = pv;
          xn_[0] = xv;
          pn_[1] = __shfl_down_sync(0xffffffffu, pv, 1);
          xn_[1] = __shfl_down_sync(0xffffffffu, xv, 1);
          apn_[0] = __shfl_down_sync(0xffffffffu, pv, 2);
          axn_[0] = __shfl_down_sync(0xffffffffu, xv, 2);
          apn_[1] = __shfl_down_sync(0xffffffffu, pv, 3);
          axn_[1] = __shfl_down_sync(0xffffffffu, xv, 3);
        } else {
        double acc[6][2];
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int k = 4 * ks + q;
          const bool kw_ok = k < kw, kp_ok = k < kp, km_ok = k < m;
          const double wv = kw_ok ? W[r * sw + k] : 0.0;
          const double awv = kw_ok ? AW[r * sw + k] : 0.0;
          const double pv = kp_ok ? P[r * sx + pcol[ks]] : 0.0;
          const double apv = kp_ok ? AP[r * sx + pcol[ks]] : 0.0;
          const double xv = km_ok ? X[r * sx + k] : 0.0;
          const double axv = km_ok ? AX[r * sx + k] : 0.0;
          // m = 16: the coefficient fragments come from shared memory each
          // chunk (12 registers fewer for the 17-tile Gram accumulators)
          const double cw_ = CSM ? coef[(MFIX + k) * CPITCH + 8 * H + rl] : cW[ks];
          const double cp_ = CSM ? coef[(2 * MFIX + k) * CPITCH + 8 * H + rl] : cP[ks];
          const double cx_ = CSM ? coef[k * CPITCH + 8 * H + rl] : cX[ks];
          dmma_8x8x4(acc[0][0], acc[0][1], wv, cw_);
          dmma_8x8x4(acc[1][0], acc[1][1], awv, cw_);
          dmma_8x8x4(acc[2][0], acc[2][1], pv, cp_);
          dmma_8x8x4(acc[3][0], acc[3][1], apv, cp_);
          dmma_8x8x4(acc[4][0], acc[4][1], xv, cx_);
          dmma_8x8x4(acc[5][0], acc[5][1], axv, cx_);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pn_[e] = (bw && bp) ? __dadd_rn(acc[0][e], acc[2][e]) : (bw ? acc[0][e] : acc[2][e]);
          apn_[e] = (bw && bp) ? __dadd_rn(acc[1][e], acc[3][e]) : (bw ? acc[1][e] : acc[3][e]);
          xn_[e] = A.xpp ? __dadd_rn(acc[4][e], pn_[e]) : acc[4][e];
          axn_[e] = A.xpp ? __dadd_rn(acc[5][e], apn_[e]) : acc[5][e];
        }
        }
        double* O0 = sm + A.out_off[0] + ob;
        double* O1 = sm + A.out_off[1] + ob;
        double* O2 = sm + A.out_off[2] + ob;
        double* O3 = sm + A.out_off[3] + ob;
        double* O4 = sm + A.out_off[4] + ob;
        const double dr = weighted ? st[A.d_off + r] : 1.0;
        const double tr = tmode == 2 ? st[A.t_off + r] : tinv;
        const int co = 8 * H + 2 * q;
        // m = 10 full block, columns 0..7: odd rows store their second column
        // first.  A lane's two 8-byte columns sit in one 16-byte slot, and at
        // the 96-byte row pitch two rows of a half-warp share every slot
        // (2-way conflicts, 4 wavefronts per store); with the odd rows'
        // halves swapped the 16 lanes cover 16 distinct bank pairs (C2 F1
        // 0.388 -> 0.374 ms).  The register-bound m = 16 kernel spills on the
        // selects and loses (5.04 -> 5.49 ms), so it keeps the plain order.
        constexpr bool SWZ = FIX && MFIX == 10 && H == 0 && B2L_STORE_SWZ;
        if constexpr (SWZ) {
          double wv_[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // W'_j = T (AX'_j - BX'_j lam_j) (lobpcg.py:429-430, :466-467)
            const double bx = weighted ? __dmul_rn(dr, xn_[e]) : xn_[e];
            const double wf = __dsub_rn(axn_[e], __dmul_rn(bx, lamc[e]));
            s_w[e] = fma(wf, wf, s_w[e]);
            if (want_ax) s_a[e] = fma(axn_[e], axn_[e], s_a[e]);
            wv_[e] = tmode == 0 ? wf : __dmul_rn(tr, wf);
          }
          const bool odd = rl & 1;
          const int a0 = r * SF + co + (odd ? 1 : 0), a1 = r * SF + co + (odd ? 0 : 1);
          O0[a0] = odd ? xn_[1] : xn_[0];
          O1[a0] = odd ? axn_[1] : axn_[0];
          O2[a0] = odd ? pn_[1] : pn_[0];
          O3[a0] = odd ? apn_[1] : apn_[0];
          O4[a0] = odd ? wv_[1] : wv_[0];
          O0[a1] = odd ? xn_[0] : xn_[1];
          O1[a1] = odd ? axn_[0] : axn_[1];
          O2[a1] = odd ? pn_[0] : pn_[1];
          O3[a1] = odd ? apn_[0] : apn_[1];
          O4[a1] = odd ? wv_[0] : wv_[1];
        } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double pn = pn_[e], apn = apn_[e], xn = xn_[e], axn = axn_[e];
          if (co + e < ldx) {
            O0[r * sx + co + e] = xn;
            O1[r * sx + co + e] = axn;
            O2[r * sx + co + e] = pn;
            O3[r * sx + co + e] = apn;
          }
          if (colok[e]) {
            // W'_j = T (AX'_j - BX'_j lam_j) (lobpcg.py:429-430, :466-467)
            const double bx = weighted ? __dmul_rn(dr, xn) : xn;
            const double wf = __dsub_rn(axn, __dmul_rn(bx, lamc[e]));
            s_w[e] = fma(wf, wf, s_w[e]);
            if (want_ax) s_a[e] = fma(axn, axn, s_a[e]);
            const double wv = tmode == 0 ? wf : __dmul_rn(tr, wf);
            if (wposc[e] >= 0) O4[r * swn + wposc[e]] = wv;
          }
        }
        }
        // W' padding columns (kw_next .. ldw_next-1) of this warp's rows
        if (H == 1)
          for (int e = lane; e < 8 * npad; e += 32) {
            const int rr = e / npad;
            O4[(8 * mt + rr) * swn + (FIX ? MFIX : A.kwn) + (e - rr * npad)] = 0.0;
          }
        }
      }
      // the stage is free once the update has read it (the B-weighted Gram
      // still reads d from it): the loader refills it while the Gram runs
      if (!WGT) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      TRACE(3);
      if constexpr (!(B2L_ABLATE & 8)) nbar_sync(pbar, 64);
      TRACE(4);
      // ---- (3) Gram over the 8 rows, this warp's tiles (m = 16: one row
      // quad's fragments live at a time)
      const uint32_t boff = 8u * (uint32_t)ob;
#pragma unroll
      for (int ks = 0; ks < ((B2L_ABLATE & 1) ? 0 : 2); ++ks) {
        const uint32_t row = (uint32_t)(8 * mt + 4 * ks + q);
        double av[NI], bv[NJ];
        if constexpr (CSM) {
          // m = 16 full block: every tile column sits at a compile-time
          // offset from one per-lane base (the output blocks are TXC apart):
          // immediates instead of 14 address registers
          constexpr uint32_t TXC = (uint32_t)((4 * NW * SF + 15) & ~15);
          constexpr uint32_t LB[3] = {0u, 4u * TXC, 2u * TXC};        // X', W', P'
          constexpr uint32_t RB[4] = {0u, 4u * TXC, 2u * TXC, 3u * TXC};  // + AP'
          const uint32_t base = obase_lane + boff + row * (8u * SF);
#pragma unroll
          for (int i = 0; i < NI; ++i)
            av[i] = ((TL.imask >> i) & 1u)
                        ? lds64(base + 8u * (LB[i / 2] + 8u * (uint32_t)(i % 2))) : 0.0;
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            bv[j] = ((TL.jmask >> j) & 1u)
                        ? lds64(base + 8u * (RB[j / 2] + 8u * (uint32_t)(j % 2))) : 0.0;
        } else {
#pragma unroll
        for (int i = 0; i < NI; ++i)
          av[i] = ((TL.imask >> i) & 1u) ? lds64(la_[i] + (ls_[i] ? boff : 0u) + row * ls_[i])
                                          : 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          bv[j] = ((TL.jmask >> j) & 1u) ? lds64(rb_[j] + (rs_[j] ? boff : 0u) + row * rs_[j])
                                          : 0.0;
        }
        if (WGT) {
          const double w = st[A.d_off + row];
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (rw_[j]) bv[j] = __dmul_rn(w, bv[j]);
        }
#pragma unroll
        for (int t = 0; t < TL.n; ++t)
          dmma_8x8x4(gacc[t][0], gacc[t][1], av[TL.ti[t]], bv[TL.tj[t]]);
      }
      TRACE(5);
      fence_async_smem();   // generic writes -> the TMA store (async proxy)
      __syncwarp();
      if (WGT && lane == 0) mbar_arrive(&empty[s]);
      nbar_arrive(NB_POFULL + b, (32 * (1 + NW)));
      TRACE(6);
      if (++s == A.nst) {
        s = 0;
        phase ^= 1u;
      }
      if (++b == NOB) {
        b = 0;
        if (it + 1 > NOB) ophase ^= 1u;
      }
    }
    if constexpr (FIX && MFIX == 10 && H == 1 && B2L_TAIL_DFMA == 2) {
      // the k-split tail keeps column 8 + c of row g in lane (c | (g & 3) << 1
      // | (g >> 2) << 4) (P side: |W'|^2) and that lane | 8 (A side: |AX'|^2);
      // the CTA reduction reads lane 4g, entry c
      const int g = lane >> 2;
      const int src = ((g & 3) << 1) | ((g >> 2) << 4);
      const double w0 = __shfl_sync(0xffffffffu, s_w[0], src);
      const double w1 = __shfl_sync(0xffffffffu, s_w[0], src | 1);
      const double a0 = __shfl_sync(0xffffffffu, s_a[0], src | 8);
      const double a1 = __shfl_sync(0xffffffffu, s_a[0], src | 9);
      const bool own = (lane & 3) == 0;
      s_w[0] = own ? w0 : 0.0;
      s_w[1] = own ? w1 : 0.0;
      s_a[0] = own ? a0 : 0.0;
      s_a[1] = own ? a1 : 0.0;
    }
    s_w0 = s_w[0];
    s_w1 = s_w[1];
    s_a0 = s_a[0];
    s_a1 = s_a[1];
    // the stage ring is idle once every warp is here: stash the accumulators
    nbar_sync(NB_PAIR_DONE, (32 * (2 + NW)));
    if constexpr (GRND) {
      // one tile set, zeroed, then pair by pair (p = 0, 1, ...: the order of
      // the stash-and-sum form) each pair adds its halves' disjoint tiles
      for (int e = (warp - 1) * 32 + lane; e < NI * NJ * 64; e += NW * 32) gred[e] = 0.0;
      nbar_sync(NB_GRND, NW * 32);
      for (int p = 0; p < NW / 2; ++p) {
        if (mt == p)
#pragma unroll
          for (int t = 0; t < TL.n; ++t) {
            const size_t o = (((size_t)TL.ti[t] * NJ + TL.tj[t]) * 32 + lane) * 2;
            gred[o] += gacc[t][0];
            gred[o + 1] += gacc[t][1];
          }
        nbar_sync(NB_GRND, NW * 32);
      }
      return;
    }
#pragma unroll
    for (int t = 0; t < TL.n; ++t) {
      const size_t o =
          (((size_t)mt * NI * NJ + TL.ti[t] * NJ + TL.tj[t]) * 32 + lane) * 2;
      gred[o] = gacc[t][0];
      gred[o + 1] = gacc[t][1];
    }
    if (MFIX && H == 0) {
      // tiles nobody computes: defined zeros
      for (int t = 0; t < NI * NJ; ++t)
        if (!((TL.need[t >> 5] >> (t & 31)) & 1u)) {
          const size_t o = (((size_t)mt * NI * NJ + t) * 32 + lane) * 2;
          gred[o] = 0.0;
          gred[o + 1] = 0.0;
        }
    }
  };

  if (warp == 0) {
    // ================= loader: refills a stage as soon as it is released
    if (lane == 0)
      for (int j = 0; j < nloc; ++j) {
        const int s = j % A.nst;
        if (j >= A.nst) mbar_wait(&empty[s], (j / A.nst - 1) & 1);
        step_issue(M, A, stages + (size_t)s * A.stage_doubles, &full[s], chunk_of(j));
      }
    __syncwarp();
    nbar_sync(NB_PAIR_DONE, (32 * (2 + NW)));
  } else if (warp == NW + 1) {
    // ================= storer: TMA stores of each finished output buffer
    for (int it = 0; it < nloc; ++it) {
      const int b = it % NOB;
      nbar_sync(NB_POFULL + b, (32 * (1 + NW)));
      if (lane == 0) {
        const int r0 = chunk_of(it) * A.rc;
        const int ob = b * A.out_stride;
        for (int k = 0; k < ((B2L_ABLATE & 4) ? 0 : 5); ++k) {
          if (k == 4 && A.kwn == 0) continue;
          tma_store_2d(&M.out[k], sm + A.out_off[k] + ob, 0, r0);
        }
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&oempty[b]);
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
    nbar_sync(NB_PAIR_DONE, (32 * (2 + NW)));
  } else if (pair_half(warp - 1) == 0) {
    run_half(std::integral_constant<int, 0>{});
  } else {
    run_half(std::integral_constant<int, 1>{});
  }
  __syncthreads();

  // ---- CTA reductions (fixed order over pairs / rows)
  double* red = sm + A.red_off;
  const int NL = NW * 64;      // [warp][lane][e]
  if (warp >= 1 && warp <= NW) {
    const int o = ((((warp - 1) & ~1) + pair_half(warp - 1)) * 32 + lane) * 2;   // [2 pair + H]
    red[o] = s_w0;
    red[o + 1] = s_w1;
    red[NL + o] = s_a0;
    red[NL + o + 1] = s_a1;
  }
  __syncthreads();
  double* out = A.partial + (size_t)blockIdx.x * (2 * m + A.a * A.b);
  if (tid < m) {
    // column j lives in warp half H = j / 8, lanes with (lane & 3) = (j % 8) / 2, e = j % 2
    const int H = tid >> 3, qq = (tid & 7) >> 1, e = tid & 1;
    double a = 0.0, bb = 0.0;
    for (int p = 0; p < NW / 2; ++p)
      for (int g = 0; g < 8; ++g) {
        const int o = (((2 * p + H) * 32) + 4 * g + qq) * 2 + e;
        a += red[o];
        bb += red[NL + o];
      }
    out[tid] = a;
    out[m + tid] = bb;
  }
  double* go = out + 2 * m;
  for (int e = tid; e < NI * NJ * 32; e += blockDim.x) {
    const int t = e / 32, ln = e & 31;
    const int i = t / NJ, j = t % NJ;
    double v0 = 0.0, v1 = 0.0;
    if constexpr (GRND) {
      v0 = gred[(size_t)e * 2];
      v1 = gred[(size_t)e * 2 + 1];
    } else {
      for (int p = 0; p < NW / 2; ++p) {
        const size_t o = (((size_t)p * NI * NJ + t) * 32 + ln) * 2;
        v0 += gred[o];
        v1 += gred[o + 1];
      }
    }
    const int row = 8 * i + (ln >> 2);
    const int col = 8 * j + 2 * (ln & 3);
    if (row < A.a) {
      if (col < A.b) go[(size_t)row * A.b + col] = v0;
      if (col + 1 < A.b) go[(size_t)row * A.b + col + 1] = v1;
    }
  }
}

using StepKernel = void (*)(StepMaps, StepArgs, StepCoef);

template <int NT, int KS, int NI, int NJ, int MFIX, int NOB = PAIR_NOB, bool GRND = false,
          int NW = PAIR_NW>
static StepKernel pick_pair(bool wgt) {
  return wgt ? step_pair_kernel<NT, KS, NI, NJ, MFIX, true, NOB, GRND, NW>
             : step_pair_kernel<NT, KS, NI, NJ, MFIX, false, NOB, GRND, NW>;
}
template <int NT, int KS, int NI, int NJ, int MFIX>
static StepKernel pick_local(bool wgt) {
  return wgt ? step_local_kernel<NT, KS, NI, NJ, MFIX, true>
             : step_local_kernel<NT, KS, NI, NJ, MFIX, false>;
}
template <int NT, int KS>
static StepKernel pick_step(bool wgt) {
  return wgt ? step_kernel<NT, KS, true> : step_kernel<NT, KS, false>;
}

int lobpcg_step(int nrows, int m, const double* x, const double* ax, int ldx,
                const double* w, const double* aw, int ldw, int kw, const double* p,
                const double* ap, int kp, const int* pcols, const double* coef,
                double* xo, double* axo, double* po, double* apo, const double* lam,
                const double* d, int tmode, double tinv, const double* tvec,
                const int* wpos, int kwn, double* wo, int ldwn, int want_ax,
                double* red_out, cudaStream_t st, const StepHostCoef* hc,
                StepDeferred* defer, int x_plus_p) {
  B2L_CHECK(m >= 1 && m <= 16, -B2L_EINVAL, "step: 1 <= m <= 16 (larger blocks: b2l_update)");
  B2L_CHECK(nrows >= 1, -B2L_EINVAL, "step: empty block");
  B2L_CHECK(ldx >= m && (ldx & 1) == 0, -B2L_EINVAL, "step: ldx must be even and >= m");
  B2L_CHECK(kw >= 0 && kw <= m && kw <= ldw && (kw == 0 || (ldw & 1) == 0), -B2L_EINVAL,
            "step: bad W");
  B2L_CHECK(kp >= 0 && kp <= m, -B2L_EINVAL, "step: bad kp");
  B2L_CHECK(kw + kp > 0, -B2L_EINVAL, "step: nothing to update (kw + kp == 0)");
  B2L_CHECK(kwn >= 0 && kwn <= m && (kwn == 0 || (ldwn >= kwn && (ldwn & 1) == 0)),
            -B2L_EINVAL, "step: bad next W");
  StepArgs A{};
  A.nrows = nrows;
  A.m = m;
  A.ldx = ldx;
  A.kw = kw;
  A.kp = kp;
  A.kwn = kwn;
  A.sx = smem_stride(ldx);
  A.sw = kw ? smem_stride(ldw) : 4;
  A.swn = smem_stride(kwn ? ldwn : 2);
  A.ldwn = kwn ? ldwn : 2;
  A.d = d;
  A.tvec = tvec;
  A.coef = coef;
  A.pcols = pcols;
  A.wpos = wpos;
  A.lam = lam;
  // host coefficients travel in the launch itself (hc: b2l_fast_iteration)
  static StepCoef cf;   // the launch copies it; one host thread drives a context
  if (hc) {
    const int nc = m * m + kw * m + kp * m;
    for (int i = 0; i < nc; ++i) cf.c[i] = hc->coef[i];
    for (int i = 0; i < m; ++i) {
      cf.lam[i] = hc->lam[i];
      cf.wpos[i] = hc->wpos[i];
    }
    for (int i = 0; i < kp; ++i) cf.pcols[i] = hc->pcols[i];
    A.coef = nullptr;
    A.lam = nullptr;
    A.pcols = nullptr;
    A.wpos = nullptr;
  }
  A.tmode = tmode;
  A.tinv = tinv;
  A.want_ax = want_ax;
  A.xpp = x_plus_p;
  // Gram of the next step: L = [X' W' P'], R = [X' W' P' AP']
  A.lcum[0] = 0;
  A.lcum[1] = m;
  A.lcum[2] = m + kwn;
  A.lcum[3] = 2 * m + kwn;
  A.rcum[0] = 0;
  A.rcum[1] = m;
  A.rcum[2] = m + kwn;
  A.rcum[3] = 2 * m + kwn;
  A.rcum[4] = 3 * m + kwn;
  A.a = 2 * m + kwn;
  A.b = 3 * m + kwn;
  A.NI = (A.a + 7) / 8;
  A.NJ = (A.b + 7) / 8;
  static const unsigned char modes[12] = {2, 1, 1, 1, 0, 2, 1, 1, 0, 0, 2, 1};
  tile_mask(A.NI, A.NJ, A.lcum, 3, A.rcum, 4, modes, A.tmask);
  A.tsI = (A.NI + 1) / 2;
  A.tsJ = (A.NJ + 3) / 4;
  A.TS = A.tsI * A.tsJ;
  const int items = STEP_NG * STEP_GI;
  // the full block at m = 16 (C3 until columns lock): the warp-pair variant
  // with two output buffers and the Gram summed in rounds
  static const bool no_pair16 = [] {
    const char* v = getenv("B2L_STEP_VARIANT");
    return v && strcmp(v, "generic16") == 0;
  }();
  const bool pair16 = !no_pair16 && m == 16 && kw == 16 && kp == 16 && kwn == 16 && ldx == 16 &&
                      ldw == 16 && ldwn == 16 && !d && tmode != 2;
  const bool local = m <= 10 || pair16;   // warp-local variant
  const int lNI = m <= 4 ? 2 : (m <= 8 ? 3 : 4);
  const int lNJ = m <= 4 ? 2 : (m <= 8 ? 4 : 5);
  B2L_CHECK(local || A.TS <= items, -B2L_EINVAL, "step: Gram tile blocks exceed one CTA");
  A.rs = 1;
  while (A.rs * 2 * A.TS <= items) A.rs *= 2;
  // chunk rows: 8 update warps x 8-row tiles = 64 rows, fewer when a stage
  // (6 blocks + d + t) would exceed ~48 KB; then the deepest TMA ring (<= 4)
  // that fits one CTA per SM.
  const int width = 4 * A.sx + 2 * (kw ? A.sw : 0) + (d ? 1 : 0) + (tmode == 2 ? 1 : 0);
  // m = 9..10: the warp-pair variant (B2L_STEP_VARIANT=local forces the
  // one-warp-per-tile variant, for A/B timing); m <= 8: one warp per tile
  static const bool force_local = [] {
    const char* v = getenv("B2L_STEP_VARIANT");
    return v && strcmp(v, "local") == 0;
  }();
  const bool one_warp = (m <= 8 || force_local) && !pair16;
  const int pair_nw = pair16 ? PAIR16_NW : PAIR_NW;
  A.rc = (local && !one_warp) ? 4 * pair_nw : 64;
  while (!pair16 && A.rc > 16 && (size_t)A.rc * width * 8 > 48 * 1024) A.rc >>= 1;
  while (A.rs > 1 && A.rc / A.rs < 4) A.rs >>= 1;
  const int rc = A.rc;
  int off = 0;
  const int sin_[6] = {A.sx, A.sx, A.sw, A.sw, A.sx, A.sx};
  const bool on[6] = {true, true, kw > 0, kw > 0, kp > 0, kp > 0};
  A.stage_tx = 0;
  for (int b = 0; b < 6; ++b) {
    A.in_off[b] = off;
    if (on[b]) {
      off += rc * sin_[b];
      A.stage_tx += (uint32_t)rc * sin_[b] * 8u;
    }
  }
  A.d_off = off; off += d ? rc : 0;
  A.t_off = off; off += tmode == 2 ? rc : 0;
  A.stage_doubles = (off + 15) & ~15;
  const int tile_x = (rc * A.sx + 15) & ~15;
  const int tile_w = (rc * A.swn + 15) & ~15;
  // output buffers: 3 for the warp-pair variant (separate storer warp), else 2
  const bool pair = local && !one_warp;
  const int nob = pair16 ? PAIR16_NOB : (pair ? PAIR_NOB : 2);
  {
    const size_t tail = (size_t)nob * (4 * tile_x + tile_w) + (m * m + kw * m + kp * m) + 3 * m +
                        64 + 80 + (pair16 ? 192 : 0) + (pair ? 0 : (size_t)4 * STEP_NU * 32) + 64;
    const size_t budget = pair ? 224 * 1024 : 200 * 1024;
    A.nst = 4;
    while (A.nst > 2 && ((size_t)A.nst * A.stage_doubles + tail) * 8 > budget) --A.nst;
  }
  off = A.nst * A.stage_doubles;
  for (int b = 0; b < 4; ++b) {
    A.out_off[b] = off;
    off += tile_x;
  }
  A.out_off[4] = off;
  off += tile_w;
  A.out_stride = off - A.out_off[0];
  off += (nob - 1) * A.out_stride;  // the other output buffers
  A.coef_off = off;
  off += pair16 ? 3 * 16 * smem_stride(16) : ((m * m + kw * m + kp * m + 1) & ~1);
  A.lam_off = off;
  off += (m + 1) & ~1;
  A.int_off = off;
  off += (kp + m + 1) / 2 + 1;
  off = (off + 15) & ~15;
  A.zero_off = off;
  off += 16;
  A.tail_off = off;
  off += 80;   // 72 used (pair kernel, m = 10 full block)
  A.bar_off = off;
  off += 16;  // mbarriers
  A.red_off = off;
  const size_t red1 = (size_t)4 * 32 * (PAIR_NW > STEP_NU ? PAIR_NW : STEP_NU);   // PAIR16_NW <= PAIR_NW
  const size_t red2 = pair16 ? (size_t)A.NI * A.NJ * 64
                     : local ? (size_t)LOC_NW * lNI * lNJ * 64 : (size_t)A.TS * A.rs * 8 * 64;
  // the Gram item reduction reuses the (idle) stage ring after the loop; the
  // pair variant also puts the column-norm partials there
  if (pair && red2 + red1 <= (size_t)A.nst * A.stage_doubles) {
    A.gred_off = 0;
    A.red_off = (int)((red2 + 15) & ~(size_t)15);
  } else if (red2 <= (size_t)A.nst * A.stage_doubles) {
    A.gred_off = 0;
    off += (int)red1;
  } else if (pair) {
    // narrow stages (few active columns and no P: the ring is smaller than
    // the Gram scratch): the pair kernel's column-norm partials and Gram
    // partials are live together, so they get disjoint regions
    const int r1 = (int)((red1 + 15) & ~(size_t)15);
    A.gred_off = A.red_off + r1;
    off += r1 + (int)red2;
  } else {
    A.gred_off = A.red_off;
    off += (int)(red1 > red2 ? red1 : red2);
  }
  const size_t smem = (size_t)off * 8;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "step: shared memory budget exceeded");
  if (pair16) {   // the m = 16 kernel addresses the output blocks by compile-time offsets
    const int txc = (4 * PAIR16_NW * smem_stride(16) + 15) & ~15;
    B2L_CHECK(tile_x == txc && tile_w == txc && A.out_off[1] - A.out_off[0] == txc &&
                  A.out_off[4] - A.out_off[0] == 4 * txc,
              -B2L_EINVAL, "step: m = 16 output layout mismatch");
  }

  StepMaps M;
  const double* ins[6] = {x, ax, w, aw, p, ap};
  const int lds[6] = {ldx, ldx, ldw, ldw, ldx, ldx};
  for (int b = 0; b < 6; ++b) {
    if (!on[b]) {
      M.in[b] = M.in[0];
      continue;
    }
    int rcode = encode_tmap_2d(&M.in[b], ins[b], lds[b], nrows, sin_[b], rc);
    if (rcode) return rcode;
  }
  double* outs[5] = {xo, axo, po, apo, wo};
  const int ldo[5] = {ldx, ldx, ldx, ldx, kwn ? ldwn : 2};
  const int so[5] = {A.sx, A.sx, A.sx, A.sx, A.swn};
  for (int b = 0; b < 5; ++b) {
    if (b == 4 && kwn == 0) {
      M.out[4] = M.out[0];
      continue;
    }
    int rcode = encode_tmap_2d(&M.out[b], outs[b], ldo[b], nrows, so[b], rc);
    if (rcode) return rcode;
  }

  const bool wgt = d != nullptr;
  StepKernel kern;
  int threads;
  if (local) {
    B2L_CHECK(rc == (one_warp ? 8 * LOC_NW : 4 * pair_nw), -B2L_EINVAL,
              "step: warp-local variants need 64- / 56-row chunks");
    if (one_warp) {
      const bool full = kwn == m;   // the compile-time needed-tile lists assume kw_next = m
      threads = LOC_THREADS;
      if (m == 4 && full) kern = pick_local<1, 1, 2, 2, 4>(wgt);
      else if (m <= 4) kern = pick_local<1, 1, 2, 2, 0>(wgt);
      else if (m == 8 && full) kern = pick_local<1, 2, 3, 4, 8>(wgt);
      else if (m <= 8) kern = pick_local<1, 2, 3, 4, 0>(wgt);
      else kern = pick_local<2, 3, 4, 5, 0>(wgt);
    } else {
      threads = 32 * (2 + pair_nw);
      // the full-block specialisation: every column active (P and W' column
      // maps are then the identity), unpadded leading dimensions
      const bool full = m == 10 && kw == 10 && kp == 10 && kwn == 10 && ldx == 10 && ldw == 10 &&
                        ldwn == 10;
      kern = pair16 ? pick_pair<2, 4, 6, 8, 16, PAIR16_NOB, true, PAIR16_NW>(wgt)
             : full ? pick_pair<2, 3, 4, 5, 10>(wgt) : pick_pair<2, 3, 4, 5, 0>(wgt);
    }
  } else {
    threads = STEP_THREADS;
    kern = m <= 4 ? pick_step<1, 1>(wgt)
                  : m <= 8 ? pick_step<1, 2>(wgt) : m <= 12 ? pick_step<2, 3>(wgt) : pick_step<2, 4>(wgt);
  }
  // persistent grid: every CTA the SMs can hold (registers / shared memory)
  int per_sm = 1;
  if (int rc = prepare_kernel(reinterpret_cast<const void*>(kern), smem, threads, &per_sm))
    return rc;
  const int nchunks = (nrows + rc - 1) / rc;
  int gx = sm_count() * per_sm;
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  const int len = 2 * m + A.a * A.b;
  int werr = 0;
  double* part = static_cast<double*>(
      workspace((size_t)gx * len * sizeof(double), &werr, defer ? 1 : 0));
  if (werr) return werr;
  A.partial = part;
  kern<<<gx, threads, smem, st>>>(M, A, cf);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  if (defer) {   // the caller reduces (on a side stream, beside the stencil pass)
    defer->part = part;
    defer->nparts = gx;
    defer->len = len;
    defer->out = red_out;
    return 0;
  }
  return sum_parts(part, gx, len, red_out, st);
}

}  // namespace b2l

#ifdef B2L_TRACE
extern "C" int b2l_debug_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, b2l::g_trace, sizeof(b2l::g_trace));
}
#endif
