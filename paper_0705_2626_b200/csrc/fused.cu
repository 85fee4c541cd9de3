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
// Warp-specialised pipeline (no CTA-wide barrier inside the chunk loop):
//   warp 0 lane 0  TMA producer + storer: refills the NST-deep input ring and
//                  stores each finished output buffer;
//   warps 1..8     update + residual, one 8-row tile (all columns) per warp,
//                  so the residual of a row needs no other warp;
//   warps 9..16    Gram of the previous chunk's output buffer (double
//                  buffered), overlapping the update of the next chunk.
// mbarriers: full[s] (TMA -> update), empty[s] (update+Gram -> producer),
// ofull[b] (update -> Gram, storer), oempty[b] (Gram + store -> update).
//
// Shared-memory rows are padded to smem_stride(ld) doubles (4 or 12 mod 16):
// the TMA box is wider than the block's row, the extra columns are zero-filled
// on load and clipped on store, and the DMMA fragment loads are free of bank
// conflicts.  Out-of-range rows of the last chunk are zero-filled by the TMA.
#include "common.cuh"
#include "gram_tile.cuh"

#include <cstdio>
#include <cstdlib>

namespace b2l {

constexpr int STEP_NU = 8;                               // update warps
constexpr int STEP_NG = 8;                               // Gram warps
constexpr int STEP_THREADS = 32 * (1 + STEP_NU + STEP_NG);  // 544

struct StepMaps {
  CUtensorMap in[6];   // X AX W AW P AP          box (stride, rc)
  CUtensorMap out[5];  // X' AX' P' AP' W'        box (stride, rc)
};

struct StepArgs {
  int nrows, m, ldx;
  int kw, kp, kwn;
  int sx, sw, swn;      // shared-memory row strides (X-like, W, W')
  const double* d;      // diag(B) or null
  const double* tvec;
  const double* coef;   // [Cx m*m | Cw kw*m | Cp kp*m]
  const int* pcols;     // kp
  const int* wpos;      // m
  const double* lam;    // m
  int tmode;
  double tinv;
  int want_ax;
  int debug;           // B2L_STEP_DEBUG bits: 1 no update, 2 no residual, 4 no Gram
  int rc, nst;
  uint32_t stage_tx;    // TMA bytes per stage (full boxes)
  // shared-memory layout, in doubles
  int in_off[6];
  int d_off, t_off;
  int stage_doubles;
  int out_off[5];       // buffer 0
  int out_stride;       // doubles between the two output buffers
  int coef_off, lam_off, int_off;
  int bar_off, red_off, gred_off;
  // Gram of the next step
  int a, b;
  int lcum[4], rcum[5];
  int NI, NJ, tsI, tsJ, ts_per_cta, rs;
  unsigned tmask[32];
  double* partial;      // [gridDim.x][2m + a*b]
  unsigned long long* dbg;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TSTAMP(slot) \
  do { if ((A.debug & 8) && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && it < 64) A.dbg[it * 16 + (slot)] = gtime(); } while (0)

// Hardware named barriers for the output-buffer handoff: waiting warps sleep
// in the barrier unit instead of polling an mbarrier (polling cost a third of
// all issue slots).  Ids: 1,2 = buffer full; 3,4 = buffer empty.
constexpr int NB_OFULL = 1;
constexpr int NB_OEMPTY = 3;
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__global__ void __launch_bounds__(STEP_THREADS, 1)
    step_kernel(const __grid_constant__ StepMaps M, const __grid_constant__ StepArgs Ain) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  // Kernel parameters (1.7 KB with the tensor maps) overflow the constant
  // cache when the hot loops keep re-reading fields; keep a shared copy.
  __shared__ StepArgs sA;
  if (threadIdx.x == 0) sA = Ain;
  __syncthreads();
  const StepArgs& A = sA;
  double* sm = reinterpret_cast<double*>(sm_raw);
  double* stages = sm;
  double* coef = sm + A.coef_off;
  double* slam = sm + A.lam_off;
  int* spc = reinterpret_cast<int*>(sm + A.int_off);
  int* swp = spc + A.kp;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + A.bar_off);
  uint64_t* empty = full + 4;
  uint64_t* ofull = full + 8;
  uint64_t* oempty = full + 10;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int m = A.m;
  const int sx = A.sx, sw = A.sw, swn = A.swn;
  const int ncoef = m * m + A.kw * m + A.kp * m;
  for (int i = tid; i < ncoef; i += blockDim.x) coef[i] = A.coef[i];
  for (int i = tid; i < m; i += blockDim.x) {
    slam[i] = A.lam[i];
    swp[i] = A.wpos[i];
  }
  for (int i = tid; i < A.kp; i += blockDim.x) spc[i] = A.pcols[i];
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], STEP_NU + STEP_NG);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ofull[b], STEP_NU);
      mbar_init(&oempty[b], STEP_NG + 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const double* Cx = coef;
  const double* Cw = coef + m * m;
  const double* Cp = Cw + A.kw * m;

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  const int nloc = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk_of = [&](int it) { return blockIdx.x + it * gridDim.x; };

  // per-thread state carried to the final reduction
  double s_w0 = 0.0, s_w1 = 0.0, s_a0 = 0.0, s_a1 = 0.0;  // update warps: cols lane, lane+32
  WarpGram<2, 4> g;
  g.zero();
  const int gw = warp - 1 - STEP_NU;                        // Gram warp index
  const int tsl = gw >= 0 ? gw % A.ts_per_cta : 0;
  const int slice = gw >= 0 ? gw / A.ts_per_cta : 0;
  const bool gactive = gw >= 0 && slice < A.rs && tsl < A.tsI * A.tsJ;
  const int ti0 = gactive ? (tsl / A.tsJ) * 2 : 0;
  const int tj0 = gactive ? (tsl % A.tsJ) * 4 : 0;

  if (warp == 0) {
    // ================= producer / storer =================
    // whole warp runs the loop (named-barrier counts are per thread); lane 0
    // issues the TMA operations
    if (lane == 0)
      for (int j = 0; j < A.nst && j < nloc; ++j)
        step_issue(M, A, stages + (size_t)j * A.stage_doubles, &full[j], chunk_of(j));
    for (int it = 0; it < nloc; ++it) {
      const int b = it & 1;
      nbar_sync(NB_OFULL + b, STEP_THREADS);
      TSTAMP(0);
      if (lane == 0) {
        const int r0 = chunk_of(it) * A.rc;
        const int ob = b * A.out_stride;
        for (int k = 0; k < 5; ++k) {
          if (k == 4 && A.kwn == 0) continue;
          tma_store_2d(&M.out[k], sm + A.out_off[k] + ob, 0, r0);
        }
        bulk_commit();
        TSTAMP(1);
        // release this buffer as soon as its store has read it
        bulk_wait_read<0>();
        TSTAMP(2);
      }
      __syncwarp();
      nbar_arrive(NB_OEMPTY + b, STEP_THREADS);
      const int jn = it + A.nst;       // refill the stage chunk `it` used
      if (lane == 0 && jn < nloc) {
        const int s = it % A.nst;
        mbar_wait(&empty[s], (it / A.nst) & 1);
        TSTAMP(3);
        step_issue(M, A, stages + (size_t)s * A.stage_doubles, &full[s], chunk_of(jn));
        TSTAMP(4);
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();
  } else if (warp <= STEP_NU) {
    // ================= update + residual =================
    const int wu = warp - 1;
    const int NT = (m + 7) >> 3;
    const int q = lane & 3, rl = lane >> 2;
    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst, b = it & 1;
      const int r0 = chunk_of(it) * A.rc;
      const int nvalid = min(A.rc, A.nrows - r0);
      if (it >= 2) nbar_sync(NB_OEMPTY + b, STEP_THREADS);
      if (warp == 1) TSTAMP(5);
      mbar_wait_sleep(&full[s], (it / A.nst) & 1);
      if (warp == 1) TSTAMP(6);
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
        for (int nt = 0; nt < ((A.debug & 1) ? 0 : NT); ++nt) {
          const int cb = 8 * nt + rl;
          const bool cv = cb < m;
          double w0 = 0.0, w1 = 0.0, aw0 = 0.0, aw1 = 0.0, p0 = 0.0, p1 = 0.0;
          double ap0 = 0.0, ap1 = 0.0, x0 = 0.0, x1 = 0.0, ax0 = 0.0, ax1 = 0.0;
          // six independent DMMA chains per k-step; (W Cw) + (P Cp) and
          // (X Cx) + P' are added as the reference does
          // Branch-free: every chain runs kmax (all three K padded with zero
          // operands), so the DMMAs are unconditional (no per-DMMA warpsync)
          // and all nine operands of a k-step are loaded before its DMMAs.
          const int kmax = max(max(A.kw, A.kp), m);
#pragma unroll 2
          for (int k0 = 0; k0 < kmax; k0 += 4) {
            const int k = k0 + q;
            const bool kw_ok = k < A.kw, kp_ok = k < A.kp, km_ok = k < m;
            const int col = kp_ok ? spc[k] : 0;
            const double bw_ = (kw_ok && cv) ? Cw[k * m + cb] : 0.0;
            const double bp_ = (kp_ok && cv) ? Cp[k * m + cb] : 0.0;
            const double bx_ = (km_ok && cv) ? Cx[k * m + cb] : 0.0;
            const double wv = kw_ok ? W[r * sw + k] : 0.0;
            const double awv = kw_ok ? AW[r * sw + k] : 0.0;
            const double pv = kp_ok ? P[r * sx + col] : 0.0;
            const double apv = kp_ok ? AP[r * sx + col] : 0.0;
            const double xv = km_ok ? X[r * sx + k] : 0.0;
            const double axv = km_ok ? AX[r * sx + k] : 0.0;
            dmma_8x8x4(w0, w1, wv, bw_);
            dmma_8x8x4(aw0, aw1, awv, bw_);
            dmma_8x8x4(p0, p1, pv, bp_);
            dmma_8x8x4(ap0, ap1, apv, bp_);
            dmma_8x8x4(x0, x1, xv, bx_);
            dmma_8x8x4(ax0, ax1, axv, bx_);
          }
          const bool bw = A.kw > 0, bp = A.kp > 0;
          const double pn0 = (bw && bp) ? __dadd_rn(w0, p0) : (bw ? w0 : p0);
          const double pn1 = (bw && bp) ? __dadd_rn(w1, p1) : (bw ? w1 : p1);
          const double apn0 = (bw && bp) ? __dadd_rn(aw0, ap0) : (bw ? aw0 : ap0);
          const double apn1 = (bw && bp) ? __dadd_rn(aw1, ap1) : (bw ? aw1 : ap1);
          const int co = 8 * nt + 2 * q;
          const double vx[2] = {__dadd_rn(x0, pn0), __dadd_rn(x1, pn1)};
          const double vax[2] = {__dadd_rn(ax0, apn0), __dadd_rn(ax1, apn1)};
          const double vp[2] = {pn0, pn1};
          const double vap[2] = {apn0, apn1};
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (co + e < A.ldx) {
              O0[r * sx + co + e] = vx[e];
              O1[r * sx + co + e] = vax[e];
              O2[r * sx + co + e] = vp[e];
              O3[r * sx + co + e] = vap[e];
            }
          }
        }
        __syncwarp();
        if (warp == 1) TSTAMP(7);
        // residual of the 8 rows of this tile.  m <= 32: lane = (rsub, j),
        // RP = 32/m rows in flight per instruction; m > 32: lane owns
        // columns j and j+32.  Each lane's columns are fixed for the whole
        // kernel, so its norm partials accumulate in registers.
        if (!(A.debug & 2)) {
          const int RP = m <= 32 ? 32 / m : 1;
          const int rsub = m <= 32 ? lane / m : 0;
          const int j0 = m <= 32 ? lane % m : lane;
          const double lam0 = (rsub < RP && j0 < m) ? slam[j0] : 0.0;
          const double lam1 = (m > 32 && lane + 32 < m) ? slam[lane + 32] : 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = j0 + 32 * h;
            const bool on = h == 0 ? (rsub < RP && j0 < m) : (m > 32 && j < m);
            if (!on) continue;
            const double lam = h == 0 ? lam0 : lam1;
            const int jpos = swp[j];
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
          const int npad = swn - A.kwn;
          for (int e = lane; e < 8 * npad; e += 32)
            O4[(8 * mt + e / npad) * swn + A.kwn + e % npad] = 0.0;
        }
      }
      fence_async_smem();   // generic writes -> the TMA store (async proxy)
      if (warp == 1) TSTAMP(8);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      nbar_arrive(NB_OFULL + b, STEP_THREADS);
    }
    // balance the output-buffer barrier: consume the last two phases
    for (int it = (nloc > 2 ? nloc : 2); it < nloc + 2; ++it)
      nbar_sync(NB_OEMPTY + (it & 1), STEP_THREADS);
  } else {
    // ================= Gram of the finished output buffers =================
    const int Lblk[3] = {0, 4, 2};        // X', W', P' (indices into out_off)
    const int Rblk[4] = {0, 4, 2, 3};     // X', W', P', AP'
    LaneCol la[2], lb[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int ci = 8 * (ti0 + i) + (lane >> 2);
      la[i] = LaneCol{0, 0, false, false};
      if (gactive && ci < A.a) {
        int l = 0;
        while (l + 1 < 3 && A.lcum[l + 1] <= ci) ++l;
        la[i] = LaneCol{A.out_off[Lblk[l]] + (ci - A.lcum[l]), l == 1 ? swn : sx, true, false};
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cj = 8 * (tj0 + j) + (lane >> 2);
      lb[j] = LaneCol{0, 0, false, false};
      if (gactive && cj < A.b) {
        int r = 0;
        while (r + 1 < 4 && A.rcum[r + 1] <= cj) ++r;
        lb[j] = LaneCol{A.out_off[Rblk[r]] + (cj - A.rcum[r]), r == 1 ? swn : sx, true,
                        A.d != nullptr && r < 3};
      }
    }
    unsigned mask = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ti = ti0 + i, tj = tj0 + j;
        if (gactive && ti < A.NI && tj < A.NJ) {
          const int t = ti * A.NJ + tj;
          if ((A.tmask[t >> 5] >> (t & 31)) & 1u) mask |= 1u << (i * 4 + j);
        }
      }
    for (int it = 0; it < nloc; ++it) {
      const int s = it % A.nst, b = it & 1;
      const int r0 = chunk_of(it) * A.rc;
      const int nvalid = min(A.rc, A.nrows - r0);
      const int nv4 = (nvalid + 3) & ~3;
      nbar_sync(NB_OFULL + b, STEP_THREADS);
      if (warp == 1 + STEP_NU) TSTAMP(10);
      if (gactive && mask && !(A.debug & 4)) {
        const double* st = stages + (size_t)s * A.stage_doubles;
        const int rps = A.rc / A.rs;
        const int lo = slice * rps;
        const int hi = min(lo + rps, nv4);
        g.run(sm + b * A.out_stride, la, lb, A.d ? st + A.d_off : nullptr, lo, hi, mask,
              DenseRows());
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      nbar_arrive(NB_OEMPTY + b, STEP_THREADS);
      if (warp == 1 + STEP_NU) TSTAMP(11);
    }
  }
  __syncthreads();

  // ---- CTA reduction: residual sums (fixed order over update warps)
  // red layout: [4][STEP_NU][32] = s_w0, s_a0, s_w1, s_a1 per (warp, lane)
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
    double a = 0.0, b = 0.0;
    const int RP = m <= 32 ? 32 / m : 1;
    for (int q = 0; q < STEP_NU; ++q) {
      if (m <= 32) {
        for (int rs_ = 0; rs_ < RP; ++rs_) {
          a += red[q * 32 + rs_ * m + tid];
          b += red[NL + q * 32 + rs_ * m + tid];
        }
      } else {
        const int h = tid >= 32;
        a += red[2 * h * NL + q * 32 + (tid & 31)];
        b += red[(2 * h + 1) * NL + q * 32 + (tid & 31)];
      }
    }
    out[tid] = a;
    out[m + tid] = b;
  }
  __syncthreads();
  // ---- Gram: fixed-order sum of row slices
  double* gred = sm + A.gred_off;
  if (gactive && slice > 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const size_t o = ((((size_t)(slice - 1) * A.ts_per_cta + tsl) * 8 + i * 4 + j) * 32 + lane) * 2;
        gred[o] = g.acc[i][j][0];
        gred[o + 1] = g.acc[i][j][1];
      }
  }
  __syncthreads();
  if (gactive && slice == 0) {
    double* go = out + 2 * m;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double v0 = g.acc[i][j][0], v1 = g.acc[i][j][1];
        for (int sl = 1; sl < A.rs; ++sl) {
          const size_t o = ((((size_t)(sl - 1) * A.ts_per_cta + tsl) * 8 + i * 4 + j) * 32 + lane) * 2;
          v0 += gred[o];
          v1 += gred[o + 1];
        }
        const int row = 8 * (ti0 + i) + (lane >> 2);
        const int col = 8 * (tj0 + j) + 2 * (lane & 3);
        if (row < A.a) {
          if (col < A.b) go[(size_t)row * A.b + col] = v0;
          if (col + 1 < A.b) go[(size_t)row * A.b + col + 1] = v1;
        }
      }
  }
}

__global__ void sum_parts_kernel(const double* partial, int nparts, int len, double* out);

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

int lobpcg_step(int nrows, int m, const double* x, const double* ax, int ldx,
                const double* w, const double* aw, int ldw, int kw, const double* p,
                const double* ap, int kp, const int* pcols, const double* coef,
                double* xo, double* axo, double* po, double* apo, const double* lam,
                const double* d, int tmode, double tinv, const double* tvec,
                const int* wpos, int kwn, double* wo, int ldwn, int want_ax,
                double* red_out, cudaStream_t st) {
  B2L_CHECK(m >= 1 && m <= 64, -B2L_EINVAL, "step: 1 <= m <= 64");
  B2L_CHECK(nrows >= 1, -B2L_EINVAL, "step: empty block");
  B2L_CHECK(ldx >= m && (ldx & 1) == 0, -B2L_EINVAL, "step: ldx must be even and >= m");
  B2L_CHECK(kw >= 0 && kw <= ldw && (kw == 0 || (ldw & 1) == 0), -B2L_EINVAL, "step: bad W");
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
  A.sw = kw ? smem_stride(ldw) : 0;
  A.swn = smem_stride(kwn ? ldwn : 2);
  A.d = d;
  A.tvec = tvec;
  A.coef = coef;
  A.pcols = pcols;
  A.wpos = wpos;
  A.lam = lam;
  A.tmode = tmode;
  A.tinv = tinv;
  A.want_ax = want_ax;
  A.debug = getenv("B2L_STEP_DEBUG") ? atoi(getenv("B2L_STEP_DEBUG")) : 0;
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
  B2L_CHECK(A.NI * A.NJ <= 1024, -B2L_EINVAL, "step: Gram too large");
  static const unsigned char modes[12] = {2, 1, 1, 1, 0, 2, 1, 1, 0, 0, 2, 1};
  tile_mask(A.NI, A.NJ, A.lcum, 3, A.rcum, 4, modes, A.tmask);
  A.tsI = (A.NI + 1) / 2;
  A.tsJ = (A.NJ + 3) / 4;
  const int TS = A.tsI * A.tsJ;
  B2L_CHECK(TS <= STEP_NG, -B2L_EINVAL, "step: Gram tile blocks exceed one CTA (m too large)");
  A.ts_per_cta = TS;
  A.rs = 1;
  while (A.rs * 2 * TS <= STEP_NG) A.rs *= 2;
  // chunk rows (multiple of 16): 8 update warps x 8-row tiles = 64 rows, or
  // fewer when a stage (6 blocks + d + t) would exceed ~48 KB; then the
  // deepest TMA ring (<= 4 stages) that fits one CTA per SM.
  const int width = 4 * A.sx + 2 * A.sw + (d ? 1 : 0) + (tmode == 2 ? 1 : 0);
  A.rc = getenv("B2L_RC") ? atoi(getenv("B2L_RC")) : 64;
  while (A.rc > 16 && (size_t)A.rc * width * 8 > 48 * 1024) A.rc >>= 1;
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
  {
    const size_t tail = (size_t)2 * (4 * tile_x + tile_w) + (m * m + kw * m + kp * m) + 3 * m +
                        64 + (size_t)2 * STEP_NU * m + 64;
    A.nst = getenv("B2L_NST") ? atoi(getenv("B2L_NST")) : 4;
    while (A.nst > 2 && ((size_t)A.nst * A.stage_doubles + tail) * 8 > 210 * 1024) --A.nst;
  }
  off = A.nst * A.stage_doubles;
  for (int b = 0; b < 4; ++b) {
    A.out_off[b] = off;
    off += tile_x;
  }
  A.out_off[4] = off;
  off += tile_w;
  A.out_stride = off - A.out_off[0];
  off += A.out_stride;  // second output buffer
  A.coef_off = off;
  off += (m * m + kw * m + kp * m + 1) & ~1;
  A.lam_off = off;
  off += (m + 1) & ~1;
  A.int_off = off;
  off += (kp + m + 1) / 2 + 1;
  off = (off + 15) & ~15;
  A.bar_off = off;
  off += 16;  // 12 mbarriers
  A.red_off = off;
  const size_t red1 = (size_t)4 * STEP_NU * 32;
  const size_t red2 = (size_t)(A.rs > 1 ? A.rs - 1 : 0) * A.ts_per_cta * 8 * 64;
  // the Gram slice reduction reuses the (idle) stage ring after the loop
  if (red2 <= (size_t)A.nst * A.stage_doubles) {
    A.gred_off = 0;
    off += (int)red1;
  } else {
    A.gred_off = A.red_off;
    off += (int)(red1 > red2 ? red1 : red2);
  }
  const size_t smem = (size_t)off * 8;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "step: shared memory budget exceeded");

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

  const int nchunks = (nrows + rc - 1) / rc;
  int gx = sm_count();
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  const int len = 2 * m + A.a * A.b;
  int werr = 0;
  double* part = static_cast<double*>(workspace((size_t)gx * len * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  static unsigned long long* dbgbuf = nullptr;
  if (A.debug & 8) {
    if (!dbgbuf) cudaMalloc(&dbgbuf, 64 * 16 * 8);
    cudaMemsetAsync(dbgbuf, 0, 64 * 16 * 8, st);
    A.dbg = dbgbuf;
  }
  B2L_CUDA(cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  step_kernel<<<gx, STEP_THREADS, smem, st>>>(M, A);
  B2L_CUDA(cudaGetLastError());
  if (A.debug & 8) {
    unsigned long long h[64 * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbgbuf, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long t0 = h[6];
    for (int i = 0; i < 24; ++i) {
      fprintf(stderr, "it %2d:", i);
      for (int k = 0; k < 12; ++k)
        fprintf(stderr, " %7lld", h[i * 16 + k] ? (long long)(h[i * 16 + k] - t0) : -1LL);
      fprintf(stderr, "\n");
    }
  }
  sum_parts_kernel<<<(len + 255) / 256, 256, 0, st>>>(part, gx, len, red_out);
  B2L_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace b2l
