// F1: one fused pass per LOBPCG iteration over the tall blocks (sm_100a).
//
// For a chunk of rows, staged in shared memory by 1-D TMA bulk copies:
//   (1) Ritz update (reference lobpcg.py:520-540, multivec.multiply :74-86)
//         P'  = W Cw + P[:, J] Cp        AP' = AW Cw + AP[:, J] Cp
//         X'  = X Cx + P'                AX' = AX Cx + AP'
//       with the Cholesky-QR factors of W and P already folded into Cw/Cp
//       (replaces tri_solve_right, multivec.py:125-146);
//   (2) the NEXT iteration's residual block and lock norms
//       (lobpcg.py:429-430, :466-467): W'_J = T (AX' - BX' Lambda'),
//       sum of squares of every residual column (and of AX' for relative tol);
//   (3) every Gram product of the next Rayleigh-Ritz step that does not
//       involve A W' (lobpcg.py:419 drift, :176 W/P orthonormalisation,
//       :328-338 pencil blocks): [X' W' P']^T B [X' W' P'] (upper) and
//       [X' W' P']^T AP', on the fp64 tensor cores (DMMA).
// X', AX', P', AP', W' are written back with TMA bulk stores.  Each row is read
// once and written once per iteration; the only other pass is the stencil
// (stencil.cu), which also produces [X' W']^T A W'.
#include "common.cuh"
#include "gram_tile.cuh"

namespace b2l {

constexpr int STEP_THREADS = 512;

struct StepArgs {
  int nrows, m, ldx;
  int kw, ldw, kp, kwn, ldwn;
  const double *x, *ax, *w, *aw, *p, *ap;
  double *xo, *axo, *po, *apo, *wo;
  const double* coef;   // [Cx m*m | Cw kw*m | Cp kp*m]
  const int* pcols;     // kp
  const int* wpos;      // m
  const double* lam;    // m
  const double* d;      // diag(B) or null
  int tmode;
  double tinv;
  const double* tvec;
  int want_ax;
  int rc, nst;
  // shared-memory layout, in doubles
  int in_off[6];        // X AX W AW P AP inside a stage
  int d_off, t_off;     // staged d / tvec inside a stage
  int stage_doubles;
  int out_off[5];       // X' AX' P' AP' W' (dense tiles, buffer 0)
  int out_stride;       // doubles between the two output-tile buffers
  int coef_off, lam_off, int_off;  // coefficient block, lam, ints (pcols|wpos)
  int red_off;
  int gred_off;         // Gram row-slice reduction (stage ring when it fits)
  // Gram of the next step
  int a, b;
  int lcum[4], rcum[5];
  int NI, NJ, tsI, tsJ, ts_per_cta, rs;
  unsigned tmask[32];
  double* partial;      // [gridDim.x][2m + a*b]
};

__device__ __forceinline__ void step_issue(const StepArgs& A, double* st, uint64_t* bar, int c) {
  const int r0 = c * A.rc;
  const int nvalid = min(A.rc, A.nrows - r0);
  const double* src[6] = {A.x, A.ax, A.w, A.aw, A.p, A.ap};
  const int ld[6] = {A.ldx, A.ldx, A.ldw, A.ldw, A.ldx, A.ldx};
  const bool on[6] = {true, true, A.kw > 0, A.kw > 0, A.kp > 0, A.kp > 0};
  uint32_t tx = 0;
  for (int b = 0; b < 6; ++b)
    if (on[b]) tx += (uint32_t)nvalid * ld[b] * 8u;
  const bool even = (nvalid % 2) == 0;
  const int nv4 = (nvalid + 3) & ~3;
  if (A.d) {
    if (even) tx += (uint32_t)nvalid * 8u;
    else
      for (int e = 0; e < nvalid; ++e) st[A.d_off + e] = A.d[r0 + e];
    for (int e = nvalid; e < nv4; ++e) st[A.d_off + e] = 0.0;  // tail rows feed the Gram
  }
  if (A.tmode == 2) {
    if (even) tx += (uint32_t)nvalid * 8u;
    else
      for (int e = 0; e < nvalid; ++e) st[A.t_off + e] = A.tvec[r0 + e];
  }
  fence_async_smem();
  mbar_expect_tx(bar, tx);
  for (int b = 0; b < 6; ++b)
    if (on[b])
      bulk_load(st + A.in_off[b], src[b] + (size_t)r0 * ld[b], (uint32_t)nvalid * ld[b] * 8u, bar);
  if (A.d && even) bulk_load(st + A.d_off, A.d + r0, (uint32_t)nvalid * 8u, bar);
  if (A.tmode == 2 && even) bulk_load(st + A.t_off, A.tvec + r0, (uint32_t)nvalid * 8u, bar);
}

__global__ void __launch_bounds__(STEP_THREADS) step_kernel(StepArgs A) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  double* sm = reinterpret_cast<double*>(sm_raw);
  double* stages = sm;
  double* O[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) O[i] = sm + A.out_off[i];
  double* coef = sm + A.coef_off;
  double* slam = sm + A.lam_off;
  int* spc = reinterpret_cast<int*>(sm + A.int_off);
  int* swp = spc + A.kp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + A.red_off) - 8;  // 8 barriers before red

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int m = A.m;
  const int ncoef = m * m + A.kw * m + A.kp * m;
  for (int i = tid; i < ncoef; i += blockDim.x) coef[i] = A.coef[i];
  for (int i = tid; i < m; i += blockDim.x) {
    slam[i] = A.lam[i];
    swp[i] = A.wpos[i];
  }
  for (int i = tid; i < A.kp; i += blockDim.x) spc[i] = A.pcols[i];
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const double* Cx = coef;
  const double* Cw = coef + m * m;
  const double* Cp = Cw + A.kw * m;

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  if (tid == 0)
    for (int s = 0; s < A.nst; ++s) {
      const int c = blockIdx.x + s * gridDim.x;
      if (c < nchunks) step_issue(A, stages + (size_t)s * A.stage_doubles, &bar[s], c);
    }

  // ---- Gram job of this warp (tile block x row slice), fixed for the kernel
  const int tsl = warp % A.ts_per_cta;
  const int slice = warp / A.ts_per_cta;
  const bool gactive = slice < A.rs && tsl < A.tsI * A.tsJ;
  const int ti0 = gactive ? (tsl / A.tsJ) * 2 : 0;
  const int tj0 = gactive ? (tsl % A.tsJ) * 4 : 0;
  const int Lblk[3] = {0, 4, 2};        // X', W', P' (indices into O)
  const int Rblk[4] = {0, 4, 2, 3};     // X', W', P', AP'
  LaneCol la[2], lb[4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int ci = 8 * (ti0 + i) + (lane >> 2);
    la[i] = LaneCol{0, 0, false, false};
    if (ci < A.a) {
      int l = 0;
      while (l + 1 < 3 && A.lcum[l + 1] <= ci) ++l;
      la[i] = LaneCol{A.out_off[Lblk[l]] + (ci - A.lcum[l]), l == 1 ? A.ldwn : A.ldx, true, false};
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = 8 * (tj0 + j) + (lane >> 2);
    lb[j] = LaneCol{0, 0, false, false};
    if (cj < A.b) {
      int r = 0;
      while (r + 1 < 4 && A.rcum[r + 1] <= cj) ++r;
      lb[j] = LaneCol{A.out_off[Rblk[r]] + (cj - A.rcum[r]), r == 1 ? A.ldwn : A.ldx, true,
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
  WarpGram<2, 4> g;
  g.zero();

  // ---- residual lanes: fixed column per thread
  const int rpp = STEP_THREADS / m;          // rows per pass
  const int rj = tid % m;
  const int rr0 = tid / m;
  const bool ron = rr0 < rpp;
  double s_w = 0.0, s_a = 0.0;
  const int jpos = ron ? swp[rj] : -1;

  int it = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int s = it % A.nst;
    double* st = stages + (size_t)s * A.stage_doubles;
    const int r0 = c * A.rc;
    const int nvalid = min(A.rc, A.nrows - r0);
    const int nv4 = (nvalid + 3) & ~3;
    // output tiles alternate between two buffers so a chunk never waits for
    // the TMA store of the previous one to drain
    const int ob = (it & 1) * A.out_stride;
#pragma unroll
    for (int i = 0; i < 5; ++i) O[i] = sm + A.out_off[i] + ob;
    mbar_wait(&bar[s], (it / A.nst) & 1);
    const double* X = st + A.in_off[0];
    const double* AX = st + A.in_off[1];
    const double* W = st + A.in_off[2];
    const double* AW = st + A.in_off[3];
    const double* P = st + A.in_off[4];
    const double* AP = st + A.in_off[5];

    // (1) update on the fp64 tensor cores: one warp per 8-row x 8-column
    //     output tile, separate DMMA chains for W Cw, P_J Cp and X Cx so the
    //     sums are formed as in the reference, (W Cw) + (P Cp) then
    //     (X Cx) + P'.  Rows >= nvalid come out zero (the tail chunk's 4-row
    //     Gram groups read them); pad columns m..ldx-1 come out zero.
    {
      const int NT = (m + 7) >> 3;
      const int npairs = (A.rc >> 3) * NT;
      const int q = lane & 3, rl = lane >> 2;
      for (int pr = warp; pr < npairs; pr += STEP_THREADS / 32) {
        const int mt = pr / NT, nt = pr - (pr / NT) * NT;
        const int r = 8 * mt + rl;
        const bool rv = r < nvalid;
        const int cb = 8 * nt + rl;
        const bool cv = cb < m;
        double w0 = 0.0, w1 = 0.0, aw0 = 0.0, aw1 = 0.0, p0 = 0.0, p1 = 0.0;
        double ap0 = 0.0, ap1 = 0.0, x0 = 0.0, x1 = 0.0, ax0 = 0.0, ax1 = 0.0;
        for (int k0 = 0; k0 < A.kw; k0 += 4) {
          const int k = k0 + q;
          const bool kv = k < A.kw;
          const double bcoef = (kv && cv) ? Cw[k * m + cb] : 0.0;
          const double av = (kv && rv) ? W[r * A.ldw + k] : 0.0;
          const double aav = (kv && rv) ? AW[r * A.ldw + k] : 0.0;
          dmma_8x8x4(w0, w1, av, bcoef);
          dmma_8x8x4(aw0, aw1, aav, bcoef);
        }
        for (int k0 = 0; k0 < A.kp; k0 += 4) {
          const int k = k0 + q;
          const bool kv = k < A.kp;
          const int col = kv ? spc[k] : 0;
          const double bcoef = (kv && cv) ? Cp[k * m + cb] : 0.0;
          const double av = (kv && rv) ? P[r * A.ldx + col] : 0.0;
          const double aav = (kv && rv) ? AP[r * A.ldx + col] : 0.0;
          dmma_8x8x4(p0, p1, av, bcoef);
          dmma_8x8x4(ap0, ap1, aav, bcoef);
        }
        for (int k0 = 0; k0 < m; k0 += 4) {
          const int k = k0 + q;
          const bool kv = k < m;
          const double bcoef = (kv && cv) ? Cx[k * m + cb] : 0.0;
          const double av = (kv && rv) ? X[r * A.ldx + k] : 0.0;
          const double aav = (kv && rv) ? AX[r * A.ldx + k] : 0.0;
          dmma_8x8x4(x0, x1, av, bcoef);
          dmma_8x8x4(ax0, ax1, aav, bcoef);
        }
        const bool bw = A.kw > 0, bp = A.kp > 0;
        const double pn0 = (bw && bp) ? __dadd_rn(w0, p0) : (bw ? w0 : p0);
        const double pn1 = (bw && bp) ? __dadd_rn(w1, p1) : (bw ? w1 : p1);
        const double apn0 = (bw && bp) ? __dadd_rn(aw0, ap0) : (bw ? aw0 : ap0);
        const double apn1 = (bw && bp) ? __dadd_rn(aw1, ap1) : (bw ? aw1 : ap1);
        const int ro = 8 * mt + rl;
        const int co = 8 * nt + 2 * q;
        const double vx[2] = {__dadd_rn(x0, pn0), __dadd_rn(x1, pn1)};
        const double vax[2] = {__dadd_rn(ax0, apn0), __dadd_rn(ax1, apn1)};
        const double vp[2] = {pn0, pn1};
        const double vap[2] = {apn0, apn1};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (co + e < A.ldx) {
            O[0][ro * A.ldx + co + e] = vx[e];
            O[1][ro * A.ldx + co + e] = vax[e];
            O[2][ro * A.ldx + co + e] = vp[e];
            O[3][ro * A.ldx + co + e] = vap[e];
          }
        }
      }
    }
    __syncthreads();

    // (2) residual of the next iteration, W' for the active columns, norms
    if (ron) {
      const double lam = slam[rj];
      for (int r = rr0; r < nv4; r += rpp) {
        double wv = 0.0;
        if (r < nvalid) {
          const double xv = O[0][r * A.ldx + rj];
          const double av = O[1][r * A.ldx + rj];
          const double bx = A.d ? __dmul_rn(st[A.d_off + r], xv) : xv;
          const double wf = __dsub_rn(av, __dmul_rn(bx, lam));
          s_w = fma(wf, wf, s_w);
          if (A.want_ax) s_a = fma(av, av, s_a);
          wv = wf;
          if (A.tmode == 1) wv = __dmul_rn(A.tinv, wf);
          else if (A.tmode == 2) wv = __dmul_rn(st[A.t_off + r], wf);
        }
        if (jpos >= 0) {
          O[4][r * A.ldwn + jpos] = wv;
          if (jpos == A.kwn - 1)
            for (int e2 = A.kwn; e2 < A.ldwn; ++e2) O[4][r * A.ldwn + e2] = 0.0;
        }
      }
    }
    __syncthreads();

    // write back the chunk (async), refill the input stage
    if (tid == 0) {
      fence_async_smem();
      double* dst[5] = {A.xo, A.axo, A.po, A.apo, A.wo};
      const int ld[5] = {A.ldx, A.ldx, A.ldx, A.ldx, A.ldwn};
      for (int b = 0; b < 5; ++b) {
        if (b == 4 && A.kwn == 0) continue;
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                dst[b] + (size_t)r0 * ld[b]),
            "r"(smem_u32(O[b])), "r"((uint32_t)nvalid * ld[b] * 8u)
            : "memory");
      }
      bulk_commit();
    }

    // (3) Gram of the next step from the output tiles
    if (gactive && mask) {
      const int rps = A.rc / A.rs;
      const int lo = slice * rps;
      const int hi = min(lo + rps, nv4);
      g.run(sm + ob, la, lb, A.d ? st + A.d_off : nullptr, lo, hi, mask, DenseRows());
    }
    // output tiles are rewritten by the next chunk: wait for the bulk store
    // to have read them and for every warp's Gram; then refill this stage
    // (its d chunk was in use by the Gram until here)
    if (tid == 0) bulk_wait_read<1>();
    __syncthreads();
    if (tid == 0) {
      const int cn = c + A.nst * gridDim.x;
      if (cn < nchunks) step_issue(A, st, &bar[s], cn);
    }
  }
  if (tid == 0) bulk_wait<0>();

  // ---- CTA reduction: residual sums (fixed order over row lanes)
  double* red = sm + A.red_off;
  if (ron) {
    red[rr0 * m + rj] = s_w;
    red[(rpp + rr0) * m + rj] = s_a;
  }
  __syncthreads();
  double* out = A.partial + (size_t)blockIdx.x * (2 * m + A.a * A.b);
  if (tid < m) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < rpp; ++q) {
      a += red[q * m + tid];
      b += red[(rpp + q) * m + tid];
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
  A.ldw = kw ? ldw : 0;
  A.kp = kp;
  A.kwn = kwn;
  A.ldwn = kwn ? ldwn : 2;
  A.x = x;
  A.ax = ax;
  A.w = w;
  A.aw = aw;
  A.p = p;
  A.ap = ap;
  A.xo = xo;
  A.axo = axo;
  A.po = po;
  A.apo = apo;
  A.wo = wo;
  A.coef = coef;
  A.pcols = pcols;
  A.wpos = wpos;
  A.lam = lam;
  A.d = d;
  A.tmode = tmode;
  A.tinv = tinv;
  A.tvec = tvec;
  A.want_ax = want_ax;
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
  const int nwarps = STEP_THREADS / 32;
  B2L_CHECK(TS <= nwarps, -B2L_EINVAL, "step: Gram tile blocks exceed one CTA (m too large)");
  A.ts_per_cta = TS;
  A.rs = 1;
  while (A.rs * 2 * TS <= nwarps) A.rs *= 2;
  // chunk rows (multiple of 8: one DMMA row tile per 8 rows): stage (6
  // blocks + d + t) <= ~40 KB; then the deepest TMA ring (<= 4 stages) that
  // fits one CTA per SM.
  const int width = 4 * ldx + 2 * (kw ? ldw : 0) + (d ? 1 : 0) + (tmode == 2 ? 1 : 0);
  A.rc = 128;
  while (A.rc > 16 && (size_t)A.rc * width * 8 > 40 * 1024) A.rc >>= 1;
  while (A.rs > 1 && A.rc / A.rs < 4) A.rs >>= 1;
  const int rc = A.rc;
  int off = 0;
  A.in_off[0] = off; off += rc * ldx;
  A.in_off[1] = off; off += rc * ldx;
  A.in_off[2] = off; off += kw ? rc * ldw : 0;
  A.in_off[3] = off; off += kw ? rc * ldw : 0;
  A.in_off[4] = off; off += kp ? rc * ldx : 0;
  A.in_off[5] = off; off += kp ? rc * ldx : 0;
  A.d_off = off; off += d ? rc : 0;
  A.t_off = off; off += tmode == 2 ? rc : 0;
  A.stage_doubles = (off + 15) & ~15;
  {
    const size_t tail = (size_t)2 * (4 * ((rc * ldx + 15) & ~15) + ((rc * A.ldwn + 15) & ~15)) +
                        (m * m + kw * m + kp * m) + 3 * m + 64 +
                        (size_t)(STEP_THREADS / m) * 2 * m + 4096;
    A.nst = 4;
    while (A.nst > 2 && ((size_t)A.nst * A.stage_doubles + tail) * 8 > 200 * 1024) --A.nst;
  }
  off = A.nst * A.stage_doubles;
  for (int b = 0; b < 4; ++b) {
    A.out_off[b] = off;
    off += (rc * ldx + 15) & ~15;
  }
  A.out_off[4] = off;
  off += (rc * A.ldwn + 15) & ~15;
  A.out_stride = off - A.out_off[0];
  off += A.out_stride;  // second output buffer
  A.coef_off = off;
  off += (m * m + kw * m + kp * m + 1) & ~1;
  A.lam_off = off;
  off += (m + 1) & ~1;
  A.int_off = off;
  off += (kp + m + 1) / 2 + 1;
  off = (off + 15) & ~15;
  off += 16;  // 8 mbarriers
  A.red_off = off;
  const int rpp = STEP_THREADS / m;
  const size_t red1 = (size_t)2 * rpp * m;
  const size_t red2 = (size_t)(A.rs > 1 ? A.rs - 1 : 0) * A.ts_per_cta * 8 * 64;
  // the Gram slice reduction may reuse the (idle) stage ring after the loop
  const size_t red_stage = (size_t)A.nst * A.stage_doubles;
  if (red2 <= red_stage) {
    A.gred_off = 0;
    off += (int)red1;
  } else {
    A.gred_off = A.red_off;
    off += (int)(red1 > red2 ? red1 : red2);
  }
  const size_t smem = (size_t)off * 8;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "step: shared memory budget exceeded");
  const int nchunks = (nrows + rc - 1) / rc;
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  int gx = per_sm * sm_count();
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  const int len = 2 * m + A.a * A.b;
  int werr = 0;
  double* part = static_cast<double*>(workspace((size_t)gx * len * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  B2L_CUDA(cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  step_kernel<<<gx, STEP_THREADS, smem, st>>>(A);
  B2L_CUDA(cudaGetLastError());
  sum_parts_kernel<<<(len + 255) / 256, 256, 0, st>>>(part, gx, len, red_out);
  B2L_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace b2l
