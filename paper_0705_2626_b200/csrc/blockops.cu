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
//                   multivec.py:125-146)
//
// Every reduction is deterministic: CTA partials in a fixed row assignment,
// then a fixed-order second stage over CTAs.
#include "common.cuh"

namespace b2l {

// =========================================================================
// K5: multi-block Gram
// =========================================================================
constexpr int GRAM_THREADS = 256;
constexpr int GRAM_MAXU = 8;
constexpr int GRAM_MAXL = 4;
constexpr int GRAM_MAXR = 8;

struct GramArgs {
  int nrows;
  int rc;      // rows per chunk
  int nu;      // unique blocks staged per chunk
  const double* up[GRAM_MAXU];
  int uld[GRAM_MAXU];
  int usld[GRAM_MAXU];   // smem row stride (multiple of 4)
  int ubase[GRAM_MAXU];  // smem offset (doubles) of the block region
  int nl, nr;
  int lu[GRAM_MAXL], lvoff[GRAM_MAXL];  // unique id, padded column offset
  int ru[GRAM_MAXR], rvoff[GRAM_MAXR];
  unsigned rw_mask;  // right block j is weighted by d
  const double* d;
  int dbase;         // smem offset of the staged d chunk
  int stage_doubles;
  int a_pad, b_pad;  // padded virtual sizes (multiples of 4)
  int tiles_n;       // b_pad / 4
  int ntiles;        // (a_pad/4) * tiles_n
  int tset;          // tiles per CTA (blockIdx.y selects the set)
  int G;             // row groups
  double* partial;   // [gridDim.x][a_pad * b_pad]
};

__device__ __forceinline__ void gram_load_chunk(const GramArgs& A, double* st,
                                                int r0) {
  const int tid = threadIdx.x;
  const int nvalid = min(A.rc, A.nrows - r0);
  for (int u = 0; u < A.nu; ++u) {
    const int h = A.uld[u] >> 1;  // double2 per row
    const int sld = A.usld[u];
    double* dst = st + A.ubase[u];
    const double* src = A.up[u] + (size_t)r0 * A.uld[u];
    const int total = A.rc * h;
    for (int f = tid; f < total; f += blockDim.x) {
      const int row = f / h;
      const int c2 = f - row * h;
      double* dptr = dst + row * sld + 2 * c2;
      if (row < nvalid)
        cp_async16(dptr, src + (size_t)row * A.uld[u] + 2 * c2);
      else
        *reinterpret_cast<double2*>(dptr) = make_double2(0.0, 0.0);
    }
  }
  if (A.d) {
    for (int row = tid; row < A.rc; row += blockDim.x)
      st[A.dbase + row] = row < nvalid ? A.d[r0 + row] : 0.0;
  }
}

__global__ void __launch_bounds__(GRAM_THREADS) gram_kernel(GramArgs A) {
  extern __shared__ __align__(128) double gsm[];
  double* st0 = gsm;
  double* st1 = gsm + A.stage_doubles;
  const int tid = threadIdx.x;

  // zero both stages once (pad columns stay zero forever)
  for (int i = tid; i < 2 * A.stage_doubles; i += blockDim.x) gsm[i] = 0.0;
  __syncthreads();

  const int tl = tid % A.tset;
  const int g = tid / A.tset;
  const int t = blockIdx.y * A.tset + tl;
  const bool active = (g < A.G) && (tl < A.tset) && (t < A.ntiles);

  int loff = 0, lsld = 4, roff = 0, rsld = 4;
  bool wgt = false;
  int i0 = 0, j0 = 0;
  if (active) {
    i0 = 4 * (t / A.tiles_n);
    j0 = 4 * (t % A.tiles_n);
    int l = 0;
    while (l + 1 < A.nl && A.lvoff[l + 1] <= i0) ++l;
    loff = A.ubase[A.lu[l]] + (i0 - A.lvoff[l]);
    lsld = A.usld[A.lu[l]];
    int r = 0;
    while (r + 1 < A.nr && A.rvoff[r + 1] <= j0) ++r;
    roff = A.ubase[A.ru[r]] + (j0 - A.rvoff[r]);
    rsld = A.usld[A.ru[r]];
    wgt = (A.rw_mask >> r) & 1u;
  }

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  const int nchunks = (A.nrows + A.rc - 1) / A.rc;
  int c = blockIdx.x;
  if (c < nchunks) gram_load_chunk(A, st0, c * A.rc);
  cp_async_commit();
  double* cur = st0;
  double* nxt = st1;
  for (; c < nchunks; c += gridDim.x) {
    const int cn = c + gridDim.x;
    if (cn < nchunks) gram_load_chunk(A, nxt, cn * A.rc);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (active) {
      const double* Ls = cur + loff;
      const double* Rs = cur + roff;
      const double* ds = cur + A.dbase;
      for (int r = g; r < A.rc; r += A.G) {
        const double2 a01 = *reinterpret_cast<const double2*>(Ls + r * lsld);
        const double2 a23 = *reinterpret_cast<const double2*>(Ls + r * lsld + 2);
        double2 b01 = *reinterpret_cast<const double2*>(Rs + r * rsld);
        double2 b23 = *reinterpret_cast<const double2*>(Rs + r * rsld + 2);
        if (wgt) {
          const double w = ds[r];
          b01.x = __dmul_rn(w, b01.x);
          b01.y = __dmul_rn(w, b01.y);
          b23.x = __dmul_rn(w, b23.x);
          b23.y = __dmul_rn(w, b23.y);
        }
        const double a[4] = {a01.x, a01.y, a23.x, a23.y};
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  cp_async_wait<0>();
  __syncthreads();

  // reduce the G row groups in fixed order (reuse stage memory)
  double* red = gsm;
  if (active && g > 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[((g - 1) * A.tset + tl) * 16 + i * 4 + j] = acc[i][j];
  }
  __syncthreads();
  if (active && g == 0) {
    for (int gg = 1; gg < A.G; ++gg)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += red[((gg - 1) * A.tset + tl) * 16 + i * 4 + j];
    double* out = A.partial + (size_t)blockIdx.x * A.a_pad * A.b_pad;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) out[(i0 + i) * A.b_pad + j0 + j] = acc[i][j];
  }
}

struct GramMap {
  int nl, nr;
  int lcols[GRAM_MAXL], lvoff[GRAM_MAXL];
  int rcols[GRAM_MAXR], rvoff[GRAM_MAXR];
  int a, b, a_pad, b_pad;
};

// second stage: fixed-order sum over CTA partials, padded -> compact (a x b)
__global__ void gram_reduce_kernel(const double* partial, int nparts, GramMap M,
                                   double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.a * M.b) return;
  int i = e / M.b, j = e - (e / M.b) * M.b;
  int pi = 0, pj = 0;
  for (int l = 0, cum = 0; l < M.nl; cum += M.lcols[l], ++l)
    if (i >= cum && i < cum + M.lcols[l]) pi = M.lvoff[l] + (i - cum);
  for (int r = 0, cum = 0; r < M.nr; cum += M.rcols[r], ++r)
    if (j >= cum && j < cum + M.rcols[r]) pj = M.rvoff[r] + (j - cum);
  const size_t stride = (size_t)M.a_pad * M.b_pad;
  const size_t idx = (size_t)pi * M.b_pad + pj;
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += partial[c * stride + idx];
  out[e] = s;
}

struct HostBlock {
  const double* p;
  int ld, cols;
};

int gram(int nrows, const HostBlock* L, int nl, const HostBlock* R, int nr,
         unsigned rw_mask, const double* d, double* out, cudaStream_t st) {
  B2L_CHECK(nl >= 1 && nl <= GRAM_MAXL && nr >= 1 && nr <= GRAM_MAXR, -B2L_EINVAL,
            "gram: 1..4 left and 1..8 right blocks");
  B2L_CHECK(nrows >= 0, -B2L_EINVAL, "gram: negative row count");
  GramArgs A{};
  GramMap M{};
  A.nrows = nrows;
  A.nu = 0;
  A.nl = nl;
  A.nr = nr;
  auto uid = [&](const HostBlock& b) -> int {
    for (int u = 0; u < A.nu; ++u)
      if (A.up[u] == b.p && A.uld[u] == b.ld) return u;
    if (A.nu >= GRAM_MAXU) return -1;
    A.up[A.nu] = b.p;
    A.uld[A.nu] = b.ld;
    A.usld[A.nu] = (b.ld + 3) & ~3;
    return A.nu++;
  };
  int voff = 0;
  M.nl = nl;
  for (int l = 0; l < nl; ++l) {
    B2L_CHECK(L[l].ld >= 2 && (L[l].ld & 1) == 0 && L[l].cols <= L[l].ld && L[l].cols >= 0,
              -B2L_EINVAL, "gram: left block needs even ld >= cols");
    B2L_CHECK((reinterpret_cast<uintptr_t>(L[l].p) & 15) == 0, -B2L_EINVAL,
              "gram: blocks must be 16-B aligned");
    const int u = uid(L[l]);
    B2L_CHECK(u >= 0, -B2L_EINVAL, "gram: too many distinct blocks");
    A.lu[l] = u;
    A.lvoff[l] = voff;
    M.lvoff[l] = voff;
    M.lcols[l] = L[l].cols;
    M.a += L[l].cols;
    voff += A.usld[u];
  }
  A.a_pad = voff;
  voff = 0;
  M.nr = nr;
  for (int r = 0; r < nr; ++r) {
    B2L_CHECK(R[r].ld >= 2 && (R[r].ld & 1) == 0 && R[r].cols <= R[r].ld && R[r].cols >= 0,
              -B2L_EINVAL, "gram: right block needs even ld >= cols");
    B2L_CHECK((reinterpret_cast<uintptr_t>(R[r].p) & 15) == 0, -B2L_EINVAL,
              "gram: blocks must be 16-B aligned");
    const int u = uid(R[r]);
    B2L_CHECK(u >= 0, -B2L_EINVAL, "gram: too many distinct blocks");
    A.ru[r] = u;
    A.rvoff[r] = voff;
    M.rvoff[r] = voff;
    M.rcols[r] = R[r].cols;
    M.b += R[r].cols;
    voff += A.usld[u];
  }
  A.b_pad = voff;
  M.a_pad = A.a_pad;
  M.b_pad = A.b_pad;
  A.rw_mask = rw_mask;
  A.d = rw_mask ? d : nullptr;
  B2L_CHECK(!rw_mask || d != nullptr, -B2L_EINVAL, "gram: weight mask without weights");
  if (M.a * M.b == 0) return 0;

  int width = 0;
  for (int u = 0; u < A.nu; ++u) width += A.usld[u];
  A.rc = width <= 96 ? 64 : (width <= 192 ? 32 : 16);
  int off = 0;
  for (int u = 0; u < A.nu; ++u) {
    A.ubase[u] = off;
    off += A.rc * A.usld[u];
  }
  A.dbase = off;
  off += A.rc;
  A.stage_doubles = (off + 15) & ~15;
  A.tiles_n = A.b_pad / 4;
  A.ntiles = (A.a_pad / 4) * A.tiles_n;
  A.tset = A.ntiles < GRAM_THREADS ? A.ntiles : GRAM_THREADS;
  A.G = GRAM_THREADS / A.tset;
  if (A.G > A.rc) A.G = A.rc;
  const int nsets = (A.ntiles + A.tset - 1) / A.tset;

  const int nchunks = nrows > 0 ? (nrows + A.rc - 1) / A.rc : 0;
  int gx = 2 * sm_count();
  if (gx > nchunks) gx = nchunks;
  if (gx < 1) gx = 1;
  size_t smem = (size_t)2 * A.stage_doubles * sizeof(double);
  const size_t red_need = (size_t)(A.G > 1 ? A.G - 1 : 0) * A.tset * 16 * sizeof(double);
  if (red_need > smem) smem = red_need;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "gram: blocks too wide for shared memory");
  int werr = 0;
  double* part = static_cast<double*>(
      workspace((size_t)gx * A.a_pad * A.b_pad * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  if (nrows == 0) {
    B2L_CUDA(cudaMemsetAsync(part, 0, (size_t)A.a_pad * A.b_pad * sizeof(double), st));
  } else {
    B2L_CUDA(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    gram_kernel<<<dim3(gx, nsets), GRAM_THREADS, smem, st>>>(A);
    B2L_CUDA(cudaGetLastError());
  }
  const int tot = M.a * M.b;
  gram_reduce_kernel<<<(tot + 255) / 256, 256, 0, st>>>(part, nrows == 0 ? 1 : gx, M, out);
  B2L_CUDA(cudaGetLastError());
  return 0;
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
    for (int r = blockIdx.x * A.rp + rr; r < A.nrows; r += gridDim.x * A.rp) {
      const double xv = A.x[(size_t)r * A.ldx + j];
      const double av = A.ax[(size_t)r * A.ldx + j];
      const double bx = A.d ? __dmul_rn(A.d[r], xv) : xv;
      const double wf = __dsub_rn(av, __dmul_rn(bx, lam));
      s_w = fma(wf, wf, s_w);
      if (A.want_ax) s_a = fma(av, av, s_a);
      if (p >= 0) {
        double tv = wf;
        if (A.tmode == 1) tv = __dmul_rn(A.tinv, wf);
        else if (A.tmode == 2) tv = __dmul_rn(A.tvec[r], wf);
        A.w[(size_t)r * A.ldw + p] = tv;
        if (padw) A.w[(size_t)r * A.ldw + A.kw] = 0.0;
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

__global__ void sum_parts_kernel(const double* partial, int nparts, int len,
                                 double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += partial[(size_t)c * len + e];
  out[e] = s;
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
  B2L_CUDA(cudaGetLastError());
  sum_parts_kernel<<<(2 * m + 127) / 128, 128, 0, st>>>(part, blocks, 2 * m, sums_out);
  B2L_CUDA(cudaGetLastError());
  return 0;
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
      const double* xr = A.x + (size_t)r * A.ldx;
      for (int i = 0; i < A.m; ++i) xs = fma(xr[i], scx[i * A.m + c], xs);
      if (A.x_plus_p) xs = __dadd_rn(xs, pn);
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

int update(int nrows, int m, const double* x, const double* ax, int ldx,
           const double* cx, const double* w, const double* aw, int ldw, int kw,
           const double* cw, const double* p, const double* ap, int ldp,
           const int* pcols, int kp, const double* cp, double* xo, double* axo,
           int ldo, double* po, double* apo, int ldpo, int x_plus_p,
           cudaStream_t st) {
  B2L_CHECK(m >= 1 && m <= 256, -B2L_EINVAL, "update: 1 <= m <= 256");
  B2L_CHECK(ldx >= m && ldo >= m, -B2L_EINVAL, "update: ld < m");
  B2L_CHECK(kw >= 0 && kp >= 0, -B2L_EINVAL, "update: negative block width");
  B2L_CHECK(!ax || axo, -B2L_EINVAL, "update: A-side input without output");
  B2L_CHECK(x != xo && (!ax || ax != axo), -B2L_EINVAL, "update: in-place not supported");
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
  const size_t smem = (size_t)(m * m + kw * m + kp * m) * sizeof(double) + kp * sizeof(int) + 16;
  B2L_CHECK(smem <= 227 * 1024, -B2L_EINVAL, "update: coefficients too large");
  int blocks = (nrows + A.rp - 1) / A.rp;
  const int cap = 8 * sm_count();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  B2L_CUDA(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  update_kernel<<<blocks, 256, smem, st>>>(A);
  B2L_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace b2l
