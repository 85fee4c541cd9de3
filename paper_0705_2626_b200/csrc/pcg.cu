// Column-batched preconditioned conjugate gradients for the inner-PCG
// preconditioner (reference operators.py:341-427: pcg_solve,
// InnerPCGPreconditioner).  The reference runs pcg_solve once per column; here
// all k columns of a block advance together, each with its own scalars, so
// A p is one fused stencil pass over the block (K1+K5b with m = 0 also gives
// the curvatures p_j^T A p_j) and the vector updates are three streaming
// kernels.  Every scalar stays on the device (no host round trip per step):
//   update    : alpha_j = rz_j / pap_j ; x += alpha p ; r -= alpha Ap ;
//               sums: r^T z (z = M r) and r^T r        (operators.py:379-386)
//   direction : stop_j (rtol, rz_next == 0) ; p = z + (rz_next / rz) p
//                                                       (operators.py:387-392)
// Elementwise arithmetic follows numpy's rounding (products rounded before
// the add, no FMA contraction); the dot products are deterministic fixed-order
// reductions.  M: 0 identity, 1 scalar, 2 row vector (Jacobi), 3 z supplied
// by the caller in a block (generic preconditioner callback).
#include "common.cuh"

namespace b2l {
namespace {

struct PcgArgs {
  int nrows, k, rp;
  int ld;
  const double* b;
  int ldb;
  double* x;
  double* r;
  double* p;
  const double* ap;
  const double* z;        // tmode 3
  int tmode;
  double tinv;
  const double* tvec;
  const double* pap;      // pap_j = pap[j * pap_stride]
  int pap_stride;
  const double* rz;       // current rz (k)
  const double* bb;       // ||b_j||^2 (k)
  const int* done;        // (k)
  double* rz_next;        // direction: rz for the next step (block 0 writes)
  int* done_next;         // direction: stop flags for the next step (block 0)
  const double* sums;     // direction: [r^T z | r^T r] of this step
  double rtol;
  int* err;               // set on nonpositive / non-finite curvature
  double* partial;        // [grid][2k]
};

__device__ __forceinline__ double apply_t(const PcgArgs& A, size_t r, double v) {
  if (A.tmode == 1) return __dmul_rn(A.tinv, v);
  if (A.tmode == 2) return __dmul_rn(A.tvec[r], v);
  return v;
}

__device__ __forceinline__ void block_sums(const PcgArgs& A, double* sm, int rr, int j, bool on,
                                           double s0, double s1) {
  if (on) {
    sm[rr * A.k + j] = s0;
    sm[(A.rp + rr) * A.k + j] = s1;
  }
  __syncthreads();
  if (threadIdx.x < A.k) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < A.rp; ++q) {
      a += sm[q * A.k + threadIdx.x];
      b += sm[(A.rp + q) * A.k + threadIdx.x];
    }
    A.partial[(size_t)blockIdx.x * 2 * A.k + threadIdx.x] = a;
    A.partial[(size_t)blockIdx.x * 2 * A.k + A.k + threadIdx.x] = b;
  }
}

// x = 0, r = b, p = z = M b; sums [b^T b | r^T z]
__global__ void __launch_bounds__(256) pcg_init_kernel(PcgArgs A) {
  extern __shared__ double psm[];
  const int rr = threadIdx.x / A.k, j = threadIdx.x - rr * A.k;
  const bool on = rr < A.rp;
  double s0 = 0.0, s1 = 0.0;
  if (on)
    for (int row = blockIdx.x * A.rp + rr; row < A.nrows; row += gridDim.x * A.rp) {
      const size_t o = (size_t)row * A.ld + j;
      const double bv = A.b[(size_t)row * A.ldb + j];
      const double zv = A.tmode == 3 ? A.z[o] : apply_t(A, row, bv);
      A.x[o] = 0.0;
      A.r[o] = bv;
      A.p[o] = zv;
      s0 = fma(bv, bv, s0);
      s1 = fma(bv, zv, s1);
    }
  block_sums(A, psm, rr, j, on, s0, s1);
}

// alpha = rz / pap ; x += alpha p ; r -= alpha Ap ; sums [r^T M r | r^T r]
__global__ void __launch_bounds__(256) pcg_update_kernel(PcgArgs A) {
  extern __shared__ double psm[];
  const int rr = threadIdx.x / A.k, j = threadIdx.x - rr * A.k;
  const bool on = rr < A.rp;
  double s0 = 0.0, s1 = 0.0;
  if (on) {
    const bool live = !A.done[j] && A.bb[j] != 0.0;
    const double pap = A.pap[(size_t)j * A.pap_stride];
    if (live && (!(pap > 0.0) || !isfinite(pap)) && blockIdx.x == 0 && rr == 0)
      atomicOr(A.err, 1);
    if (live) {
      const double alpha = A.rz[j] / pap;
      for (int row = blockIdx.x * A.rp + rr; row < A.nrows; row += gridDim.x * A.rp) {
        const size_t o = (size_t)row * A.ld + j;
        A.x[o] = __dadd_rn(A.x[o], __dmul_rn(alpha, A.p[o]));
        const double rv = __dsub_rn(A.r[o], __dmul_rn(alpha, A.ap[o]));
        A.r[o] = rv;
        if (A.tmode != 3) s0 = fma(rv, apply_t(A, row, rv), s0);
        s1 = fma(rv, rv, s1);
      }
    }
  }
  block_sums(A, psm, rr, j, on, s0, s1);
}

// tmode 3: sums [r^T z | r^T r] once the caller has formed z = M r
__global__ void __launch_bounds__(256) pcg_dot_kernel(PcgArgs A) {
  extern __shared__ double psm[];
  const int rr = threadIdx.x / A.k, j = threadIdx.x - rr * A.k;
  const bool on = rr < A.rp;
  double s0 = 0.0, s1 = 0.0;
  if (on && !A.done[j] && A.bb[j] != 0.0)
    for (int row = blockIdx.x * A.rp + rr; row < A.nrows; row += gridDim.x * A.rp) {
      const size_t o = (size_t)row * A.ld + j;
      const double rv = A.r[o];
      s0 = fma(rv, A.z[o], s0);
      s1 = fma(rv, rv, s1);
    }
  block_sums(A, psm, rr, j, on, s0, s1);
}

// stop test, then p = M r + (rz_next / rz) p on the live columns
__global__ void __launch_bounds__(256) pcg_direction_kernel(PcgArgs A) {
  const int rr = threadIdx.x / A.k, j = threadIdx.x - rr * A.k;
  if (rr >= A.rp) return;
  const double rzn = A.sums[j], rnorm2 = A.sums[A.k + j];
  bool stop = A.done[j] || A.bb[j] == 0.0;
  if (!stop && A.rtol > 0.0 && sqrt(rnorm2) <= A.rtol * sqrt(A.bb[j])) stop = true;
  if (!stop && rzn == 0.0) stop = true;
  if (blockIdx.x == 0 && rr == 0) {
    A.done_next[j] = stop ? 1 : 0;
    A.rz_next[j] = stop ? A.rz[j] : rzn;
  }
  if (stop) return;
  const double beta = rzn / A.rz[j];
  for (int row = blockIdx.x * A.rp + rr; row < A.nrows; row += gridDim.x * A.rp) {
    const size_t o = (size_t)row * A.ld + j;
    const double zv = A.tmode == 3 ? A.z[o] : apply_t(A, row, A.r[o]);
    A.p[o] = __dadd_rn(zv, __dmul_rn(beta, A.p[o]));
  }
}

int pcg_launch(int phase, PcgArgs& A, cudaStream_t st, double* sums_out) {
  A.rp = 256 / A.k;
  int blocks = (A.nrows + A.rp - 1) / A.rp;
  const int cap = 4 * sm_count();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const size_t smem = (size_t)2 * A.rp * A.k * sizeof(double);
  if (phase == 2) {
    pcg_direction_kernel<<<blocks, 256, 0, st>>>(A);
    count_launch();
    B2L_CUDA(cudaGetLastError());
    return 0;
  }
  int werr = 0;
  double* part =
      static_cast<double*>(workspace((size_t)blocks * 2 * A.k * sizeof(double), &werr));
  if (werr) return werr;
  A.partial = part;
  if (phase == 0) { pcg_init_kernel<<<blocks, 256, smem, st>>>(A); count_launch(); }
  else if (phase == 1) { pcg_update_kernel<<<blocks, 256, smem, st>>>(A); count_launch(); }
  else { pcg_dot_kernel<<<blocks, 256, smem, st>>>(A); count_launch(); }
  B2L_CUDA(cudaGetLastError());
  return sum_parts(part, blocks, 2 * A.k, sums_out, st);
}

}  // namespace
}  // namespace b2l

using namespace b2l;

#define PCG_COMMON_CHECKS()                                                              \
  do {                                                                                   \
    if (k < 1 || k > 256 || ld < k || nrows < 1)                                        \
      return fail(-B2L_EINVAL, "pcg: need 1 <= k <= 256, ld >= k, nrows >= 1");          \
    if (tmode < 0 || tmode > 3 || (tmode == 2 && !tvec) || (tmode == 3 && !z))          \
      return fail(-B2L_EINVAL, "pcg: bad preconditioner mode");                          \
  } while (0)

extern "C" int b2l_pcg_init(int nrows, int k, const double* b, int ldb, double* x, double* r,
                            double* p, int ld, const double* z, int tmode, double tinv,
                            const double* tvec, double* sums_out, void* stream) {
  PCG_COMMON_CHECKS();
  if (!b || ldb < k) return fail(-B2L_EINVAL, "pcg_init: bad right-hand side");
  PcgArgs A{};
  A.nrows = nrows;
  A.k = k;
  A.ld = ld;
  A.b = b;
  A.ldb = ldb;
  A.x = x;
  A.r = r;
  A.p = p;
  A.z = z;
  A.tmode = tmode;
  A.tinv = tinv;
  A.tvec = tvec;
  return pcg_launch(0, A, (cudaStream_t)stream, sums_out);
}

extern "C" int b2l_pcg_update(int nrows, int k, double* x, double* r, const double* p,
                              const double* ap, int ld, const double* pap, int pap_stride,
                              const double* rz, const double* bb, const int* done, int tmode,
                              double tinv, const double* tvec, double* sums_out, int* err,
                              void* stream) {
  const double* z = tmode == 3 ? r : nullptr;   // z is not read by the update
  PCG_COMMON_CHECKS();
  PcgArgs A{};
  A.nrows = nrows;
  A.k = k;
  A.ld = ld;
  A.x = x;
  A.r = r;
  A.p = const_cast<double*>(p);
  A.ap = ap;
  A.tmode = tmode;
  A.tinv = tinv;
  A.tvec = tvec;
  A.pap = pap;
  A.pap_stride = pap_stride;
  A.rz = rz;
  A.bb = bb;
  A.done = done;
  A.err = err;
  return pcg_launch(1, A, (cudaStream_t)stream, sums_out);
}

extern "C" int b2l_pcg_dot(int nrows, int k, const double* r, const double* z, int ld,
                           const double* bb, const int* done, double* sums_out, void* stream) {
  const int tmode = 3;
  const double* tvec = nullptr;
  (void)tvec;
  PCG_COMMON_CHECKS();
  PcgArgs A{};
  A.nrows = nrows;
  A.k = k;
  A.ld = ld;
  A.r = const_cast<double*>(r);
  A.z = z;
  A.tmode = 3;
  A.bb = bb;
  A.done = done;
  return pcg_launch(3, A, (cudaStream_t)stream, sums_out);
}

extern "C" int b2l_pcg_direction(int nrows, int k, const double* r, double* p, int ld,
                                 const double* z, int tmode, double tinv, const double* tvec,
                                 const double* rz, const double* sums, const double* bb,
                                 double rtol, const int* done, int* done_next, double* rz_next,
                                 void* stream) {
  PCG_COMMON_CHECKS();
  PcgArgs A{};
  A.nrows = nrows;
  A.k = k;
  A.ld = ld;
  A.r = const_cast<double*>(r);
  A.p = p;
  A.z = z;
  A.tmode = tmode;
  A.tinv = tinv;
  A.tvec = tvec;
  A.rz = rz;
  A.sums = sums;
  A.bb = bb;
  A.rtol = rtol;
  A.done = done;
  A.done_next = done_next;
  A.rz_next = rz_next;
  return pcg_launch(2, A, (cudaStream_t)stream, nullptr);
}
