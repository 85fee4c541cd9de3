// Host side of one LOBPCG iteration: the Rayleigh-Ritz step on the projected
// pencil, with the reference's basis-repair ladders (reference lobpcg.py:475-519
// and the small dense algebra of multivec.py:89-211).
//
// Input is the Gram data the device passes produced (F1 / K5: G1; K1+K5b: G2);
// output is the next Ritz values and the update coefficients with the
// Cholesky-QR factors of W and P folded in (so the tall blocks are never
// rewritten).  Everything here is O(m^3) on <= 3m x 3m matrices; it sits on
// the critical path between two device passes, which is why it is native.
//
// The small dense algebra (Cholesky in the reference's row-by-row form,
// triangular solves, the symmetric eigensolver) is native by default.  With
// B2L_RR_LAPACK=1 it runs through LAPACK routines the caller registered with
// b2l_set_lapack (dpotrf / dtrtrs / dtrtri / dsyevr, Fortran-style C
// signatures of scipy.linalg.cython_lapack: the routines the reference's
// scipy calls run).  The small matrix products are plain loops.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

// phase timers for the standalone host harness (tools/rr_harness.cu); empty
// in the library
#ifdef B2L_RR_PROF
#define RR_MARK(k) rr_mark(k)
#else
#define RR_MARK(k) ((void)0)
#endif

namespace b2l {
namespace {

using potrf_t = void(char*, int*, double*, int*, int*);
using trtrs_t = void(char*, char*, char*, int*, int*, double*, int*, double*, int*, int*);
using trtri_t = void(char*, char*, int*, double*, int*, int*);
using syevr_t = void(char*, char*, char*, int*, double*, int*, double*, double*, int*, int*,
                     double*, int*, double*, double*, int*, int*, double*, int*, int*, int*,
                     int*);

potrf_t* g_potrf = nullptr;
trtrs_t* g_trtrs = nullptr;
trtri_t* g_trtri = nullptr;
syevr_t* g_syevr = nullptr;
// dsyevr's own stages (scipy.linalg.cython_lapack): for all pairs dsyevr runs
// dsytrd, dstemr (MRRR) and dormtr; calling them directly lets the MRRR
// vectors be formed for the wanted pairs only
using sytrd_t = void(char*, int*, double*, int*, double*, double*, double*, double*, int*,
                     int*);
using stemr_t = void(char*, char*, int*, double*, double*, double*, double*, int*, int*, int*,
                     double*, double*, int*, int*, int*, int*, double*, int*, int*, int*, int*);
using ormtr_t = void(char*, char*, char*, int*, int*, double*, int*, double*, double*, int*,
                     double*, int*, int*);
sytrd_t* g_sytrd = nullptr;
stemr_t* g_stemr = nullptr;
ormtr_t* g_ormtr = nullptr;

// column-major dense matrix
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0.0) {}
  double& operator()(int i, int j) { return a[(size_t)i + (size_t)j * r]; }
  double operator()(int i, int j) const { return a[(size_t)i + (size_t)j * r]; }
  double* p() { return a.data(); }
};

struct NotSPD {
  int pivot;
};
struct LapackError {
  const char* what;
  int info;
};

// optional BLAS dgemm (Fortran signature of scipy.linalg.cython_blas) for
// the larger pencils (m = 64: 64 x 64 blocks)
using dgemm_t = void(char*, char*, int*, int*, int*, double*, const double*, int*, const double*,
                     int*, double*, double*, int*);
dgemm_t* g_dgemm = nullptr;

Mat matmul(const Mat& x, const Mat& y) {
  if (g_dgemm && x.r * x.c * y.c >= 32 * 32 * 32) {
    Mat z(x.r, y.c);
    char n = 'N';
    int mm = x.r, nn = y.c, kk = x.c, lda = x.r, ldb = y.r, ldc = z.r;
    double one = 1.0, zero = 0.0;
    g_dgemm(&n, &n, &mm, &nn, &kk, &one, x.a.data(), &lda, y.a.data(), &ldb, &zero, z.p(), &ldc);
    return z;
  }
  // column-major j-k-i order: the inner loop runs down contiguous columns of
  // z and x (vectorisable, cache-friendly at the 192 x 192 sizes of m = 64)
  Mat z(x.r, y.c);
  for (int j = 0; j < y.c; ++j) {
    double* zc = z.p() + (size_t)j * z.r;
    for (int k = 0; k < x.c; ++k) {
      const double ykj = y(k, j);
      const double* xc = x.a.data() + (size_t)k * x.r;
      for (int i = 0; i < x.r; ++i) zc[i] += xc[i] * ykj;
    }
  }
  return z;
}

Mat transpose(const Mat& x) {
  Mat z(x.c, x.r);
  for (int j = 0; j < x.c; ++j)
    for (int i = 0; i < x.r; ++i) z(j, i) = x(i, j);
  return z;
}

// The small dense algebra runs natively by default (n <= 3m <= 48: library
// call overheads dominate LAPACK here, and dsyevr on 30 x 30 costs ~2x the
// native tridiagonal QL).  B2L_RR_LAPACK=1 routes it through the registered
// LAPACK routines instead (same factorisations, LAPACK rounding).
// B2L_RR_LAPACK=1: always LAPACK; =0: never; unset: LAPACK for pencils
// larger than 64 (m > 21; the blocked, vectorised routines win there: 192 x
// 192 at m = 64 ~2x faster than the native scalar code), native below.
// dimension of the pencil being solved, set by rr_begin; per host thread so
// two threads' Rayleigh-Ritz steps never see each other's LAPACK choice
thread_local int g_rr_dim = 0;
// The pencil eigensolve.  Default (pencils up to 64 x 64): the native
// substitution congruence + tridiagonal QR with the computed eigenvectors
// of numerically degenerate clusters aligned to the current Ritz vectors
// (align_clusters below).  b2l_set_rr_reference(1) / B2L_RR_EIG=ref: the
// reference's own sequence (two dtrtrs, dsyevr on all pairs -- scipy's eigh
// driver), ~50 us slower per C2 iteration.  Inside (near-)degenerate clusters
// the basis an eigensolver returns steers which Ritz column locks first; on
// C1 over 128 perturbed problems (tools/c1_band32.py 64): the reference
// converges without a basis fallback 117 times, the dsyevr sequence here 97,
// the plain QR 39, the aligned QR 128.  Above 64 x 64 (m >= 22) the LAPACK
// sequence runs either way.
thread_local int g_rr_ref = -1;   // -1: not set by the caller (native aligned QR)
bool eig_lapack() {
  static const int forced = [] {
    const char* v = getenv("B2L_RR_EIG");
    return v ? (v[0] == 'q' ? 0 : (v[0] == 'r' ? 1 : -1)) : -1;
  }();
  if (g_syevr == nullptr || g_trtrs == nullptr) return false;
  if (forced >= 0) return forced == 1;
  return g_rr_ref == 1;
}

bool use_lapack() {
  static const int mode = [] {
    const char* v = getenv("B2L_RR_LAPACK");
    return v ? (v[0] == '1' ? 1 : 0) : -1;
  }();
  if (g_potrf == nullptr) return false;
  if (mode >= 0) return mode == 1;
  return g_rr_dim > 64;
}

// Symmetric eigensolver for the `want` smallest pairs of an n x n matrix
// (the small dense eigenproblem of the Rayleigh-Ritz step; the reference
// calls LAPACK dsyevr through scipy.linalg.eigh, multivec.py:161-211).
// Written from the textbook statements of the two classic stages (Golub &
// Van Loan, Matrix Computations, 4th ed.: Householder vectors Alg. 5.1.1,
// Householder tridiagonalisation Alg. 8.3.1, the symmetric tridiagonal QR
// step with implicit Wilkinson shift Alg. 8.3.2 and its deflation loop
// Alg. 8.3.3):
//   1. T = Q^T A Q by Householder reflections from the left/right of
//      columns 0 .. n-3 (A is read in full; symmetric input);
//   2. implicit shifted QR sweeps (bulge chasing from the top) on (d, e)
//      WITHOUT touching vectors -- each Givens rotation is logged;
//   3. the wanted eigenvectors Q G_1 ... G_K e_k formed by replaying the log
//      backwards on the wanted unit vectors only (O(K want) instead of the
//      O(K n) of rotating a full basis; 30 x 30: ~3x fewer flops), then the
//      reflectors applied to those `want` columns (Q is never formed).
// a: n x n column-major (destroyed); vals (want) ascending; vecs (n x want,
// column-major).  Returns 1 if the QR sweeps do not converge.
int symeig_tridiag_qr(int n, double* a, int want, double* vals, double* vecs) {
  auto A = [&](int i, int j) -> double& { return a[i + (size_t)j * n]; };
  thread_local std::vector<double> dbuf, ebuf, vbuf, pbuf, betas, rs, rc;
  thread_local std::vector<int> ri, perm;
  dbuf.assign(n, 0.0);
  ebuf.assign(n > 1 ? n - 1 : 1, 0.0);
  vbuf.assign((size_t)n * n, 0.0);   // Householder vectors, column k holds v_k
  pbuf.assign(n, 0.0);
  betas.assign(n, 0.0);
  double* d = dbuf.data();
  double* e = ebuf.data();
  double* V = vbuf.data();
  double* pw = pbuf.data();
  // ---- 1. tridiagonalisation
  for (int k = 0; k + 2 < n; ++k) {
    const int m0 = k + 1, len = n - m0;
    double* v = V + (size_t)k * n;   // entries m0 .. n-1 used
    double sigma = 0.0;
    for (int i = 1; i < len; ++i) sigma += A(m0 + i, k) * A(m0 + i, k);
    const double x0 = A(m0, k);
    double beta = 0.0, alpha = x0;   // alpha: the new sub-diagonal entry
    v[m0] = 1.0;
    for (int i = 1; i < len; ++i) v[m0 + i] = A(m0 + i, k);
    if (sigma != 0.0) {
      const double mu = std::sqrt(x0 * x0 + sigma);
      const double v0 = x0 <= 0.0 ? x0 - mu : -sigma / (x0 + mu);
      beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
      for (int i = 1; i < len; ++i) v[m0 + i] /= v0;
      alpha = mu;
    }
    betas[k] = beta;
    d[k] = A(k, k);
    e[k] = alpha;
    if (beta == 0.0) continue;
    // p = beta A22 v ; w = p - (beta p^T v / 2) v ; A22 -= v w^T + w v^T,
    // on the lower triangle of A22 only (symmetric matrix-vector product and
    // rank-2 update by columns)
    for (int i = m0; i < n; ++i) pw[i] = 0.0;
    for (int j = m0; j < n; ++j) {
      const double vj = v[j];
      double t2 = 0.0;
      pw[j] += A(j, j) * vj;
      const double* aj = a + (size_t)j * n;
      for (int i = j + 1; i < n; ++i) {
        pw[i] += aj[i] * vj;
        t2 += aj[i] * v[i];
      }
      pw[j] += t2;
    }
    double pv = 0.0;
    for (int i = m0; i < n; ++i) {
      pw[i] *= beta;
      pv += pw[i] * v[i];
    }
    const double half = 0.5 * beta * pv;
    for (int i = m0; i < n; ++i) pw[i] -= half * v[i];
    for (int j = m0; j < n; ++j) {
      const double vj = v[j], wj = pw[j];
      double* aj = a + (size_t)j * n;
      for (int i = j; i < n; ++i) aj[i] -= v[i] * wj + pw[i] * vj;
    }
  }
  if (n >= 2) {
    d[n - 2] = A(n - 2, n - 2);
    e[n - 2] = A(n - 1, n - 2);
  }
  d[n - 1] = A(n - 1, n - 1);
  RR_MARK(7);
  RR_MARK(8);
  // ---- 2. implicit Wilkinson-shift QR on (d, e), rotations logged
  ri.clear();
  rs.clear();
  rc.clear();
  const double eps = 2.220446049250313e-16;
  int hi = n - 1, sweeps = 0;
  while (hi > 0) {
    if (std::fabs(e[hi - 1]) <= eps * (std::fabs(d[hi - 1]) + std::fabs(d[hi]))) {
      e[hi - 1] = 0.0;
      --hi;
      continue;
    }
    int lo = hi - 1;
    while (lo > 0 && std::fabs(e[lo - 1]) > eps * (std::fabs(d[lo - 1]) + std::fabs(d[lo]))) --lo;
    if (lo > 0) e[lo - 1] = 0.0;
    if (++sweeps > 30 * n) return 1;
    // Wilkinson shift: the eigenvalue of the trailing 2 x 2 nearer d[hi]
    const double t = e[hi - 1];
    const double delta = 0.5 * (d[hi - 1] - d[hi]);
    const double rad = std::hypot(delta, t);
    const double mu = d[hi] - t * t / (delta + (delta >= 0.0 ? rad : -rad));
    double x = d[lo] - mu, z = e[lo];
    for (int k = lo; k < hi; ++k) {
      // Givens: [c s; -s c]^T [x; z] = [r; 0]
      // |(x, z)| without hypot's overflow guard: x and z are bounded by the
      // matrix norm, far from the fp64 range limits here
      const double r = std::sqrt(x * x + z * z);
      const double rinv = r == 0.0 ? 0.0 : 1.0 / r;
      const double c = r == 0.0 ? 1.0 : x * rinv;
      const double s = -z * rinv;
      if (k > lo) e[k - 1] = r;
      const double dk = d[k], dk1 = d[k + 1], ek = e[k];
      d[k] = c * c * dk - 2.0 * c * s * ek + s * s * dk1;
      d[k + 1] = s * s * dk + 2.0 * c * s * ek + c * c * dk1;
      e[k] = c * s * (dk - dk1) + (c * c - s * s) * ek;
      if (k + 1 < hi) {   // the bulge at (k, k + 2)
        x = e[k];
        z = -s * e[k + 1];
        e[k + 1] = c * e[k + 1];
      }
      ri.push_back(k);
      rc.push_back(c);
      rs.push_back(s);
    }
  }
  RR_MARK(9);
  // ---- ascending order: selection sort on (value, column) pairs
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int i = 0; i < n - 1 && i < want; ++i) {
    int k = i;
    for (int j = i + 1; j < n; ++j)
      if (d[j] < d[k]) k = j;
    if (k != i) {
      std::swap(d[i], d[k]);
      std::swap(perm[i], perm[k]);
    }
  }
  // ---- 3. wanted vectors: Y = G_1 ... G_K [e_perm(0) .. e_perm(want-1)]
  // (the log replayed backwards on all wanted columns at once; Y row-major
  // n x want, so a rotation updates two contiguous rows), then the
  // reflectors applied to Y itself, V = H_0 ... H_{n-3} Y (O(n^2 want); Q is
  // never formed)
  thread_local std::vector<double> ybuf;
  ybuf.assign((size_t)n * want, 0.0);
  double* Y = ybuf.data();
  for (int w = 0; w < want; ++w) {
    vals[w] = d[w];
    Y[(size_t)perm[w] * want + w] = 1.0;
  }
  for (int t = (int)ri.size() - 1; t >= 0; --t) {
    double* y0 = Y + (size_t)ri[t] * want;
    double* y1 = y0 + want;
    const double s = rs[t], c = rc[t];
    for (int w = 0; w < want; ++w) {
      const double yi = y0[w], yj = y1[w];
      y0[w] = c * yi + s * yj;
      y1[w] = c * yj - s * yi;
    }
  }
  for (int k = n - 3; k >= 0; --k) {
    const double beta = betas[k];
    if (beta == 0.0) continue;
    const double* v = V + (size_t)k * n;
    double* wv = pw;   // beta v^T Y (want values)
    for (int w = 0; w < want; ++w) wv[w] = 0.0;
    for (int i = k + 1; i < n; ++i) {
      const double vi = v[i];
      const double* yi = Y + (size_t)i * want;
      for (int w = 0; w < want; ++w) wv[w] += vi * yi[w];
    }
    for (int w = 0; w < want; ++w) wv[w] *= beta;
    for (int i = k + 1; i < n; ++i) {
      const double vi = v[i];
      double* yi = Y + (size_t)i * want;
      for (int w = 0; w < want; ++w) yi[w] -= vi * wv[w];
    }
  }
  for (int w = 0; w < want; ++w) {
    double* vcol = vecs + (size_t)w * n;
    for (int r = 0; r < n; ++r) vcol[r] = Y[(size_t)r * want + w];
  }
  return 0;
}

// Upper R with g = R^T R from g's upper triangle, row by row as the
// reference's multivec.cholesky (multivec.py:89-122): pivot d_j = g_jj -
// sum_k r_kj^2 must be finite and > floor * g_jj, else NotSPD(j).
Mat cholesky_native(const Mat& g, double floor_) {
  const int k = g.r;
  Mat r(k, k);
  for (int j = 0; j < k; ++j) {
    double d = g(j, j);
    for (int t = 0; t < j; ++t) d -= r(t, j) * r(t, j);
    if (!(d > floor_ * g(j, j)) || !std::isfinite(d)) throw NotSPD{j};
    const double rjj = std::sqrt(d);
    r(j, j) = rjj;
    for (int c = j + 1; c < k; ++c) {
      double v = g(j, c);
      for (int t = 0; t < j; ++t) v -= r(t, j) * r(t, c);
      r(j, c) = v / rjj;
    }
  }
  return r;
}

// R^{-T} b (trans: forward substitution with R^T) or R^{-1} b (back substitution)
Mat trsolve_native(const Mat& r, const Mat& b, bool trans) {
  const int n = r.r;
  Mat x = b;
  for (int c = 0; c < b.c; ++c) {
    if (trans) {
      for (int i = 0; i < n; ++i) {
        double v = x(i, c);
        for (int t = 0; t < i; ++t) v -= r(t, i) * x(t, c);
        x(i, c) = v / r(i, i);
      }
    } else {
      for (int i = n - 1; i >= 0; --i) {
        double v = x(i, c);
        for (int t = i + 1; t < n; ++t) v -= r(i, t) * x(t, c);
        x(i, c) = v / r(i, i);
      }
    }
  }
  return x;
}

// Upper R with g = R^T R from g's upper triangle; a pivot <= floor * g_jj (or
// non-finite) throws NotSPD(j)  (small.cholesky; multivec.py:89-122).
Mat cholesky(const Mat& g, double floor_) {
  if (!use_lapack()) return cholesky_native(g, floor_);
  const int k = g.r;
  Mat r = g;
  if (k == 0) return r;
  char uplo = 'U';
  int n = k, lda = k, info = 0;
  g_potrf(&uplo, &n, r.p(), &lda, &info);
  if (info < 0) throw LapackError{"dpotrf", info};
  for (int j = 0; j < k; ++j)
    for (int i = j + 1; i < k; ++i) r(i, j) = 0.0;   // clean
  const int ok = info == 0 ? k : info - 1;
  for (int j = 0; j < ok; ++j) {
    const double piv = r(j, j) * r(j, j);
    if (!(piv > floor_ * g(j, j)) || !std::isfinite(piv)) throw NotSPD{j};
  }
  if (info > 0) throw NotSPD{info - 1};
  return r;
}

// R^{-T} b (trans) or R^{-1} b for upper R
Mat trsolve(const Mat& r, const Mat& b, bool trans, bool force_lapack = false) {
  if (!use_lapack() && !(force_lapack && g_trtrs)) return trsolve_native(r, b, trans);
  Mat x = b;
  if (r.r == 0 || b.c == 0) return x;
  char uplo = 'U', tr = trans ? 'T' : 'N', diag = 'N';
  int n = r.r, nrhs = b.c, lda = r.r, ldb = b.r, info = 0;
  Mat rc = r;
  g_trtrs(&uplo, &tr, &diag, &n, &nrhs, rc.p(), &lda, x.p(), &ldb, &info);
  if (info != 0) throw LapackError{"dtrtrs", info};
  return x;
}

Mat upper_inverse(const Mat& r) {
  if (!use_lapack()) {
    Mat eye(r.r, r.r);
    for (int i = 0; i < r.r; ++i) eye(i, i) = 1.0;
    return trsolve_native(r, eye, false);
  }
  Mat inv = r;
  if (r.r == 0) return inv;
  char uplo = 'U', diag = 'N';
  int n = r.r, lda = r.r, info = 0;
  g_trtri(&uplo, &diag, &n, inv.p(), &lda, &info);
  if (info != 0) throw LapackError{"dtrtri", info};
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i) inv(i, j) = 0.0;
  return inv;
}

// Cholesky-QR factor of a block from its raw Gram (small.scaled_cholesky,
// b_orthonormalize lobpcg.py:147-179): returns inv(R D).
Mat scaled_cholesky_inv(const Mat& g, double floor_) {
  const int k = g.r;
  std::vector<double> s(k);
  for (int j = 0; j < k; ++j) {
    const double sq = g(j, j);
    if (!(sq > 0.0) || !std::isfinite(sq)) throw NotSPD{j};
    s[j] = std::sqrt(sq);
  }
  Mat gs(k, k);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) gs(i, j) = g(i, j) / s[i] / s[j];
  Mat r = cholesky(gs, floor_);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) r(i, j) *= s[j];
  return upper_inverse(r);
}

// gb = R^T R (small.gen_sym_eig, multivec.py:174-211): the factor half of the
// generalized eigensolve -- it is all the repair ladder needs (NotSPD comes
// from here), and it only involves B-Gram blocks, so b2l_fast_iteration runs
// it while the stencil pass that produces A W is still on the GPU.
struct PencilFactor {
  double floor_ = 1e-8;    // the pivot floor the factor was formed with
  Mat r;                   // upper Cholesky factor of gb
  std::vector<double> Ri;  // R^-1 row-major upper (native path)
  int d = 0;
};

void pencil_factor(const Mat& gb, double floor_, PencilFactor& f) {
  f.d = gb.r;
  f.floor_ = floor_ > 0.0 ? floor_ : 1e-8;
  f.r = cholesky(gb, floor_);
  RR_MARK(4);   // pencil Cholesky
  f.Ri.clear();
  if (use_lapack() || eig_lapack()) return;   // no explicit inverse needed
  // B2L_RR_CONG=explicit: the congruence through R^-1 (two matrix products;
  // ~17 us faster per C2 iteration, but its error grows with cond(gb)^2: on
  // 16^3, m = 8, tol 1e-8 a run stalls at a residual of 5e-8 -- kept for A/B)
  static const bool cong_explicit = [] {
    const char* e = getenv("B2L_RR_CONG");
    return e && e[0] == 'e';
  }();
  if (!cong_explicit) return;
  const int d = f.d;
  f.Ri.assign((size_t)d * d, 0.0);
  double* Ri = f.Ri.data();
  for (int i = d - 1; i >= 0; --i) {
    const double inv = 1.0 / f.r(i, i);
    double* row = Ri + (size_t)i * d;
    row[i] = inv;
    for (int t = i + 1; t < d; ++t) {
      const double rit = f.r(i, t);
      const double* rt = Ri + (size_t)t * d;
      for (int j = t; j < d; ++j) row[j] -= rit * rt[j];
    }
    for (int j = i + 1; j < d; ++j) row[j] *= inv;
  }
}


// Cluster alignment of the native eigensolve.  Inside a cluster of wanted
// eigenvalues that the Rayleigh-Ritz procedure cannot tell apart, every
// orthonormal basis is a valid eigensolver output, and the choice steers the
// iteration: a tridiagonal QR returns an arbitrary rotation of the cluster
// each step (the Ritz columns of a degenerate group are re-mixed every
// iteration, their residuals fall together and late, locked columns are
// disturbed: C1 over 128 perturbed problems converges without a basis
// fallback 39 times), LAPACK's MRRR (the reference's scipy eigh) stays close
// to the identity on a nearly diagonal pencil (97 of 128 here, 117 in the
// reference).  align_clusters makes that property explicit: the computed
// eigenvectors of a cluster S are rotated to the basis closest to the current
// Ritz vectors -- V[:, S] <- V[:, S] Q with V[S, S] Q symmetric positive
// definite (Q = the transposed polar factor of V[S, S], Newton's iteration)
// -- 128 of 128 converge, second lock by iteration 215 in 83 (reference
// 107), quartiles 409 / 409 / 411 (reference 404 / 408 / 411).
// A cluster: consecutive wanted eigenvalues whose gaps are below
// min(pivot_floor * max|lambda|, g_align_abs): the reference's own floor for
// numerical dependence in the basis (1e-8, lobpcg.py:57), and a tenth of the
// run's residual tolerance (set per call by the solver, b2l_set_rr_align).
// The gap must stay below what the Rayleigh-Ritz step can resolve: inside a
// cluster whose eigenvalues it can tell apart, the true Ritz vectors put the
// cluster's unconverged direction into one (active) column, while an aligned
// basis can leave part of it in soft-locked columns, where no residual
// direction works on it -- with the gap at the tolerance itself one of 16
// seeds of 20^3 / m = 10 stalls for 200 iterations, with the relative floor
// alone 11 of 16 seeds of 16^3 / m = 8 / tol 1e-8 run into max_iter; at a
// tenth of the tolerance both sweeps match the reference's iteration ranges
// (DESIGN.md).  0 (the library default for direct callers):
// no alignment; B2L_RR_ALIGN=<x> scales the solver's gap for A/B runs.
thread_local double g_align_abs = 0.0;
// B2L_RR_ALIGN=<x>: the solver's gap times x (A/B runs; 0 = off)
const double g_align_mult = [] {
  const char* v = getenv("B2L_RR_ALIGN");
  return v ? atof(v) : 1.0;
}();

bool small_inverse(int s, const double* a, double* inv) {
  double w[8 * 16];
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) {
      w[i * 2 * s + j] = a[i * s + j];
      w[i * 2 * s + s + j] = i == j ? 1.0 : 0.0;
    }
  for (int c = 0; c < s; ++c) {
    int piv = c;
    for (int r = c + 1; r < s; ++r)
      if (std::fabs(w[r * 2 * s + c]) > std::fabs(w[piv * 2 * s + c])) piv = r;
    if (!(std::fabs(w[piv * 2 * s + c]) > 1e-6)) return false;
    if (piv != c)
      for (int j = 0; j < 2 * s; ++j) std::swap(w[c * 2 * s + j], w[piv * 2 * s + j]);
    const double d = 1.0 / w[c * 2 * s + c];
    for (int j = 0; j < 2 * s; ++j) w[c * 2 * s + j] *= d;
    for (int r = 0; r < s; ++r) {
      if (r == c) continue;
      const double f = w[r * 2 * s + c];
      if (f != 0.0)
        for (int j = 0; j < 2 * s; ++j) w[r * 2 * s + j] -= f * w[c * 2 * s + j];
    }
  }
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) inv[i * s + j] = w[i * 2 * s + s + j];
  return true;
}

// vecs: column w at vecs + w * d (d rows); vals ascending
void align_clusters(int d, int want, const double* vals, double* vecs, double gap) {
  int j0 = 0;
  while (j0 < want) {
    int j1 = j0 + 1;
    while (j1 < want && vals[j1] - vals[j1 - 1] <= gap) ++j1;
    const int s = j1 - j0;
    if (s >= 2 && s <= 8) {
      double y[64], yi[64];
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) y[i * s + j] = vecs[(size_t)(j0 + j) * d + (j0 + i)];
      bool ok = true;
      for (int it = 0; it < 30 && ok; ++it) {
        ok = small_inverse(s, y, yi);
        if (!ok) break;
        double delta = 0.0;
        for (int i = 0; i < s; ++i)
          for (int j = 0; j < s; ++j) {
            const double nv = 0.5 * (y[i * s + j] + yi[j * s + i]);
            delta = std::max(delta, std::fabs(nv - y[i * s + j]));
            y[i * s + j] = nv;
          }
        if (delta < 1e-15) break;
      }
      // the rotation must be orthogonal to rounding (Newton stalls on a
      // nearly singular block: then the cluster keeps the solver's basis)
      for (int i = 0; i < s && ok; ++i)
        for (int j = 0; j < s && ok; ++j) {
          double dot = 0.0;
          for (int k = 0; k < s; ++k) dot += y[k * s + i] * y[k * s + j];
          if (std::fabs(dot - (i == j ? 1.0 : 0.0)) > 1e-13) ok = false;
        }
      if (ok) {
        // y = polar factor U_p; Q = U_p^T: new column j = sum_i old column i * U_p(j, i)
        std::vector<double> tmp((size_t)d * s);
        for (int j = 0; j < s; ++j)
          for (int r = 0; r < d; ++r) {
            double acc = 0.0;
            for (int i = 0; i < s; ++i) acc += vecs[(size_t)(j0 + i) * d + r] * y[j * s + i];
            tmp[(size_t)j * d + r] = acc;
          }
        for (int j = 0; j < s; ++j)
          for (int r = 0; r < d; ++r) vecs[(size_t)(j0 + j) * d + r] = tmp[(size_t)j * d + r];
      }
    }
    j0 = j1;
  }
}

// H R^-1 for upper R (d x d, column-major), column by column of the result:
// Z[:, i] = (H[:, i] - sum_{t < i} R(t, i) Z[:, t]) / R(i, i).  The same
// substitution as a triangular solve with R^T (each entry subtracts its
// products in ascending t, then divides), but the inner loop runs over the
// independent entries of a column instead of one dependent dot product.
void right_solve_upper(int d, const double* R, const double* H, double* Z) {
  for (int i = 0; i < d; ++i) {
    double* zi = Z + (size_t)i * d;
    const double* hi = H + (size_t)i * d;
    for (int k = 0; k < d; ++k) zi[k] = hi[k];
    for (int t = 0; t < i; ++t) {
      const double rti = R[(size_t)t + (size_t)i * d];
      const double* zt = Z + (size_t)t * d;
      for (int k = 0; k < d; ++k) zi[k] -= rti * zt[k];
    }
    const double rii = R[(size_t)i + (size_t)i * d];
    for (int k = 0; k < d; ++k) zi[k] /= rii;
  }
}

// M = R^-T ga R^-1 by substitution (the reference's two triangular solves,
// multivec.py:206-208), symmetrised; ga symmetric, everything column-major.
void congruence_solve(int d, const double* R, const double* ga, double* M) {
  thread_local std::vector<double> z1, z1t, z2;
  z1.resize((size_t)d * d);
  z1t.resize((size_t)d * d);
  z2.resize((size_t)d * d);
  right_solve_upper(d, R, ga, z1.data());               // ga R^-1 = (R^-T ga)^T
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) z1t[(size_t)i + (size_t)j * d] = z1[(size_t)j + (size_t)i * d];
  right_solve_upper(d, R, z1t.data(), z2.data());        // (R^-T ga) R^-1
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i)
      M[(size_t)i + (size_t)j * d] =
          0.5 * (z2[(size_t)i + (size_t)j * d] + z2[(size_t)j + (size_t)i * d]);
}

// C = R^-1 V for upper R: back substitution on all `want` columns at once
// (V row-major d x want, so a row is contiguous); C column-major d x want.
void back_solve_upper(int d, int want, const double* R, const double* vcols, Mat* c_out) {
  thread_local std::vector<double> y;
  y.resize((size_t)d * want);
  for (int w = 0; w < want; ++w)
    for (int i = 0; i < d; ++i) y[(size_t)i * want + w] = vcols[(size_t)w * d + i];
  for (int i = d - 1; i >= 0; --i) {
    double* yi = y.data() + (size_t)i * want;
    for (int t = i + 1; t < d; ++t) {
      const double rit = R[(size_t)i + (size_t)t * d];
      const double* yt = y.data() + (size_t)t * want;
      for (int w = 0; w < want; ++w) yi[w] -= rit * yt[w];
    }
    const double rii = R[(size_t)i + (size_t)i * d];
    for (int w = 0; w < want; ++w) yi[w] /= rii;
  }
  Mat c(d, want);
  for (int w = 0; w < want; ++w)
    for (int i = 0; i < d; ++i) c(i, w) = y[(size_t)i * want + w];
  *c_out = std::move(c);
}

// Smallest `want` pairs of ga c = lam gb c given gb's factor; only the upper
// triangle of ga is read.
void pencil_solve(const Mat& ga_in, const PencilFactor& f, int want, double* vals_out,
                  Mat* c_out) {
  const int d = ga_in.r;
  Mat ga(d, d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i <= j; ++i) ga(i, j) = ga(j, i) = ga_in(i, j);
  if (f.Ri.empty() && !use_lapack() && !eig_lapack()) {
    // the default for pencils up to 64 x 64: substitution congruence (as
    // accurate as the reference's two triangular solves), tridiagonal QR,
    // cluster alignment, back substitution
    thread_local std::vector<double> m_, v_;
    m_.resize((size_t)d * d);
    congruence_solve(d, f.r.a.data(), ga.a.data(), m_.data());
    v_.assign((size_t)d * want, 0.0);
    RR_MARK(5);   // R^-T A R^-1
    if (d > 0 && symeig_tridiag_qr(d, m_.data(), want, vals_out, v_.data()) != 0)
      throw LapackError{"tql2 (no convergence)", 1};
    if (g_align_abs * g_align_mult > 0.0) {
      double scale = 0.0;
      for (int j = 0; j < want; ++j) scale = std::max(scale, std::fabs(vals_out[j]));
      align_clusters(d, want, vals_out, v_.data(),
                     std::min(f.floor_ * scale, g_align_abs * g_align_mult));
    }
    RR_MARK(6);   // symmetric eigensolve
    back_solve_upper(d, want, f.r.a.data(), v_.data(), c_out);
    return;
  }
  if (!f.Ri.empty()) {
    // M = R^-T ga R^-1 through the explicit inverse: row-oriented loops whose
    // inner index runs over independent entries (the substitution form is a
    // chain of dependent dot products, latency-bound at these sizes)
    const double* Ri = f.Ri.data();
    thread_local std::vector<double> t_, m_, u_, v_;
    m_.assign((size_t)d * d, 0.0);    // column-major (the eigensolver's layout)
    double* M = m_.data();
    if (g_dgemm) {
      // two BLAS products (one thread at these sizes): T = ga R^-1, then
      // U = R^-T T; Ri is R^-1 row-major, i.e. R^-T as a column-major array
      t_.assign((size_t)d * d, 0.0);
      u_.assign((size_t)d * d, 0.0);
      char nn = 'N', tt = 'T';
      int n_ = d;
      double one = 1.0, zero = 0.0;
      g_dgemm(&nn, &tt, &n_, &n_, &n_, &one, ga.a.data(), &n_, Ri, &n_, &zero, t_.data(), &n_);
      g_dgemm(&nn, &nn, &n_, &n_, &n_, &one, Ri, &n_, t_.data(), &n_, &zero, u_.data(), &n_);
      const double* U = u_.data();   // column-major
      for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i)
          M[i + (size_t)j * d] = 0.5 * (U[i + (size_t)j * d] + U[j + (size_t)i * d]);
    } else {
    t_.assign((size_t)d * d, 0.0);    // ga R^-1, row-major
    double* T = t_.data();
    for (int i = 0; i < d; ++i) {
      double* ti = T + (size_t)i * d;
      for (int k = 0; k < d; ++k) {
        const double g = ga(i, k);
        const double* rk = Ri + (size_t)k * d;
        for (int j = k; j < d; ++j) ti[j] += g * rk[j];
      }
    }
    // M(i, j) = sum_k Ri(k, i) T(k, j), k <= i; symmetrised as the reference
    u_.assign((size_t)d * d, 0.0);
    double* U = u_.data();   // row-major full product
    for (int i = 0; i < d; ++i) {
      double* ui = U + (size_t)i * d;
      for (int k = 0; k <= i; ++k) {
        const double rki = Ri[(size_t)k * d + i];
        const double* tk = T + (size_t)k * d;
        for (int j = 0; j < d; ++j) ui[j] += rki * tk[j];
      }
    }
    for (int j = 0; j < d; ++j)
      for (int i = 0; i < d; ++i)
        M[i + (size_t)j * d] = 0.5 * (U[(size_t)i * d + j] + U[(size_t)j * d + i]);
    }
    v_.assign((size_t)d * want, 0.0);
    RR_MARK(5);   // R^-T A R^-1
    if (d > 0 && symeig_tridiag_qr(d, M, want, vals_out, v_.data()) != 0) {
      throw LapackError{"tql2 (no convergence)", 1};
    }
    if (g_align_abs * g_align_mult > 0.0) {
      double scale = 0.0;
      for (int j = 0; j < want; ++j) scale = std::max(scale, std::fabs(vals_out[j]));
      align_clusters(d, want, vals_out, v_.data(),
                     std::min(f.floor_ * scale, g_align_abs * g_align_mult));
    }
    RR_MARK(6);   // symmetric eigensolve
    // C = R^-1 V
    Mat c(d, want);
    for (int w = 0; w < want; ++w) {
      const double* v = v_.data() + (size_t)w * d;
      for (int i = 0; i < d; ++i) {
        const double* ri = Ri + (size_t)i * d;
        double acc = 0.0;
        for (int k = i; k < d; ++k) acc += ri[k] * v[k];
        c(i, w) = acc;
      }
    }
    *c_out = std::move(c);
    return;
  }
  // the reference's sequence (multivec.gen_sym_eig, multivec.py:174-211):
  // M = R^-T ga R^-1 by two triangular solves (dtrtrs), symmetrised, eigh
  // (dsyevr, all pairs), C = R^-1 V -- used for every pencil size when the
  // eigensolve is dsyevr (B2L_RR_EIG=ref, or a pencil above 64 x 64; the
  // native forms above are the default below that size)
  const bool fl = eig_lapack();
  const Mat& r = f.r;
  Mat t = trsolve(r, ga, true, fl);
  t = trsolve(r, transpose(t), true, fl);
  Mat ts(d, d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) ts(i, j) = 0.5 * (t(i, j) + t(j, i));
  RR_MARK(5);   // R^-T A R^-1
  std::vector<double> w(d), z((size_t)d * d);
  // B2L_RR_MRRR=i: dsyevr's own stages with the MRRR vectors formed for the
  // `want` smallest only (cheaper; 20 / 32 converged on the C1 band against
  // the full call's 24 / 32 and the reference's 27 / 32, so off by default)
  static const bool mrrr_want = [] {
    const char* v = getenv("B2L_RR_MRRR");
    return v && v[0] == 'i';
  }();
  if (g_sytrd && g_stemr && g_ormtr && want < d && mrrr_want) {
    char uplo = 'U', jobz = 'V', range = 'I', side = 'L', trans = 'N';
    int n = d, lda = d, info = 0, il = 1, iu = want, mfound = 0, ldz = d, nzc = want;
    int tryrac = 1;
    double vl = 0.0, vu = 0.0;
    std::vector<double> dd(d), ee(d), tau(d), work((size_t)64 * d + 64);
    std::vector<int> isuppz(2 * d + 2), iwork((size_t)10 * d + 16);
    int lwork = (int)work.size(), liwork = (int)iwork.size();
    g_sytrd(&uplo, &n, ts.p(), &lda, dd.data(), ee.data(), tau.data(), work.data(), &lwork,
            &info);
    if (info != 0) throw LapackError{"dsytrd", info};
    ee[d - 1] = 0.0;
    g_stemr(&jobz, &range, &n, dd.data(), ee.data(), &vl, &vu, &il, &iu, &mfound, w.data(),
            z.data(), &ldz, &nzc, isuppz.data(), &tryrac, work.data(), &lwork, iwork.data(),
            &liwork, &info);
    if (info != 0 || mfound != want) throw LapackError{"dstemr", info ? info : -1};
    int nc = want;
    g_ormtr(&side, &uplo, &trans, &n, &nc, ts.p(), &lda, tau.data(), z.data(), &ldz, work.data(),
            &lwork, &info);
    if (info != 0) throw LapackError{"dormtr", info};
  } else {
    // dsyevr, range 'A', upper, abstol 0 (scipy.linalg.eigh defaults)
    char jobz = 'V', range = 'A', uplo = 'U';
    int n = d, lda = d, il = 1, iu = d, mfound = 0, ldz = d, info = 0;
    double vl = 0.0, vu = 0.0, abstol = 0.0;
    std::vector<double> work((size_t)26 * d + 64);
    std::vector<int> isuppz(2 * d + 2), iwork((size_t)10 * d + 16);
    int lwork = (int)work.size(), liwork = (int)iwork.size();
    g_syevr(&jobz, &range, &uplo, &n, ts.p(), &lda, &vl, &vu, &il, &iu, &abstol, &mfound,
            w.data(), z.data(), &ldz, isuppz.data(), work.data(), &lwork, iwork.data(), &liwork,
            &info);
    if (info != 0) throw LapackError{"dsyevr", info};
  }
  RR_MARK(6);   // symmetric eigensolve
  Mat v(d, want);
  for (int j = 0; j < want; ++j)
    for (int i = 0; i < d; ++i) v(i, j) = z[(size_t)i + (size_t)j * d];
  *c_out = trsolve(r, v, false, fl);
  for (int j = 0; j < want; ++j) vals_out[j] = w[j];
}

}  // namespace
}  // namespace b2l

using namespace b2l;

extern "C" int b2l_set_blas(void* dgemm) {
  g_dgemm = reinterpret_cast<dgemm_t*>(dgemm);
  return 0;
}

extern "C" int b2l_set_lapack_mrrr(void* dsytrd, void* dstemr, void* dormtr) {
  g_sytrd = reinterpret_cast<sytrd_t*>(dsytrd);
  g_stemr = reinterpret_cast<stemr_t*>(dstemr);
  g_ormtr = reinterpret_cast<ormtr_t*>(dormtr);
  return 0;
}

extern "C" int b2l_set_rr_align(double abs_gap) {
  g_align_abs = abs_gap > 0.0 ? abs_gap : 0.0;
  return 0;
}

namespace b2l {
void rr_set_align(double abs_gap) { g_align_abs = abs_gap > 0.0 ? abs_gap : 0.0; }
}  // namespace b2l

extern "C" int b2l_set_rr_reference(int on) {
  g_rr_ref = on < 0 ? -1 : (on ? 1 : 0);
  return 0;
}

extern "C" int b2l_set_lapack(void* dpotrf, void* dtrtrs, void* dtrtri, void* dsyevr) {
  if (!dpotrf || !dtrtrs || !dtrtri || !dsyevr)
    return fail(-B2L_EINVAL, "set_lapack: null routine");
  g_potrf = reinterpret_cast<potrf_t*>(dpotrf);
  g_trtrs = reinterpret_cast<trtrs_t*>(dtrtrs);
  g_trtri = reinterpret_cast<trtri_t*>(dtrtri);
  g_syevr = reinterpret_cast<syevr_t*>(dsyevr);
  return 0;
}

namespace b2l {

struct RRPlan;
inline RRPlan*& rr_tls_plan() {
  thread_local RRPlan* p = nullptr;
  return p;
}

// State between the two halves of the Rayleigh-Ritz step.
struct RRPlan {
  int m = 0, kst = 0, kj = 0, nw = 0, pending = 0;
  bool use_p = false;
  Mat mw, mp;
  std::vector<int> wcols, jact;
  Mat gXAP, gWAP, gPAP;   // A-side blocks that come from G1
  Mat axp, awp, app;      // ... folded with the W / P factors (first half)
  PencilFactor fac;       // of the final gb (after the repair ladder)
};

// First half (G1 only: B-Gram blocks and A P): Cholesky-QR of W and P with
// their ladders, gb and its factor with the pencil ladder (lobpcg.py:475-519).
int rr_begin(RRPlan& P, int m, int kst, int have_p, const double* g1, int ldg1, const int* jact,
             int kj, const int* sel, double pivot_floor, int* fallbacks_out) {
  if (m < 1 || kst < 0 || kj < 1 || kj > kst || kj > m || !g1 || !jact || !sel)
    return fail(-B2L_EINVAL, "rayleigh_ritz: bad arguments");
  g_rr_dim = m + kst + (have_p ? kj : 0);
  const int rW = m, rP = m + kst;
  const int cW = m, cP = m + kst, cAP = 2 * m + kst;
  auto G1 = [&](int i, int j) { return g1[(size_t)i * ldg1 + j]; };
  RR_MARK(-1);
  P = RRPlan{};
  P.m = m;
  P.kst = kst;
  P.kj = kj;
  P.jact.assign(jact, jact + kj);
  *fallbacks_out = 0;
  try {
    // W: Cholesky-QR with column dropping on the J sub-block (lobpcg.py:475-481)
    std::vector<int> keep(kj);
    for (int i = 0; i < kj; ++i) keep[i] = i;
    while (!keep.empty()) {
      const int k = (int)keep.size();
      Mat gww(k, k);
      for (int b = 0; b < k; ++b)
        for (int a = 0; a < k; ++a) gww(a, b) = G1(rW + sel[keep[a]], cW + sel[keep[b]]);
      try {
        P.mw = scaled_cholesky_inv(gww, pivot_floor);
        break;
      } catch (const NotSPD& e) {
        keep.erase(keep.begin() + e.pivot);
      }
    }
    P.pending += kj - (int)keep.size();
    if (keep.empty()) {
      *fallbacks_out = P.pending;
      return fail(-B2L_EDEGENERATE, "BasisDegeneracy");
    }
    P.nw = (int)keep.size();
    P.wcols.resize(P.nw);
    for (int i = 0; i < P.nw; ++i) P.wcols[i] = sel[keep[i]];

    // P_J: Cholesky-QR with floor; NotSPD drops P (lobpcg.py:484-494)
    if (have_p) {
      Mat gpp(kj, kj);
      for (int b = 0; b < kj; ++b)
        for (int a = 0; a < kj; ++a) gpp(a, b) = G1(rP + jact[a], cP + jact[b]);
      try {
        P.mp = scaled_cholesky_inv(gpp, pivot_floor);
        P.use_p = true;
      } catch (const NotSPD&) {
        P.pending += 1;
      }
    }
    RR_MARK(0);   // W and P Cholesky-QR
    auto block1 = [&](int r0, const int* ri, int nr, int c0, const int* ci, int nc) {
      Mat z(nr, nc);
      for (int b = 0; b < nc; ++b)
        for (int a = 0; a < nr; ++a) z(a, b) = G1(r0 + (ri ? ri[a] : a), c0 + ci[b]);
      return z;
    };
    const int nw = P.nw;
    Mat gXBW = block1(0, nullptr, m, cW, P.wcols.data(), nw);
    Mat gXBP, gWBP;
    if (have_p) {
      P.gXAP = block1(0, nullptr, m, cAP, jact, kj);
      P.gWAP = block1(rW, P.wcols.data(), nw, cAP, jact, kj);
      gXBP = block1(0, nullptr, m, cP, jact, kj);
      gWBP = block1(rW, P.wcols.data(), nw, cP, jact, kj);
      P.gPAP = block1(rP, jact, kj, cAP, jact, kj);
    }
    // the pencil's B side and its repair ladder (lobpcg.py:501-519): NotSPD
    // drops P, then a W column, then fails
    while (true) {
      const int kw = P.mw.c;
      const int kp = P.use_p ? kj : 0;
      const int d = m + kw + kp;
      Mat gb(d, d);
      for (int i = 0; i < m; ++i) gb(i, i) = 1.0;
      const Mat mwT = transpose(P.mw);
      const Mat bxw = matmul(gXBW, P.mw);
      for (int j = 0; j < kw; ++j) {
        gb(m + j, m + j) = 1.0;
        for (int i = 0; i < m; ++i) gb(i, m + j) = bxw(i, j);
      }
      if (kp) {
        const Mat bxp = matmul(gXBP, P.mp);
        const Mat bwp = matmul(matmul(mwT, gWBP), P.mp);
        const int o = m + kw;
        for (int j = 0; j < kp; ++j) {
          gb(o + j, o + j) = 1.0;
          for (int i = 0; i < m; ++i) gb(i, o + j) = bxp(i, j);
          for (int i = 0; i < kw; ++i) gb(m + i, o + j) = bwp(i, j);
        }
      }
      RR_MARK(1);   // blocks + pencil assembly (B side)
      try {
        pencil_factor(gb, pivot_floor, P.fac);
        break;
      } catch (const NotSPD& e) {
        P.pending += 1;
        if (P.use_p) {
          P.use_p = false;
        } else if (m <= e.pivot && e.pivot < m + kw && kw > 1) {
          Mat mw2(P.mw.r, kw - 1);
          int jj = 0;
          for (int j = 0; j < kw; ++j) {
            if (j == e.pivot - m) continue;
            for (int i = 0; i < P.mw.r; ++i) mw2(i, jj) = P.mw(i, j);
            ++jj;
          }
          P.mw = mw2;
        } else {
          *fallbacks_out = P.pending;
          return fail(-B2L_EDEGENERATE, "BasisDegeneracy");
        }
      }
    }
    // the pencil's A side that G1 already determines (the P blocks), so the
    // second half -- on the critical path once A W lands -- only adds the
    // blocks of [X ; W]^T A W
    if (P.use_p) {
      const Mat mwT = transpose(P.mw), mpT = transpose(P.mp);
      P.axp = matmul(P.gXAP, P.mp);
      P.awp = matmul(matmul(mwT, P.gWAP), P.mp);
      P.app = matmul(matmul(mpT, P.gPAP), P.mp);
    }
    *fallbacks_out = P.pending;
    return 0;
  } catch (const LapackError& e) {
    return fail(-B2L_ELAPACK, std::string("rayleigh_ritz: ") + e.what + " info " +
                                   std::to_string(e.info));
  } catch (const std::bad_alloc&) {
    return fail(-B2L_ENOMEM, "rayleigh_ritz: out of host memory");
  }
}

// Second half (needs G2 = [X ; W]^T A W): the pencil's A side, the
// eigensolve on the factor of the first half, the coefficient folding.
int rr_finish(RRPlan& P, const double* g2, const double* lam, double* lam_out, double* coef_out,
              int* pcols_out, int* kp_out, int* fallbacks_out) {
  if (!g2 || !lam) return fail(-B2L_EINVAL, "rayleigh_ritz: bad arguments");
  const int m = P.m, kst = P.kst, kj = P.kj, nw = P.nw;
  auto G2 = [&](int i, int j) { return g2[(size_t)i * kst + j]; };
  try {
    Mat gXAW(m, nw), gWAW(nw, nw);
    for (int b = 0; b < nw; ++b) {
      for (int a = 0; a < m; ++a) gXAW(a, b) = G2(a, P.wcols[b]);
      for (int a = 0; a < nw; ++a) gWAW(a, b) = G2(m + P.wcols[a], P.wcols[b]);
    }
    const int kw = P.mw.c;
    const int kp = P.use_p ? kj : 0;
    const int d = m + kw + kp;
    Mat ga(d, d);
    for (int i = 0; i < m; ++i) ga(i, i) = lam[i];
    const Mat mwT = transpose(P.mw);
    const Mat aww = matmul(matmul(mwT, gWAW), P.mw);
    const Mat axw = matmul(gXAW, P.mw);
    for (int j = 0; j < kw; ++j) {
      for (int i = 0; i < kw; ++i) ga(m + i, m + j) = aww(i, j);
      for (int i = 0; i < m; ++i) ga(i, m + j) = axw(i, j);
    }
    if (kp) {
      const Mat& axp = P.axp;
      const Mat& awp = P.awp;
      const Mat& app = P.app;
      const int o = m + kw;
      for (int j = 0; j < kp; ++j) {
        for (int i = 0; i < m; ++i) ga(i, o + j) = axp(i, j);
        for (int i = 0; i < kw; ++i) ga(m + i, o + j) = awp(i, j);
        for (int i = 0; i < kp; ++i) ga(o + i, o + j) = app(i, j);
      }
    }
    Mat c;
    std::vector<double> vals(m);
    pencil_solve(ga, P.fac, m, vals.data(), &c);
    RR_MARK(2);   // generalized eigensolve
    // fold the orthonormalization into raw-block coefficients
    Mat cw(kw, m), cp(kp, m);
    for (int j = 0; j < m; ++j) {
      for (int i = 0; i < kw; ++i) cw(i, j) = c(m + i, j);
      for (int i = 0; i < kp; ++i) cp(i, j) = c(m + kw + i, j);
    }
    const Mat cwr = matmul(P.mw, cw);   // nw x m -> rows wcols of the kst x m block
    double* cx_o = coef_out;
    double* cw_o = coef_out + (size_t)m * m;
    double* cp_o = cw_o + (size_t)kst * m;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) cx_o[(size_t)i * m + j] = c(i, j);
    for (size_t e = 0; e < (size_t)kst * m; ++e) cw_o[e] = 0.0;
    for (int i = 0; i < nw; ++i)
      for (int j = 0; j < m; ++j) cw_o[(size_t)P.wcols[i] * m + j] = cwr(i, j);
    if (kp) {
      const Mat cpr = matmul(P.mp, cp);
      for (int i = 0; i < kp; ++i) {
        pcols_out[i] = P.jact[i];
        for (int j = 0; j < m; ++j) cp_o[(size_t)i * m + j] = cpr(i, j);
      }
    }
    for (int j = 0; j < m; ++j) lam_out[j] = vals[j];
    *kp_out = kp;
    *fallbacks_out = P.pending;
    RR_MARK(3);   // coefficient folding
    return 0;
  } catch (const LapackError& e) {
    return fail(-B2L_ELAPACK, std::string("rayleigh_ritz: ") + e.what + " info " +
                                   std::to_string(e.info));
  } catch (const std::bad_alloc&) {
    return fail(-B2L_ENOMEM, "rayleigh_ritz: out of host memory");
  }
}

// The two halves on a per-thread plan (b2l_fast_iteration).
int rr_begin_tls(int m, int kst, int have_p, const double* g1, int ldg1, const int* jact, int kj,
                 const int* sel, double pivot_floor, int* fallbacks_out) {
  thread_local RRPlan plan_;
  rr_tls_plan() = &plan_;
  return rr_begin(plan_, m, kst, have_p, g1, ldg1, jact, kj, sel, pivot_floor, fallbacks_out);
}
int rr_finish_tls(const double* g2, const double* lam, double* lam_out, double* coef_out,
                  int* pcols_out, int* kp_out, int* fallbacks_out) {
  RRPlan* p = rr_tls_plan();
  if (!p) return fail(-B2L_EINVAL, "rayleigh_ritz: finish without begin");
  return rr_finish(*p, g2, lam, lam_out, coef_out, pcols_out, kp_out, fallbacks_out);
}

// Drift repair, folded (_refresh_ritz lobpcg.py:280-296): from the Grams
// gxx = X^T B X and gxa = X^T A X of the drifted block (m x m row-major,
// upper triangles read), the rotation M = R_eff^-1 Q that the reference
// applies in two steps -- X <- X R_eff^-1 (b_orthonormalize) then X <- X Q
// with (lam, Q) = eigh of the re-projected X^T A X -- computed on the small
// matrices: Q diagonalises R_eff^-T gxa R_eff^-1.  The LAPACK routines the
// Python path uses (small.scaled_cholesky / sym_eig: dpotrf, dtrtri, dsyevr)
// when registered.  m_out row-major m x m; lam_out ascending.  Returns 0,
// or 1 when gxx is not SPD (the caller's path reports BasisDegeneracy).
int repair_coef(int m, const double* gxx, const double* gxa, double* lam_out, double* m_out) {
  const int saved = g_rr_dim;
  g_rr_dim = 1 << 20;   // use_lapack(): the routines small.py calls
  struct Restore {
    int v;
    ~Restore() { g_rr_dim = v; }
  } restore{saved};
  try {
    Mat G(m, m), A(m, m);
    for (int i = 0; i < m; ++i)
      for (int j = i; j < m; ++j) {
        G(i, j) = G(j, i) = gxx[(size_t)i * m + j];
        A(i, j) = A(j, i) = gxa[(size_t)i * m + j];
      }
    const Mat minv = scaled_cholesky_inv(G, 0.0);
    const Mat T = matmul(transpose(minv), matmul(A, minv));
    Mat S(m, m);   // upper triangle of T read, as eigh(lower=False)
    for (int j = 0; j < m; ++j)
      for (int i = 0; i <= j; ++i) S(i, j) = S(j, i) = T(i, j);
    Mat V(m, m);
    if (g_syevr) {
      char jobz = 'V', range = 'A', uplo = 'U';
      int n = m, lda = m, il = 1, iu = m, mfound = 0, ldz = m, info = 0;
      double vl = 0.0, vu = 0.0, abstol = 0.0;
      std::vector<double> z((size_t)m * m), work((size_t)26 * m + 64);
      std::vector<int> isuppz(2 * m + 2), iwork((size_t)10 * m + 16);
      int lwork = (int)work.size(), liwork = (int)iwork.size();
      g_syevr(&jobz, &range, &uplo, &n, S.p(), &lda, &vl, &vu, &il, &iu, &abstol, &mfound,
              lam_out, z.data(), &ldz, isuppz.data(), work.data(), &lwork, iwork.data(), &liwork,
              &info);
      if (info != 0) throw LapackError{"dsyevr", info};
      V.a = z;
    } else if (symeig_tridiag_qr(m, S.p(), m, lam_out, V.p()) != 0) {
      throw LapackError{"tql2 (no convergence)", 1};
    }
    const Mat M = matmul(minv, V);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) m_out[(size_t)i * m + j] = M(i, j);
    return 0;
  } catch (const NotSPD&) {
    return 1;
  } catch (const LapackError& e) {
    return fail(-B2L_ELAPACK, std::string("drift repair: ") + e.what + " info " +
                                   std::to_string(e.info));
  }
}

}  // namespace b2l

extern "C" int b2l_rayleigh_ritz_begin(int m, int kst, int have_p, const double* g1, int ldg1,
                                       const int* jact, int kj, const int* sel,
                                       double pivot_floor, int* fallbacks_out) {
  return rr_begin_tls(m, kst, have_p, g1, ldg1, jact, kj, sel, pivot_floor, fallbacks_out);
}

extern "C" int b2l_rayleigh_ritz_finish(const double* g2, const double* lam, double* lam_out,
                                        double* coef_out, int* pcols_out, int* kp_out,
                                        int* fallbacks_out) {
  *kp_out = 0;
  return rr_finish_tls(g2, lam, lam_out, coef_out, pcols_out, kp_out, fallbacks_out);
}

extern "C" int b2l_rayleigh_ritz(int m, int kst, int have_p, const double* g1, int ldg1,
                                 const double* g2, const double* lam, const int* jact, int kj,
                                 const int* sel, double pivot_floor, double* lam_out,
                                 double* coef_out, int* pcols_out, int* kp_out,
                                 int* fallbacks_out) {
  if (!g2 || !lam) return fail(-B2L_EINVAL, "rayleigh_ritz: bad arguments");
  thread_local RRPlan plan;
  *kp_out = 0;
  const int rc = rr_begin(plan, m, kst, have_p, g1, ldg1, jact, kj, sel, pivot_floor,
                          fallbacks_out);
  if (rc) return rc;
  return rr_finish(plan, g2, lam, lam_out, coef_out, pcols_out, kp_out, fallbacks_out);
}
