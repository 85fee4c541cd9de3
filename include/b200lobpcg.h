/*
 * libb200lobpcg -- C ABI of the B200 (sm_100a) LOBPCG hot path.
 *
 * Drop-in boundary for the reference package `blockeig`
 * (/root/reference/pkg/src/blockeig).  The reference's Python entry point
 * `solve(a, b=None, t=None, y=None, x0=None, config=None)`
 * (lobpcg.py:343) stays in host Python; every operation it performs on the
 * long dimension n is one of the calls below.  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *  - A "block" is a row-major (point-major) fp64 array of shape (n, ld): row r
 *    holds the k <= ld columns of grid point r, exactly the reference's numpy
 *    C-order (n, k) multivector (multivec.py:1-15, :220-229) padded to an even
 *    leading dimension ld (16-byte rows, required by TMA).
 *  - Grid point p = i + nx*(j + ny*k), x fastest (operators.py:63-67).
 *  - All pointers are device pointers unless stated; all calls are
 *    asynchronous on `stream` (a cudaStream_t / CUstream passed as void*).
 *    The library never frees or retains caller memory.
 *  - Every call returns 0 on success, a negative code on failure (-cudaError
 *    for CUDA runtime errors, -1000.. for argument/driver errors); the message
 *    is in b2l_last_error() (thread-local).
 *  - Reductions are deterministic (fixed CTA row assignment, fixed-order
 *    second stage): a given device, shape and input give identical bits.
 *  - One host thread / one stream per device: the library keeps one growable
 *    scratch buffer per device for CTA partials.
 */
#ifndef B200LOBPCG_H
#define B200LOBPCG_H

#ifdef __cplusplus
extern "C" {
#endif

#define B2L_ABI_VERSION 1

typedef struct {
  const double* ptr; /* device pointer to an (n, ld) block */
  int ld;            /* leading dimension (doubles per row), even */
  int cols;          /* number of columns used, <= ld */
} b2l_block;

/* Last error message of this thread ("" if none). */
const char* b2l_last_error(void);

/* B2L_ABI_VERSION of the loaded library. */
int b2l_abi_version(void);

/* Fails unless the current device is sm_100 (B200). */
int b2l_device_info(int* sm_count, int* cc_major, int* cc_minor);

/*
 * K1 -- 7-point Dirichlet Laplacian, fused over all ld columns of a block.
 * Replaces Laplacian3D._apply (operators.py:184-196) and the harness scaling
 * MatrixFreeOperator(n, lambda v: s*L(v)) (operators.py:104-121):
 *   out = scale * ((((((6x - x[i-1]) - x[i+1]) - x[j-1]) - x[j+1]) - x[k-1]) - x[k+1])
 * bitwise equal to the reference (same operation order, no FMA contraction).
 * `in` and `out` are (nx*ny*nz, ld) blocks of the nz locally owned z-planes.
 * `halo` (nullable) holds two ghost planes [lo; hi] of shape (2*nx*ny, ld)
 * for a z-slab partition; has_lo/has_hi select them, otherwise the missing
 * neighbour plane is the Dirichlet zero.  in != out.
 */
int b2l_stencil7(const double* in, double* out, int nx, int ny, int nz, int ld,
                 const double* halo, int has_lo, int has_hi, double scale,
                 void* stream);

/*
 * K5 -- multi-block tall-skinny Gram  out = [L_0 .. L_{nl-1}]^T diag(w)^? [R_0 ..]
 * Replaces multivec.gram (multivec.py:58-71) for all the Gram products of one
 * LOBPCG step (lobpcg.py:419, :176, :318-338) in a single pass over the rows.
 * Right block j is multiplied row-wise by `weight` (diag(B), DiagonalOperator
 * operators.py:151-152) when bit j of right_weighted_mask is set.
 * `out` is a dense row-major (sum L cols) x (sum R cols) device matrix.
 * pair_mode (host array nleft*nright, nullable = all 1): 0 = the block pair
 * (l, r) is not needed, 1 = full, 2 = upper triangle only (a symmetric
 * diagonal pair such as X^T B X); entries outside requested pairs are
 * unspecified.  nleft <= 4, nright <= 8, at most 8 distinct blocks, at most
 * 1024 8x8 output tiles.  Computed on the fp64 tensor cores (DMMA).
 */
int b2l_gram(int nrows, const b2l_block* left, int nleft, const b2l_block* right,
             int nright, unsigned right_weighted_mask, const double* weight,
             const unsigned char* pair_mode, double* out, void* stream);

/*
 * K4+K2 -- residual, preconditioner, squared column norms.
 * Replaces lobpcg.py:429-430 (W_full = AX - BX*lam; column_norms,
 * multivec.py:214-217) and the preconditioner callback t(W) of lobpcg.py:467
 * for the built-in Jacobi/identity preconditioners (operators.py:280-298):
 *   wf[:, j] = AX[:, j] - (bdiag? bdiag*X[:, j] : X[:, j]) * lam[j]
 *   sums_out[j]      = sum_r wf[r, j]^2                      (j < m)
 *   sums_out[m + j]  = sum_r AX[r, j]^2  if want_ax_norms      (relative tol)
 *   W[:, wpos[j]]    = T wf[:, j]  for every j with wpos[j] >= 0
 * T: tmode 0 identity, 1 scalar tinv, 2 row vector tvec.  X and AX share ldx;
 * lam, wpos and sums_out are device arrays of m (sums_out: 2m).
 */
int b2l_residual(int nrows, int m, const double* x, const double* ax, int ldx,
                 const double* bdiag, const double* lam, int tmode, double tinv,
                 const double* tvec, const int* wpos, int kw, double* w, int ldw,
                 int want_ax_norms, double* sums_out, void* stream);

/*
 * K6 -- Ritz block update (lobpcg.py:520-540, multivec.multiply
 * multivec.py:74-86), with the Cholesky-QR factors of W and P already folded
 * into cw/cp (replaces tri_solve_right, multivec.py:125-146, at
 * lobpcg.py:177-178 and :491):
 *   P'  = W Cw + P[:, pcols] Cp        AP' = AW Cw + AP[:, pcols] Cp
 *   X'  = X Cx (+ P' if x_plus_p)      AX' = AX Cx (+ AP')
 * cx (m x m), cw (kw x m), cp (kp x m) row-major device matrices; pcols
 * (kp ints) device.  ax/axo/aw/ap may be NULL (no A side); po/apo NULL skips
 * writing P'.  x = NULL (cx ignored, no A side): xo = W Cw + P Cp, the plain
 * block product multivec.multiply.  Outputs must not alias inputs.
 */
int b2l_update(int nrows, int m, const double* x, const double* ax, int ldx,
               const double* cx, const double* w, const double* aw, int ldw, int kw,
               const double* cw, const double* p, const double* ap, int ldp,
               const int* pcols, int kp, const double* cp, double* xo, double* axo,
               int ldo, double* po, double* apo, int ldpo, int x_plus_p,
               void* stream);

/*
 * K1+K5b -- b2l_stencil7 fused with the Rayleigh-Ritz Gram blocks that
 * involve A W (reference lobpcg.py:325 gram(w, aw), :327 gram(x, aw)):
 *   out = A in  (as b2l_stencil7)   and
 *   gram_out ((m + kw) x kw, row-major, device) = [X[:, :m] ; in[:, :kw]]^T out[:, :kw]
 * X is an (n, ldx) block of the same grid rows.  A W is never re-read.
 * m = 0 (x may be NULL): gram_out = in^T out (kw x kw) -- the curvatures
 * p_j^T A p_j of the column-batched PCG (b2l_pcg_*).
 */
int b2l_stencil7_gram(const double* in, double* out, int nx, int ny, int nz, int ld,
                      const double* halo, int has_lo, int has_hi, double scale,
                      const double* x, int ldx, int m, int kw, double* gram_out,
                      void* stream);

/*
 * F1 -- one fused pass of the LOBPCG iteration (lobpcg.py:520-540 for this
 * iteration, then :419-467 and the non-AW Gram blocks of :299-340 for the
 * next one):
 *   P' = W Cw + P[:, pcols] Cp ; AP' likewise ; X' = X Cx + P' ; AX' likewise
 *   W'[:, wpos[j]] = T (AX'[:, j] - (bdiag? bdiag*X' : X')[:, j] lam[j])
 *   red_out = [ sum_r wf^2 (m) | sum_r AX'^2 (m, if want_ax_norms) |
 *               G (a x b) ]      with a = 2m + kw_next, b = 3m + kw_next,
 *   G = [X' W' P']^T [B X', B W', B P', AP']  -- only the upper triangles of
 *   the three symmetric diagonal pairs and the pairs X'-W', X'-P', W'-P',
 *   X'-AP', W'-AP', P'-AP' are defined.
 * coef = [Cx (m x m) | Cw (kw x m) | Cp (kp x m)] row-major, device.
 * x/ax/p/ap and xo/axo/po/apo are (n, ldx); w/aw (n, ldw); w_next (n, ldw_next).
 * Outputs must not alias inputs.  m <= 16.
 */
int b2l_lobpcg_step(int nrows, int m, const double* x, const double* ax, int ldx,
                    const double* w, const double* aw, int ldw, int kw, const double* p,
                    const double* ap, int kp, const int* pcols, const double* coef,
                    double* xo, double* axo, double* po, double* apo, const double* lam,
                    const double* bdiag, int tmode, double tinv, const double* tvec,
                    const int* wpos, int kw_next, double* w_next, int ldw_next,
                    int want_ax_norms, double* red_out, void* stream);

/*
 * K9 -- the seeded initial block on the device, bit for bit the reference's
 * multivec.seeded_random_fill (multivec.py:220-229):
 *   Generator(PCG64(seed)).uniform(low, high, (n, m))  (C order)
 * out[r*ld + j] (r < nrows, j < m) = draw (first_draw + r*m + j) of the PCG64
 * stream whose state before its first draw is (state_hi:state_lo) with
 * increment (inc_hi:inc_lo) -- numpy's bit_generator.state['state'].
 * first_draw = row0*m gives a z-slab its rows of the global block.  Columns
 * m..ld-1 are not written.
 */
int b2l_seeded_fill(double* out, int ld, long long nrows, int m, long long first_draw,
                    unsigned long long state_hi, unsigned long long state_lo,
                    unsigned long long inc_hi, unsigned long long inc_lo, double low,
                    double high, void* stream);

/*
 * Inner-PCG preconditioner, column-batched (reference operators.py:341-427,
 * pcg_solve / InnerPCGPreconditioner): the k columns of an (n, ld) block run
 * pcg_solve side by side, each with its own scalars, all kept on the device.
 * M (the PCG's own preconditioner): tmode 0 identity, 1 scalar tinv, 2 row
 * vector tvec (Jacobi), 3 z = M r supplied by the caller in the block z.
 *   init      : x = 0, r = b, p = M b ; sums_out = [b^T b | r^T M r]     (2k)
 *   (A p and pap_j = p_j^T A p_j: b2l_stencil7_gram with m = 0, or any
 *    operator + b2l_gram)
 *   update    : alpha_j = rz_j / pap_j ; x += alpha p ; r -= alpha A p ;
 *               sums_out = [r^T M r | r^T r] (tmode 3: [0 | r^T r]);
 *               *err |= 1 if a live column has pap <= 0 or non-finite
 *               (the reference's PCGBreakdown)
 *   dot       : tmode 3 only: sums_out = [r^T z | r^T r]
 *   direction : a column stops when ||r|| <= rtol ||b|| (rtol > 0) or
 *               r^T M r == 0; live columns get p = M r + (rz_next / rz) p;
 *               done_next / rz_next are the next step's flags / rz.
 * Columns with b = 0 or done[j] != 0 are left untouched.  Elementwise
 * arithmetic rounds like numpy (product, then sum); reductions are
 * deterministic.
 */
int b2l_pcg_init(int nrows, int k, const double* b, int ldb, double* x, double* r, double* p,
                 int ld, const double* z, int tmode, double tinv, const double* tvec,
                 double* sums_out, void* stream);
int b2l_pcg_update(int nrows, int k, double* x, double* r, const double* p, const double* ap,
                   int ld, const double* pap, int pap_stride, const double* rz,
                   const double* bb, const int* done, int tmode, double tinv,
                   const double* tvec, double* sums_out, int* err, void* stream);
int b2l_pcg_dot(int nrows, int k, const double* r, const double* z, int ld, const double* bb,
                const int* done, double* sums_out, void* stream);
int b2l_pcg_direction(int nrows, int k, const double* r, double* p, int ld, const double* z,
                      int tmode, double tinv, const double* tvec, const double* rz,
                      const double* sums, const double* bb, double rtol, const int* done,
                      int* done_next, double* rz_next, void* stream);

/*
 * Host, small dense: register the LAPACK routines the Rayleigh-Ritz step uses
 * (dpotrf, dtrtrs, dtrtri, dsyevr with the Fortran-style signatures of
 * scipy.linalg.cython_lapack, i.e. the routines scipy.linalg.cholesky /
 * solve_triangular / eigh run for the reference, multivec.py:89-211).
 */
int b2l_set_lapack(void* dpotrf, void* dtrtrs, void* dtrtri, void* dsyevr);

/*
 * Host, small dense: optionally register dsyevr's three stages (dsytrd,
 * dstemr, dormtr; same signatures as scipy.linalg.cython_lapack): the
 * reference-form eigensolve then runs dsyevr's all-pairs path (MRRR) but
 * forms and back-transforms only the wanted vectors.
 */
int b2l_set_lapack_mrrr(void* dsytrd, void* dstemr, void* dormtr);

/*
 * Host, small dense: optionally register BLAS dgemm (Fortran-style signature
 * of scipy.linalg.cython_blas) for the block products of large pencils
 * (m >= 32); null keeps the native loops.
 */
int b2l_set_blas(void* dgemm);

/*
 * Host, small dense: which form the next Rayleigh-Ritz calls of this thread
 * use for pencils up to 64 x 64.  0 / -1 (default): the native
 * substitution congruence + tridiagonal QR, with the computed
 * eigenvectors of numerically degenerate clusters aligned to the current Ritz
 * vectors (b2l_set_rr_align); 1: the reference's own sequence
 * (multivec.gen_sym_eig: two dtrtrs, dsyevr on all pairs, dtrtrs), ~50 us
 * slower per C2 iteration.  Inside (near-)degenerate clusters the basis an
 * eigensolver returns steers which Ritz column locks first: on C1 over 128
 * perturbed problems the reference converges without a basis fallback 117
 * times, form 1 97, the plain QR 39, the aligned QR 128.  The
 * environment B2L_RR_EIG=qr / =ref pins one form.
 */
int b2l_set_rr_reference(int on);

/*
 * Host, small dense: the absolute eigenvalue gap below which the native
 * eigensolve of this thread treats wanted eigenvalues as one cluster and
 * returns the cluster's basis closest to the current Ritz vectors (capped at
 * pivot_floor * max|lambda|).  The solver sets a tenth of its smallest lock
 * threshold before every Rayleigh-Ritz call (lobpcg.py:429-437 thresholds):
 * wide enough to pin the basis of a numerically degenerate cluster, narrow
 * enough that the step still separates eigenvalues it can resolve;
 * 0 (the initial value): no alignment, any valid basis.
 */
int b2l_set_rr_align(double abs_gap);

/*
 * Host, small dense -- the Rayleigh-Ritz step of one iteration with the
 * reference's repair ladders (lobpcg.py:475-519; b_orthonormalize :147-200;
 * rayleigh_ritz :299-340 on the projected blocks), given the device Grams:
 *   g1 (a x ldg1, row-major): rows [X (m) | W (kst) | P (m, if have_p)],
 *       cols [BX (m) | BW (kst) | BP (m) | AP (m)]  (b2l_lobpcg_step / b2l_gram)
 *   g2 ((m + kst) x kst, row-major): [X ; W]^T A W  (b2l_stencil7_gram)
 *   lam (m) current Ritz values; jact (kj) active columns; sel (kj) their
 *   positions among the kst stored W columns.
 * Outputs: lam_out (m) next Ritz values; coef_out = [Cx (m x m) | Cw (kst x m)
 * | Cp (kp x m)] row-major with the W / P Cholesky-QR factors folded in (the
 * b2l_lobpcg_step / b2l_update layout); pcols_out (kp = *kp_out, 0 when P was
 * dropped); *fallbacks_out = basis repairs taken (dropped W columns, dropped
 * P, eigensolve retries).  Returns -B2L_EDEGENERATE (-1003) when the ladder
 * is exhausted (the reference's BasisDegeneracy status).
 */
int b2l_rayleigh_ritz(int m, int kst, int have_p, const double* g1, int ldg1,
                      const double* g2, const double* lam, const int* jact, int kj,
                      const int* sel, double pivot_floor, double* lam_out, double* coef_out,
                      int* pcols_out, int* kp_out, int* fallbacks_out);

/*
 * The same step in two halves on a per-thread plan, so a caller can run the
 * first while the pass producing g2 (A W) is still on the GPU:
 *   _begin: the G1-only half -- W / P Cholesky-QR with their ladders, the
 *           pencil's B side, its Cholesky factor and repair ladder;
 *   _finish: the pencil's A side from g2, the eigensolve, the coefficients.
 * Arguments and return codes as b2l_rayleigh_ritz (kst is the g2 row stride).
 */
int b2l_rayleigh_ritz_begin(int m, int kst, int have_p, const double* g1, int ldg1,
                            const int* jact, int kj, const int* sel, double pivot_floor,
                            int* fallbacks_out);
int b2l_rayleigh_ritz_finish(const double* g2, const double* lam, double* lam_out,
                             double* coef_out, int* pcols_out, int* kp_out, int* fallbacks_out);

/*
 * Steady-state iteration, host driven natively (lobpcg.py:418-540 when the
 * previous step ran b2l_lobpcg_step + b2l_stencil7_gram): one stream
 * synchronisation fetching red_dev (2m + a*b, a = 2m + kst, b = 3m + kst) and
 * g2_dev ((m + kst) x kst) into the pinned h_red / h_g2; the drift test; the
 * lock test (updates active, lock_iteration; writes norms, newly); the
 * Rayleigh-Ritz step (b2l_rayleigh_ritz, output staged in the pinned
 * h_stage (>= 3m^2 + m doubles) / h_istage (>= 2m ints)); then the launches
 * of the next b2l_lobpcg_step (x,ax,p,ap,w_cur -> x2,ax2,p2,ap2,w_next; the
 * coefficients, Ritz values, pcols and wpos travel by value in the launch)
 * and b2l_stencil7_gram (w_next -> aw, [x2 ; w_next]^T aw).  Their
 * reductions are written straight into h_red / h_g2 when those are
 * device-mapped pinned buffers (red_on_host = 1), else into red_dev / g2_dev
 * and copied at the next call.  coef_dev / lam_dev / pcols_dev are unused.
 * Returns B2L_ITER_OK (next passes queued; lam_next, k_next, kp, fallbacks
 * set), B2L_ITER_DRIFT (the block lost B-orthonormality beyond repair by
 * the native path -- X^T B X not SPD, or B2L_NATIVE_REPAIR=0 -- nothing changed
 * but drift and the fetched h_red / h_g2: the caller repairs), B2L_ITER_DONE (lock test applied, loop over),
 * -1003 (B2L_EDEGENERATE, lock test applied) or another negative error.
 */
#define B2L_ITER_OK 0
#define B2L_ITER_DRIFT 1
#define B2L_ITER_DONE 2

typedef struct {
  int n, m, ldx;                      /* rows, block size, leading dim of X-like blocks */
  int nx, ny, nz;                     /* grid of the built-in stencil */
  double scale;                       /* stencil scale s */
  int tmode;                          /* preconditioner: 0 none, 1 scalar, 2 vector */
  double tinv;
  const double* tvec;
  const double* bdiag;                /* diag(B) or NULL */
  double tol;
  int relative_tol, max_iter;
  double drift_limit, pivot_floor;
  double *x, *ax, *p, *ap;            /* current blocks (device) */
  double *x2, *ax2, *p2, *ap2;        /* next blocks (device) */
  double *w_cur, *w_next, *aw;        /* W buffers and the AW buffer (device) */
  double *red_dev, *g2_dev;           /* reductions of F1 / the stencil pass (device) */
  double *coef_dev, *lam_dev;         /* device staging */
  int* pcols_dev;                     /* device staging, 2m ints */
  double *h_red, *h_g2, *h_stage;     /* pinned host */
  int* h_istage;                      /* pinned host */
  double* lam;                        /* (m) current Ritz values (host) */
  unsigned char* active;              /* (m) in/out */
  long long* lock_iteration;          /* (m) in/out */
  int it, have_p, kst;                /* iteration, P valid, stored W columns */
  void* stream;
  double* norms;                      /* out (m) */
  unsigned char* newly;               /* out (m) */
  double* lam_next;                   /* out (m) */
  double drift;                       /* out */
  int fallbacks, k_next, kp;          /* out */
  int red_on_host;                    /* in/out: 1 when the queued passes write
                                         h_red / h_g2 directly (mapped pinned
                                         memory); the caller sets 0 whenever it
                                         queued the passes itself; 3 when a
                                         z-slab step left them reduced over
                                         the ranks in h_red / h_g2 */
  int repaired;                       /* out: 1 when the drift test fired and
                                         the step repaired the block natively
                                         (the repaired Ritz values are in lam;
                                         the step's outputs then sit in x, ax,
                                         p, ap, w_cur -- DONE / EDEGENERATE:
                                         in x2, ax2, p2, ap2, w_next) */
  struct b2l_slab* slab;              /* z-slab context (b2l_slab_create) or
                                         NULL: one GPU holds the whole grid.
                                         With a communicator, the halo of W'
                                         is exchanged under the interior
                                         stencil planes and F1's reductions
                                         and the stencil pass's Gram are
                                         summed over the ranks (NCCL) before
                                         the host reads them. */
} b2l_iter_state;

int b2l_fast_iteration(b2l_iter_state* state);

/* sizeof(b2l_iter_state) as compiled into the library (binding checks). */
int b2l_iter_state_size(void);

/*
 * Diagnostics: host-side phase times of b2l_fast_iteration, accumulated when
 * the environment has B2L_ITER_PROFILE=1 (returns 1 then, else 0).
 * out[8] = calls, fetch enqueue, wait in the synchronisation, drift + lock
 * tests, Rayleigh-Ritz second half, uploads + launches, Rayleigh-Ritz first
 * half, wait for the stencil pass's Gram (microseconds, summed over calls).
 */
int b2l_iter_profile(double* out, int reset);

/*
 * z-slab decomposition over the GPUs of one node (the survey's
 * b2l_ctx_create with its NCCL communicator), one process per GPU.  Rank r
 * owns z-planes [floor(r N/P), floor((r+1) N/P)) -- a contiguous row range of
 * every block.  Replaces nothing in the reference (single process,
 * SPEC.md:317); the paper's runs used the same decomposition through MPI
 * inside hypre.
 *
 * NCCL is bound at run time to the libnccl.so.2 already in the process
 * (PyTorch's), else `path`.  b2l_nccl_unique_id fills a 128-byte id on one
 * rank; the caller broadcasts it (torch.distributed) and every rank calls
 * b2l_slab_create with it.  nccl_id NULL (world 1 only): no communicator,
 * every collective is the identity.
 *
 * b2l_slab_stencil7 / _gram: b2l_stencil7 / b2l_stencil7_gram on this rank's
 * nz_local planes; the two boundary planes of `in` go to the neighbours on
 * the context's communication stream while the interior planes are
 * computed, the two edge planes after the halo landed.  gram_out is this
 * rank's part (sum it with b2l_slab_allreduce).
 * b2l_slab_allreduce: in-place fp64 sum over the ranks on `stream`.
 * b2l_stencil7_gram_split: b2l_stencil7_gram in the same interior + edge
 * launches with a caller-supplied halo and no communication (tests).
 */
typedef struct b2l_slab b2l_slab;
int b2l_nccl_load(const char* path);
int b2l_nccl_unique_id(unsigned char* out, int len);
int b2l_slab_create(const unsigned char* nccl_id, int world, int rank, int nx, int ny,
                    int nz_local, b2l_slab** out);
int b2l_slab_destroy(b2l_slab* slab);
int b2l_slab_info(const b2l_slab* slab, int* world, int* rank, int* has_comm);
int b2l_slab_allreduce(b2l_slab* slab, double* buf, long long count, void* stream);
int b2l_slab_stencil7(b2l_slab* slab, const double* in, double* out, int ld, double scale,
                      void* stream);
int b2l_slab_stencil7_gram(b2l_slab* slab, const double* in, double* out, int ld, double scale,
                           const double* x, int ldx, int m, int kw, double* gram_out,
                           void* stream);
int b2l_stencil7_gram_split(const double* in, double* out, int nx, int ny, int nz, int ld,
                            const double* halo, int has_lo, int has_hi, double scale,
                            const double* x, int ldx, int m, int kw, double* gram_out,
                            void* stream);

/* Number of kernels this library has launched in the process (all entry
 * points, including the ones b2l_fast_iteration queues). */
long long b2l_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* B200LOBPCG_H */
