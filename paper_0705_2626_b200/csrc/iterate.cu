// Steady-state LOBPCG iteration driven natively (host side of one step of
// reference lobpcg.py:418-540 when the previous step ran the fused passes):
//   fetch F1's reductions and the stencil pass's [X W]^T A W (one
//   synchronisation) -> drift test -> lock test -> Rayleigh-Ritz with the
//   repair ladders (b2l_rayleigh_ritz) -> upload of the coefficients ->
//   launch of the next F1 (b2l_lobpcg_step) and stencil pass
//   (b2l_stencil7_gram).
// Same decisions, same order as the Python driver (paper_0705_2626_b200/
// lobpcg.py, LOBPCGRun.step); the Python side keeps every other path (first
// iteration, drift repair, callbacks, constraints) and records the history
// from the outputs.  A z-slab rank (s->slab with a communicator) runs the same
// step with NCCL inside: halo under the interior stencil planes, one
// all-reduce per fused pass (slab.cu).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "../../include/b200lobpcg.h"
#include "common.cuh"

namespace b2l {
int rr_begin_tls(int m, int kst, int have_p, const double* g1, int ldg1, const int* jact, int kj,
                 const int* sel, double pivot_floor, int* fallbacks_out);
int rr_finish_tls(const double* g2, const double* lam, double* lam_out, double* coef_out,
                  int* pcols_out, int* kp_out, int* fallbacks_out);
void rr_set_align(double abs_gap);
int lobpcg_step(int nrows, int m, const double* x, const double* ax, int ldx, const double* w,
                const double* aw, int ldw, int kw, const double* p, const double* ap, int kp,
                const int* pcols, const double* coef, double* xo, double* axo, double* po,
                double* apo, const double* lam, const double* d, int tmode, double tinv,
                const double* tvec, const int* wpos, int kwn, double* wo, int ldwn, int want_ax,
                double* red_out, cudaStream_t st, const StepHostCoef* hc,
                StepDeferred* defer, int x_plus_p = 1);
int stencil7_gram(const double* in, double* out, int nx, int ny, int nz, int ld,
                  const double* halo, int has_lo, int has_hi, double scale, const double* x,
                  int ldx, int m, int kw, double* gram_out, cudaStream_t st);
// z-slab context (slab.cu)
bool slab_multi(const b2l_slab* s);
cudaStream_t slab_comm_stream(b2l_slab* s);
cudaEvent_t slab_event(b2l_slab* s, int which);   // 0 f1, 1 red, 2 sg, 3 g2
int slab_halo_start(b2l_slab* s, const double* in, int ld, cudaStream_t st);
int slab_sgram_after_halo(b2l_slab* s, const double* in, double* out, int ld, double scale,
                          const double* x, int ldx, int m, int kw, double* gram_out,
                          cudaStream_t st);
int slab_allreduce(b2l_slab* s, double* buf, size_t count, cudaStream_t st);
int repair_coef(int m, const double* gxx, const double* gxa, double* lam_out, double* m_out);
struct HostBlock {
  const double* p;
  int ld, cols;
};
int gram(int nrows, const HostBlock* L, int nl, const HostBlock* R, int nr, unsigned rw_mask,
         const double* d, const unsigned char* pair_mode, double* out, cudaStream_t st);
}  // namespace b2l

using namespace b2l;

namespace {
inline int even(int k) { return k < 2 ? 2 : k + (k & 1); }

// Host-side phase timer of b2l_fast_iteration (B2L_ITER_PROFILE=1):
// [0] calls, [1] enqueue of the fetch, [2] wait in the synchronisation,
// [3] drift + lock tests, [4] Rayleigh-Ritz second half (after G2 landed),
// [5] uploads + launches, [6] Rayleigh-Ritz first half, [7] wait for G2 (us).
double g_prof[8];
const bool g_prof_on = [] {
  const char* v = getenv("B2L_ITER_PROFILE");
  return v && v[0] == '1';
}();
inline double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

// A non-blocking side stream + fork/join events per device (lazily created;
// null if creation fails, then everything stays on the caller's stream).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  const void* owner = nullptr;   // the iteration state whose F1 `join` marks
  bool tried = false;
};
SideStream* side_stream() {
  static SideStream g[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  SideStream& x = g[dev & 63];
  if (!x.tried) {
    x.tried = true;
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x.s = nullptr;
    }
  }
  return x.s ? &x : nullptr;
}

// Device address of a pinned host buffer (cudaHostGetDevicePointer), cached
// for the last two buffers; null when it is not device-mapped (then copied).
double* mapped(double* h) {
  static double* hs[2] = {nullptr, nullptr};
  static double* ds[2] = {nullptr, nullptr};
  for (int i = 0; i < 2; ++i)
    if (hs[i] == h) return ds[i];
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) {
    cudaGetLastError();
    d = nullptr;
  }
  hs[1] = hs[0];
  ds[1] = ds[0];
  hs[0] = h;
  ds[0] = static_cast<double*>(d);
  return ds[0];
}

extern "C" int b2l_iter_profile(double* out, int reset) {
  if (out)
    for (int i = 0; i < 8; ++i) out[i] = g_prof[i];
  if (reset)
    for (int i = 0; i < 8; ++i) g_prof[i] = 0.0;
  return g_prof_on ? 1 : 0;
}

// Drift repair on the device state (_refresh_ritz, lobpcg.py:280-296, at the
// top of the iteration, lobpcg.py:419-428), without leaving the native loop:
// X^T A X by one Gram pass (X^T B X is F1's), the folded rotation
// M = R_eff^-1 Q on the host (repair_coef), then ONE F1 pass in its
// no-update form -- X'' = X M, AX'' = AX M (x_plus_p = 0), P and AP carried
// through (Cp = I), the residual W'' with the repaired Ritz values, its
// norms and the Grams -- and the stencil pass on W''.  On return h_red /
// h_g2 hold the repaired iteration's reductions (the main stream is
// synchronised), s->lam the repaired Ritz values, and the state's block
// pointers are swapped to the repaired blocks.  B2L_ITER_DRIFT: X^T B X is
// not SPD, the caller's path reports the failure.
static int native_repair(b2l_iter_state* s, b2l_slab* S, bool multi, cudaStream_t st) {
  const int m = s->m, kst = s->kst;
  const int b = 3 * m + kst;
  if (!s->have_p) return B2L_ITER_DRIFT;
  std::vector<double> gxx((size_t)m * m), gxa((size_t)m * m), M((size_t)m * m), lam(m);
  const double* G1 = s->h_red + 2 * m;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) gxx[(size_t)i * m + j] = G1[(size_t)i * b + j];
  // X^T A X (upper), into the reduction scratch, summed over the slab ranks
  const HostBlock L[1] = {{s->x, s->ldx, m}};
  const HostBlock R[1] = {{s->ax, s->ldx, m}};
  const unsigned char upper = 2;
  if (int r = gram(s->n, L, 1, R, 1, 0u, nullptr, &upper, s->red_dev, st)) return r;
  if (multi)
    if (int r = slab_allreduce(S, s->red_dev, (size_t)m * m, st)) return r;
  B2L_CUDA(cudaMemcpyAsync(gxa.data(), s->red_dev, (size_t)m * m * sizeof(double),
                           cudaMemcpyDeviceToHost, st));
  B2L_CUDA(cudaStreamSynchronize(st));
  const int rc = repair_coef(m, gxx.data(), gxa.data(), lam.data(), M.data());
  if (rc == 1) return B2L_ITER_DRIFT;
  if (rc) return rc;
  for (int j = 0; j < m; ++j) s->lam[j] = lam[j];
  // coefficients by value: [Cx = M | Cw = 0 | Cp = I].  P also fills the W
  // slot (Cw = 0): the pass then has the shape of a full-block step, whose
  // compile-time kernel is ~25% faster than the general one, for one extra
  // read of P and AP
  std::vector<double> coef((size_t)3 * m * m, 0.0);
  for (size_t i = 0; i < (size_t)m * m; ++i) coef[i] = M[i];
  for (int i = 0; i < m; ++i) coef[(size_t)2 * m * m + (size_t)i * m + i] = 1.0;
  std::vector<int> pcols(m), wpos(m, -1);
  for (int j = 0; j < m; ++j) pcols[j] = j;
  for (int j = 0, q = 0; j < m; ++j)
    if (s->active[j]) wpos[j] = q++;
  const StepHostCoef hc{coef.data(), lam.data(), pcols.data(), wpos.data()};
  const size_t nred = (size_t)2 * m + (size_t)(2 * m + kst) * b;
  const size_t ng2 = (size_t)(m + kst) * kst;
  double* red_h = multi ? nullptr : mapped(s->h_red);
  double* g2_h = multi ? nullptr : mapped(s->h_g2);
  int r = lobpcg_step(s->n, m, s->x, s->ax, s->ldx, s->p, s->ap, s->ldx, m, s->p, s->ap, m,
                      nullptr, nullptr, s->x2, s->ax2, s->p2, s->ap2, nullptr, s->bdiag, s->tmode,
                      s->tinv, s->tvec, nullptr, kst, s->w_next, even(kst), s->relative_tol,
                      red_h ? red_h : s->red_dev, st, &hc, nullptr, /*x_plus_p=*/0);
  if (r) return r;
  if (multi) {
    if ((r = slab_halo_start(S, s->w_next, even(kst), st))) return r;
    if ((r = slab_sgram_after_halo(S, s->w_next, s->aw, even(kst), s->scale, s->x2, s->ldx, m,
                                   kst, s->g2_dev, st)))
      return r;
    if ((r = slab_allreduce(S, s->red_dev, nred, st))) return r;
    if ((r = slab_allreduce(S, s->g2_dev, ng2, st))) return r;
  } else {
    r = stencil7_gram(s->w_next, s->aw, s->nx, s->ny, s->nz, even(kst), nullptr, 0, 0, s->scale,
                      s->x2, s->ldx, m, kst, g2_h ? g2_h : s->g2_dev, st);
    if (r) return r;
  }
  if (!red_h)
    B2L_CUDA(cudaMemcpyAsync(s->h_red, s->red_dev, nred * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
  if (!g2_h)
    B2L_CUDA(cudaMemcpyAsync(s->h_g2, s->g2_dev, ng2 * sizeof(double), cudaMemcpyDeviceToHost,
                             st));
  B2L_CUDA(cudaStreamSynchronize(st));
  std::swap(s->x, s->x2);
  std::swap(s->ax, s->ax2);
  std::swap(s->p, s->p2);
  std::swap(s->ap, s->ap2);
  std::swap(s->w_cur, s->w_next);
  return 0;
}

extern "C" int b2l_fast_iteration(b2l_iter_state* s) {
  if (!s || s->m < 1 || s->kst < 1 || s->kst > s->m)
    return fail(-B2L_EINVAL, "fast_iteration: bad state");
  const int m = s->m, kst = s->kst;
  cudaStream_t st = (cudaStream_t)s->stream;
  const int a = 2 * m + kst, b = 3 * m + kst;
  const size_t nred = (size_t)2 * m + (size_t)a * b;
  const size_t ng2 = (size_t)(m + kst) * kst;

  double t0 = g_prof_on ? now_us() : 0.0, t1 = 0.0;
  auto mark = [&](int slot) {
    if (!g_prof_on) return;
    t1 = now_us();
    g_prof[slot] += t1 - t0;
    t0 = t1;
  };
  if (g_prof_on) g_prof[0] += 1.0;
  b2l_slab* S = s->slab;
  const bool multi = slab_multi(S);
  // ---- one synchronisation: F1's reductions + the stencil pass's Gram.  The
  // passes this function queued wrote them straight into the pinned h_red /
  // h_g2 (device-mapped; a z-slab step: reduced over the ranks and copied on
  // the communication stream); passes queued elsewhere left them on the
  // device, unreduced.
  if (!s->red_on_host) {
    if (multi) {
      if (int r = slab_allreduce(S, s->red_dev, nred, st)) return r;
      if (int r = slab_allreduce(S, s->g2_dev, ng2, st)) return r;
    }
    B2L_CUDA(cudaMemcpyAsync(s->h_red, s->red_dev, nred * sizeof(double), cudaMemcpyDeviceToHost,
                             st));
    B2L_CUDA(cudaMemcpyAsync(s->h_g2, s->g2_dev, ng2 * sizeof(double), cudaMemcpyDeviceToHost,
                             st));
  }
  mark(1);
  // red_on_host == 2: F1's reductions went through the side stream into the
  // mapped h_red -- wait only for them (the stencil pass, which produces A W
  // and h_g2, may still run) and do the G1-only half of the Rayleigh-Ritz
  // step meanwhile; the main stream is synchronised before the G2 half.
  SideStream* side0 = side_stream();
  const bool early_slab = s->red_on_host == 3 && multi;
  const bool early =
      early_slab || (s->red_on_host == 2 && side0 != nullptr && side0->owner == s);
  if (early_slab) {
    B2L_CUDA(cudaEventSynchronize(slab_event(S, 1)));
  } else if (early) {
    B2L_CUDA(cudaEventSynchronize(side0->join));
  } else {
    B2L_CUDA(cudaStreamSynchronize(st));
  }
  s->red_on_host = 0;
  bool main_synced = !early;
  auto sync_main = [&]() -> int {
    if (!main_synced) {
      B2L_CUDA(cudaStreamSynchronize(st));
      main_synced = true;
    }
    return 0;
  };
  mark(2);
  const double* sums = s->h_red;
  const double* G1 = s->h_red + 2 * m;

  // ---- drift (lobpcg.py:419-428): max |X^T B X - I| over the upper triangle
  double drift = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) {
      const double v = std::fabs(G1[(size_t)i * b + j] - (i == j ? 1.0 : 0.0));
      if (!(v <= drift)) drift = v;   // NaN-propagating max
    }
  s->drift = drift;
  s->repaired = 0;
  if (!(drift <= s->drift_limit)) {
    if (int r = sync_main()) return r;   // the caller reads h_g2 too
    static const bool python_repair = [] {
      const char* v = getenv("B2L_NATIVE_REPAIR");
      return v && v[0] == '0';
    }();
    if (python_repair) return B2L_ITER_DRIFT;
    const int r = native_repair(s, S, multi, st);
    if (r) return r;   // B2L_ITER_DRIFT: the caller's repair path
    s->repaired = 1;   // h_red / h_g2 and the block pointers are the repaired ones
  }

  // ---- lock test (lobpcg.py:429-437)
  std::vector<int> jprev, jact;
  for (int j = 0; j < m; ++j)
    if (s->active[j]) jprev.push_back(j);
  if ((int)jprev.size() != kst) {
    sync_main();
    return fail(-B2L_EINVAL, "fast_iteration: kst != |active|");
  }
  double thr_min = INFINITY;
  for (int j = 0; j < m; ++j) {
    const double nrm = std::sqrt(sums[j]);
    const double thr = s->relative_tol ? s->tol * std::sqrt(sums[m + j]) : s->tol;
    if (thr < thr_min) thr_min = thr;
    s->norms[j] = nrm;
    const bool lock = s->active[j] && nrm < thr;
    s->newly[j] = lock ? 1 : 0;
    if (lock) {
      s->lock_iteration[j] = s->it;
      s->active[j] = 0;
    }
  }
  for (int j = 0; j < m; ++j)
    if (s->active[j]) jact.push_back(j);
  if (jact.empty() || s->it == s->max_iter) {
    if (int r = sync_main()) return r;
    return B2L_ITER_DONE;
  }

  mark(3);
  // ---- Rayleigh-Ritz (lobpcg.py:475-519) on the fetched Grams
  const int kj = (int)jact.size();
  std::vector<int> sel(kj);
  for (int q = 0, t = 0; q < kj; ++q) {
    while (jprev[t] != jact[q]) ++t;
    sel[q] = t;
  }
  double* coef = s->h_stage;                        // [Cx | Cw | Cp]
  double* lam_next = s->h_stage + (size_t)3 * m * m;
  int* pcols = s->h_istage;
  int* wpos = s->h_istage + m;
  int kp = 0, fb = 0;
  // eigenvalue gaps below a tenth of the smallest lock threshold count as one
  // cluster in the eigensolve (rr.cu: align_clusters; wider gaps keep the
  // Rayleigh-Ritz step from separating a cluster's unconverged direction from
  // its locked columns); the Python driver sets the same value
  rr_set_align(0.1 * thr_min);
  int rc = rr_begin_tls(m, kst, s->have_p, G1, b, jact.data(), kj, sel.data(), s->pivot_floor,
                        &fb);
  mark(6);
  if (int r = sync_main()) return r;   // G2 = [X ; W]^T A W has landed
  mark(7);
  if (!rc) rc = rr_finish_tls(s->h_g2, s->lam, lam_next, coef, pcols, &kp, &fb);
  s->fallbacks = fb;
  mark(4);
  if (rc) return rc;
  for (int j = 0; j < m; ++j) {
    wpos[j] = -1;
    s->lam_next[j] = lam_next[j];
  }
  for (int q = 0; q < kj; ++q) wpos[jact[q]] = q;
  s->kp = kp;
  s->k_next = kj;

  if (multi) {
    // ---- z-slab: F1 (row-local), then on the communication stream the halo
    // of W' (under the interior stencil planes), F1's second reduction stage,
    // its all-reduce and D2H (the host starts the G1 half on it); the stencil
    // pass's Gram is all-reduced and copied behind the edge planes.
    const size_t nred_n = (size_t)2 * m + (size_t)(2 * m + kj) * (3 * m + kj);
    const size_t ng2_n = (size_t)(m + kj) * kj;
    cudaStream_t cs = slab_comm_stream(S);
    const StepHostCoef hc_m{coef, lam_next, pcols, wpos};
    StepDeferred dfr;
    int r = lobpcg_step(s->n, m, s->x, s->ax, s->ldx, s->w_cur, s->aw, even(kst), kst,
                        kp ? s->p : nullptr, kp ? s->ap : nullptr, kp, nullptr, nullptr,
                        s->x2, s->ax2, s->p2, s->ap2, nullptr, s->bdiag, s->tmode, s->tinv,
                        s->tvec, nullptr, kj, s->w_next, even(kj), s->relative_tol,
                        s->red_dev, st, &hc_m, &dfr);
    if (r) return r;
    if ((r = slab_halo_start(S, s->w_next, even(kj), st))) return r;   // cs waits for F1
    if ((r = sum_parts(dfr.part, dfr.nparts, dfr.len, dfr.out, cs))) return r;
    if ((r = slab_allreduce(S, s->red_dev, nred_n, cs))) return r;
    B2L_CUDA(cudaMemcpyAsync(s->h_red, s->red_dev, nred_n * sizeof(double),
                             cudaMemcpyDeviceToHost, cs));
    B2L_CUDA(cudaEventRecord(slab_event(S, 1), cs));
    if ((r = slab_sgram_after_halo(S, s->w_next, s->aw, even(kj), s->scale, s->x2, s->ldx, m,
                                   kj, s->g2_dev, st)))
      return r;
    B2L_CUDA(cudaEventRecord(slab_event(S, 2), st));
    B2L_CUDA(cudaStreamWaitEvent(cs, slab_event(S, 2), 0));
    if ((r = slab_allreduce(S, s->g2_dev, ng2_n, cs))) return r;
    B2L_CUDA(cudaMemcpyAsync(s->h_g2, s->g2_dev, ng2_n * sizeof(double),
                             cudaMemcpyDeviceToHost, cs));
    B2L_CUDA(cudaEventRecord(slab_event(S, 3), cs));
    B2L_CUDA(cudaStreamWaitEvent(st, slab_event(S, 3), 0));
    s->red_on_host = 3;
    mark(5);
    return B2L_ITER_OK;
  }
  // ---- the next fused passes: coefficients by value in the F1 launch (no
  // H2D copies), reductions written into the mapped pinned buffers (no D2H)
  double* red_h = mapped(s->h_red);
  double* g2_h = mapped(s->h_g2);
  const StepHostCoef hc{coef, lam_next, pcols, wpos};
  // F1's second reduction stage runs on a side stream beside the stencil
  // pass (it only feeds the host); the main stream joins it before the next
  // synchronisation
  StepDeferred dfr;
  SideStream* side = side_stream();
  int r = lobpcg_step(s->n, m, s->x, s->ax, s->ldx, s->w_cur, s->aw, even(kst), kst,
                      kp ? s->p : nullptr, kp ? s->ap : nullptr, kp, nullptr, nullptr,
                      s->x2, s->ax2, s->p2, s->ap2, nullptr, s->bdiag, s->tmode, s->tinv,
                      s->tvec, nullptr, kj, s->w_next, even(kj), s->relative_tol,
                      red_h ? red_h : s->red_dev, st, &hc, side ? &dfr : nullptr);
  if (r) return r;
  if (side) {
    B2L_CUDA(cudaEventRecord(side->fork, st));
    B2L_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
    r = sum_parts(dfr.part, dfr.nparts, dfr.len, dfr.out, side->s);
    if (r) return r;
    B2L_CUDA(cudaEventRecord(side->join, side->s));
    side->owner = s;
  }
  r = stencil7_gram(s->w_next, s->aw, s->nx, s->ny, s->nz, even(kj), nullptr, 0, 0, s->scale,
                    s->x2, s->ldx, m, kj, g2_h ? g2_h : s->g2_dev, st);
  if (r) return r;
  if (side) B2L_CUDA(cudaStreamWaitEvent(st, side->join, 0));
  // the next call skips its D2H copies only when both landed on the host
  if (red_h && !g2_h)
    B2L_CUDA(cudaMemcpyAsync(s->h_g2, s->g2_dev, (size_t)(m + kj) * kj * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
  if (!red_h && g2_h)
    B2L_CUDA(cudaMemcpyAsync(s->h_red, s->red_dev,
                             (2 * (size_t)m + (size_t)(2 * m + kj) * (3 * m + kj)) * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
  // 2: both reductions land in mapped memory, F1's through the side stream
  // (the next call may then start on G1 before the stencil pass is done)
  s->red_on_host = (red_h && g2_h && side) ? 2 : ((red_h || g2_h) ? 1 : 0);
  mark(5);
  return B2L_ITER_OK;
}

extern "C" int b2l_iter_state_size(void) { return (int)sizeof(b2l_iter_state); }
