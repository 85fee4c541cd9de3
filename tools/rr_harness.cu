// Standalone host harness: phase times of b2l_rayleigh_ritz (rr.cu compiled
// with B2L_RR_PROF) on Gram data dumped by tools/bench_rr.py --dump.
// Diagnostic only: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -Xcompiler -O2 -std=c++17 --expt-relaxed-constexpr -DB2L_RR_PROF
//   -o rr_harness tools/rr_harness.cu
#include <chrono>
#include <dlfcn.h>
#include <cstdio>
#include <string>
#include <vector>
static double g_t[16], g_last;
static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void rr_mark(int k) {
  const double t = now_us();
  if (k >= 0) g_t[k] += t - g_last;
  g_last = t;
}
#include "../paper_0705_2626_b200/csrc/rr.cu"
namespace b2l {
int fail(int c, const std::string&) { return c; }
}
int main(int argc, char** argv) {
  // optional: B2L_HARNESS_BLAS=<libscipy_openblas.so> registers its LAPACK /
  // BLAS as the library does from scipy (cython_lapack / cython_blas)
  if (const char* lib = getenv("B2L_HARNESS_BLAS")) {
    void* h = dlopen(lib, RTLD_NOW);
    auto sym = [&](const char* a, const char* b) {
      void* f = h ? dlsym(h, a) : nullptr;
      return f ? f : (h ? dlsym(h, b) : nullptr);
    };
    if (h) {
      b2l_set_lapack(sym("scipy_dpotrf_", "dpotrf_"), sym("scipy_dtrtrs_", "dtrtrs_"),
                     sym("scipy_dtrtri_", "dtrtri_"), sym("scipy_dsyevr_", "dsyevr_"));
      b2l_set_blas(sym("scipy_dgemm_", "dgemm_"));
      b2l_set_lapack_mrrr(sym("scipy_dsytrd_", "dsytrd_"), sym("scipy_dstemr_", "dstemr_"),
                          sym("scipy_dormtr_", "dormtr_"));
    }
  }
  for (int a = 1; a < argc; ++a) {
    FILE* f = fopen(argv[a], "rb");
    long long hd[5];
    if (!f || fread(hd, 8, 5, f) != 5) return 1;
    const int m = (int)hd[0];
    std::vector<double> g1(hd[1] * hd[2]), g2(hd[3] * hd[4]), lam(m);
    if (fread(g1.data(), 8, g1.size(), f) != g1.size() ||
        fread(g2.data(), 8, g2.size(), f) != g2.size() || fread(lam.data(), 8, m, f) != (size_t)m)
      return 1;
    fclose(f);
    std::vector<int> j(m);
    for (int i = 0; i < m; ++i) j[i] = i;
    std::vector<double> lo(m), coef(3 * m * m);
    std::vector<int> pc(2 * m);
    int kp, fb;
    const int reps = m >= 32 ? 50 : 5000;
    for (int r = 0; r < 200; ++r)
      b2l_rayleigh_ritz(m, m, 1, g1.data(), (int)hd[2], g2.data(), lam.data(), j.data(), m,
                        j.data(), 1e-8, lo.data(), coef.data(), pc.data(), &kp, &fb);
    for (double& t : g_t) t = 0.0;
    const double t0 = now_us();
    for (int r = 0; r < reps; ++r)
      b2l_rayleigh_ritz(m, m, 1, g1.data(), (int)hd[2], g2.data(), lam.data(), j.data(), m,
                        j.data(), 1e-8, lo.data(), coef.data(), pc.data(), &kp, &fb);
    const double tot = (now_us() - t0) / reps;
    printf("m=%d: %.2f us/call | W,P chol-QR %.2f, blocks+pencil %.2f, gen_sym_eig %.2f "
           "[chol %.2f, R^-T A R^-1 %.2f, eig-replay %.2f], fold %.2f | tred %.2f accum %.2f ql %.2f | lam0 %.17g\n",
           m, tot, g_t[0] / reps, g_t[1] / reps, g_t[2] / reps, g_t[4] / reps, g_t[5] / reps,
           g_t[6] / reps, g_t[3] / reps, g_t[7] / reps, g_t[8] / reps, g_t[9] / reps, lo[0]);
  }
  return 0;
}
