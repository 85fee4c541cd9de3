// Shared device/host helpers for libb200lobpcg (sm_100a only).
//
// mbarrier + TMA (cp.async.bulk / cp.async.bulk.tensor) wrappers written as
// inline PTX, error plumbing for the C ABI, and the per-device workspace.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libb200lobpcg targets sm_100a only"
#endif

namespace b2l {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define B2L_CUDA(expr)                                                     \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess)                                                 \
      return ::b2l::fail(-(int)_e, std::string(#expr) + ": " +             \
                                       cudaGetErrorString(_e));            \
  } while (0)

#define B2L_CHECK(cond, code, msg)                                         \
  do {                                                                     \
    if (!(cond)) return ::b2l::fail((code), (msg));                        \
  } while (0)

enum : int {
  B2L_OK = 0,
  B2L_EINVAL = 1000,   // returned negated
  B2L_ENOMEM = 1001,
  B2L_EDRIVER = 1002,
  B2L_EDEGENERATE = 1003,   // Rayleigh-Ritz basis repair exhausted
  B2L_ELAPACK = 1004,
  B2L_ENCCL = 1005,         // NCCL unavailable or a collective failed
};

// ------------------------------------------------------------- workspace
// One growable device scratch buffer per device (CTA partials of the
// deterministic two-stage reductions).  Stream-ordered: the library is
// driven by one host thread / one stream per device.
// slot 1 holds F1's partials while the stencil pass (slot 0) runs beside their
// reduction (b2l_fast_iteration)
void* workspace(size_t bytes, int* err, int slot = 0);
// F1's second reduction stage, left to the caller when requested
struct StepDeferred {
  const double* part = nullptr;
  int nparts = 0, len = 0;
  double* out = nullptr;
};
int sm_count();
// cudaFuncSetAttribute(max dynamic smem) + occupancy query, cached per
// (kernel, smem, threads): both are host API round trips on every launch
// otherwise.  per_sm may be null.
int prepare_kernel(const void* kern, size_t smem, int threads, int* per_sm);
// every kernel launch of the library is counted (b2l_launch_count)
void count_launch();
// Host-side Rayleigh-Ritz output handed to the F1 launch by value (no H2D copy)
struct StepHostCoef {
  const double* coef;   // [Cx m*m | Cw kw*m | Cp kp*m]
  const double* lam;    // m
  const int* pcols;     // kp
  const int* wpos;      // m
};
// out[e] = sum over parts c of partial[c * len + e] (fixed order, deterministic)
int sum_parts(const double* partial, int nparts, int len, double* out, cudaStream_t st);

// ------------------------------------------------------------ tensor maps
int encode_tmap_4d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1,
                   uint64_t d2, uint64_t d3, uint32_t b0, uint32_t b1,
                   uint32_t b2, uint32_t b3);

// ------------------------------------------------------------ device PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Waiting variant for warps that idle a long time (warp-specialised kernels):
// the thread is suspended in hardware until the phase completes (or the time
// hint, in ns, expires) instead of re-polling, so it does not steal issue
// slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}

// TMA tiled 4-D load global -> shared, completion on an mbarrier.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map,
                                            uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// TMA tiled 4-D store shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map,
                                             const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, "
      "%3, %4, %5}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// TMA tiled 2-D load / store (a box of rows of a row-major block).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}

// Shared-memory row stride (doubles) for a block of `ld` doubles per row:
// >= ld and == 4 or 12 (mod 16), so the DMMA fragment patterns (4 rows x 4
// doubles per half-warp) hit 16 distinct bank pairs.  The TMA box is this
// wide; the columns past `ld` are out of bounds, zero-filled on load and
// clipped on store.
__host__ __device__ constexpr inline int smem_stride(int ld) {
  int s = ld < 4 ? 4 : ld;
  while ((s & 15) != 4 && (s & 15) != 12) ++s;
  return s;
}

int encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                   uint32_t box_cols, uint32_t box_rows);

// 1-D bulk copy global -> shared (16-B aligned, size multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src,
                                          uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
      "[%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Ampere-style 16-B async copy (LDGSTS), used by the row-chunk kernels.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace b2l
