// TMA streaming microbenchmark for F1's data path at m = 10 (80-byte rows):
// 148 persistent CTAs, one producer thread filling a ring of stages with six
// input boxes per chunk of 56 rows, one consumer thread that (optionally)
// stores five of them back out and releases the stage.  No math: this is the
// ceiling of the pass's load / store skeleton for each box geometry.
//
//   mode 0: 2-D map of a (rows x 10) block, box 12 x 56 (96-byte shared rows,
//           two out-of-bounds columns per row)          -- what F1 uses
//   mode 1: 2-D map, box 10 x 56 (dense 80-byte shared rows)
//   mode 2: 1-D bulk copies of 4480 bytes (a chunk of an unpadded block is
//           contiguous)
//   mode 3: 2-D map of the same bytes as (bytes / 128) lines of 16 doubles,
//           box 16 x 35
//   mode 4: 1-D bulk copies, one per 8-row tile (640 bytes each)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_stream_bench
//      tools/tma_stream_bench.cu -lcuda ;  tools/tma_stream_bench [N=128]
// Diagnostic only (not part of the library).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s: %s\n", #x, cudaGetErrorString(e_));                              \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(s32(b)), "r"(ph)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_ld2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                        int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3}], [%4];" ::"r"(s32(dst)),
      "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_st2(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::
                   "l"((uint64_t)m),
               "r"(s32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_ld(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_st(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(s32(src)), "r"(bytes)
               : "memory");
}

struct Maps {
  CUtensorMap in[6], out[5];
};
struct Args {
  const double* in[6];
  double* out[5];
  int nchunks, mode, nst, nstore, box_bytes, rc;   // box_bytes: shared bytes of one box
};

constexpr int M = 10;
__constant__ int RC_d;

__global__ void __launch_bounds__(64)
    stream_kernel(const __grid_constant__ Maps mp, const __grid_constant__ Args A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[8], empty[8];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < A.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int stage_bytes = 6 * A.box_bytes;
  const int nloc =
      blockIdx.x < A.nchunks ? (A.nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int RC = A.rc;
  const uint32_t tx = (A.mode == 0 ? 6u * 12 * RC * 8 : 6u * RC * M * 8);
  if (tid == 0) {
    for (int j = 0; j < nloc; ++j) {
      const int s = j % A.nst;
      if (j >= A.nst) mbar_wait(&empty[s], (j / A.nst - 1) & 1);
      const int c = blockIdx.x + j * gridDim.x;
      unsigned char* st = smem + (size_t)s * stage_bytes;
      mbar_expect(&full[s], tx);
      for (int b = 0; b < 6; ++b) {
        unsigned char* dst = st + (size_t)b * A.box_bytes;
        if (A.mode == 0 || A.mode == 1) tma_ld2(dst, &mp.in[b], &full[s], 0, c * RC);
        else if (A.mode == 2) bulk_ld(dst, A.in[b] + (size_t)c * RC * M, RC * M * 8, &full[s]);
        else if (A.mode == 3) tma_ld2(dst, &mp.in[b], &full[s], 0, c * (RC * 5 / 8));
        else
          for (int t = 0; t < RC / 8; ++t)
            bulk_ld(dst + t * 640, A.in[b] + (size_t)c * RC * M + t * 80, 640, &full[s]);
      }
    }
  } else if (tid == 32) {
    for (int j = 0; j < nloc; ++j) {
      const int s = j % A.nst;
      mbar_wait(&full[s], (j / A.nst) & 1);
      const int c = blockIdx.x + j * gridDim.x;
      unsigned char* st = smem + (size_t)s * stage_bytes;
      if (A.nstore) {
        for (int b = 0; b < A.nstore; ++b) {
          unsigned char* src = st + (size_t)b * A.box_bytes;
          if (A.mode == 0 || A.mode == 1) tma_st2(&mp.out[b], src, 0, c * RC);
          else if (A.mode == 2) bulk_st(A.out[b] + (size_t)c * RC * M, src, RC * M * 8);
          else if (A.mode == 3) tma_st2(&mp.out[b], src, 0, c * (RC * 5 / 8));
          else
            for (int t = 0; t < RC / 8; ++t)
              bulk_st(A.out[b] + (size_t)c * RC * M + t * 80, src + t * 640, 640);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      mbar_arrive(&empty[s]);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 128;
  const size_t n = (size_t)N * N * N;
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr));
  double* in[6];
  double* out[5];
  for (auto& p : in) {
    CK(cudaMalloc(&p, n * M * 8));
    CK(cudaMemset(p, 0, n * M * 8));
  }
  for (auto& p : out) CK(cudaMalloc(&p, n * M * 8));
  auto mk = [&](CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 8};
    cuuint32_t box[2] = {bc, br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      exit(1);
    }
  };
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const char* names[5] = {"2-D box 12xRC of 10 cols (F1 today)", "2-D box 10xRC (dense)",
                          "1-D bulk", "2-D 128-B lines", "1-D bulk per 8-row tile"};
  struct Cfg { int mode, rc, nst, per_sm; };
  const Cfg cfgs[] = {{0, 56, 4, 1}, {2, 56, 4, 1}, {0, 56, 2, 2}, {2, 56, 2, 2}, {2, 56, 3, 2},
                      {0, 112, 2, 1}, {2, 112, 2, 1}, {2, 112, 3, 1}, {2, 224, 2, 1}, {0, 32, 6, 1},
                      {2, 32, 6, 1}, {2, 32, 3, 2}, {2, 24, 4, 2}, {2, 16, 6, 2}, {2, 56, 1, 3},
                      {2, 56, 1, 4}, {0, 56, 1, 4}};
  for (const Cfg& cf : cfgs) {
    const int mode = cf.mode, RC = cf.rc;
    const int nchunks = (int)(n / RC);
    Maps mp;
    Args A;
    for (int b = 0; b < 6; ++b) A.in[b] = in[b];
    for (int b = 0; b < 5; ++b) A.out[b] = out[b];
    for (int b = 0; b < 11; ++b) {
      CUtensorMap* m = b < 6 ? &mp.in[b] : &mp.out[b - 6];
      void* base = b < 6 ? (void*)in[b] : (void*)out[b - 6];
      if (mode == 0) mk(m, base, M, n, 12, RC);
      else if (mode == 3) mk(m, base, 16, n * M / 16, 16, RC * 5 / 8);
      else mk(m, base, M, n, 10, RC);
    }
    A.nchunks = nchunks;
    A.mode = mode;
    A.rc = RC;
    A.box_bytes = mode == 0 ? 12 * RC * 8 : ((RC * M * 8 + 127) & ~127);
    A.nst = cf.nst;
    for (int nstore : {0, 5}) {
      A.nstore = nstore;
      const size_t smem = (size_t)cf.nst * 6 * A.box_bytes;
      if (smem * cf.per_sm > 220 * 1024) continue;
      std::vector<float> ts;
      for (int it = 0; it < 12; ++it) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        stream_kernel<<<148 * cf.per_sm, 64, smem>>>(mp, A);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (it >= 2) ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      const double ms = ts[ts.size() / 2];
      const double bytes = (double)nchunks * RC * M * 8 * (6 + nstore);
      printf("mode %d (%s) rows %d stages %d CTAs/SM %d stores %d: %.4f ms  %.0f GB/s\n", mode,
             names[mode], RC, cf.nst, cf.per_sm, nstore, ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
