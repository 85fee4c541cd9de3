// fp64 throughput microbenchmark for the roofline denominators of the
// DMMA-bound kernels (C5's Gram / update at m = 64).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
//   tools/fp64_peaks            # prints one JSON line
//
// Two loops, each with independent accumulator chains per warp so the pipe
// (not latency) is the limit, every SM fully occupied, timed with CUDA
// events after a warm-up launch:
//   dmma  mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.884): 512 flop / warp
//   dfma  fma.rn.f64 (SASS DFMA): 2 flop / thread
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CHAINS = 8;

__global__ void dmma_loop(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
          : "+d"(c[k][0]), "+d"(c[k][1])
          : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[blockIdx.x] = s;   // keep the work alive
}

__global__ void dfma_loop(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k] = k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) c[k] = fma(c[k], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <class F>
static float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();   // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5.f;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int threads = 256, blocks = sms * 4;
  const float tm = time_ms([&] { dmma_loop<<<blocks, threads>>>(out, 1.0); });
  const double warps = (double)blocks * threads / 32;
  const double fl_mma = warps * ITERS * CHAINS * 512.0;
  const float tf = time_ms([&] { dfma_loop<<<blocks, threads>>>(out, 1.0); });
  const double fl_fma = (double)blocks * threads * ITERS * CHAINS * 2.0;
  printf("{\"sms\": %d, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"dmma_ms\": %.3f, "
         "\"dfma_ms\": %.3f, \"err\": \"%s\"}\n",
         sms, fl_mma / (tm * 1e-3) / 1e12, fl_fma / (tf * 1e-3) / 1e12, tm, tf,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
