// K9: the reference's seeded initial block generated on the device
// (multivec.seeded_random_fill, multivec.py:220-229):
//     Generator(PCG64(seed)).uniform(low, high, (n, m)),  C order,
// i.e. element (i, j) is draw i*m + j of numpy's PCG64 stream, bit for bit.
//
// PCG64 (numpy): 128-bit LCG  S <- a S + c  (c = the stream increment, odd),
// each draw steps first and outputs XSL-RR of the new state; next_double =
// (draw >> 11) * 2^-53; uniform = low + (high - low) * next_double.
// A warp owns 32*per_lane consecutive draws, lane l starting at draw
// base + l and striding by 32 -- a fixed jump (a^32, c_32) per step, so every
// store instruction of the warp is coalesced and a step costs one 128-bit
// multiply-add, as in the sequential generator.
#include "common.cuh"

namespace b2l {
namespace {

using u128 = unsigned __int128;

constexpr u128 kPcgMult =
    ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

struct Jump {
  u128 mult, plus;
};

// (A, C) with S_{k} = A S_0 + C after `delta` steps of S <- a S + c
__host__ __device__ inline Jump lcg_jump(u128 delta, u128 c) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kPcgMult, cur_plus = c;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return {acc_mult, acc_plus};
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct FillArgs {
  double* out;
  long long ld, nrows, m;
  long long first;      // draw index of element (0, 0)
  u128 s0, c;           // state before draw 0 of the stream, increment
  u128 j32_mult, j32_plus;
  double low, scale;
  long long per_warp;   // draws per warp (multiple of 32)
};

__global__ void __launch_bounds__(256) seeded_fill_kernel(const FillArgs A) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long total = A.nrows * A.m;
  const long long d0 = warp * A.per_warp + lane;          // local draw index
  if (warp * A.per_warp >= total) return;
  // state after draw (first + d0): S_{first + d0 + 1}
  const Jump j = lcg_jump((u128)(A.first + d0 + 1), A.c);
  u128 s = j.mult * A.s0 + j.plus;
  const long long d1 = min(total, warp * A.per_warp + A.per_warp);
  for (long long d = d0; d < d1; d += 32) {
    const uint64_t r = xsl_rr(s);
    const double u = (double)(r >> 11) * 0x1.0p-53;
    const long long row = d / A.m, col = d - row * A.m;
    A.out[row * A.ld + col] = __dadd_rn(A.low, __dmul_rn(A.scale, u));
    s = A.j32_mult * s + A.j32_plus;
  }
}

}  // namespace
}  // namespace b2l

using namespace b2l;

extern "C" int b2l_seeded_fill(double* out, int ld, long long nrows, int m, long long first_draw,
                               unsigned long long state_hi, unsigned long long state_lo,
                               unsigned long long inc_hi, unsigned long long inc_lo, double low,
                               double high, void* stream) {
  if (!out || m < 1 || ld < m || nrows < 0 || first_draw < 0)
    return fail(-B2L_EINVAL, "seeded_fill: bad arguments");
  if (nrows == 0) return 0;
  FillArgs A{};
  A.out = out;
  A.ld = ld;
  A.nrows = nrows;
  A.m = m;
  A.first = first_draw;
  A.s0 = ((u128)state_hi << 64) | (u128)state_lo;
  A.c = ((u128)inc_hi << 64) | (u128)inc_lo;
  const Jump j32 = lcg_jump(32, A.c);
  A.j32_mult = j32.mult;
  A.j32_plus = j32.plus;
  A.low = low;
  A.scale = high - low;
  const long long total = nrows * (long long)m;
  // ~4 resident 256-thread CTAs per SM, each warp a contiguous run of draws
  const long long warps = (long long)sm_count() * 4 * 8;
  long long per_warp = (total + warps - 1) / warps;
  per_warp = ((per_warp + 31) / 32) * 32;
  if (per_warp < 32) per_warp = 32;
  A.per_warp = per_warp;
  const long long nw = (total + per_warp - 1) / per_warp;
  const long long blocks = (nw + 7) / 8;
  seeded_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(A);
  count_launch();
  B2L_CUDA(cudaGetLastError());
  return 0;
}
