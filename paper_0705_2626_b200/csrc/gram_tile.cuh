// Warp-level fp64 tensor-core (DMMA, mma.sync m8n8k4) Gram microkernel.
//
// C[8*TI x 8*TJ] += L[rows, cols_i]^T (w .* R[rows, cols_j]) for a warp's
// tile block, reading rows from shared memory.  Used by the standalone Gram
// kernel and by the fused update/stencil kernels on tiles they already hold
// in shared memory.
//
// Fragment layout of mma.sync.aligned.m8n8k4.row.col.f64 (PTX ISA):
//   A (8x4, row):   lane holds A[lane>>2][lane&3]
//   B (4x8, col):   lane holds B[lane&3][lane>>2]
//   C/D (8x8):      lane holds C[lane>>2][2*(lane&3) + {0,1}]
// With A = L^T and B = R over 4 rows r0..r0+3, lane (q = lane&3, c = lane>>2)
// loads L[r0+q][i0+c] and R[r0+q][j0+c]: one double each per DMMA pair.
#pragma once

#include "common.cuh"

namespace b2l {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Per-lane view of one 8-column slab of L or R: the lane's column lives at
// smem offset `off` (doubles, relative to the row-0 base of its block) with
// row stride `str`; `ok` is false for padding columns beyond the matrix (then
// off = str = 0: a valid dummy element, see WarpGram::run).
struct LaneCol {
  int off;
  int str;
  bool ok;
  bool weighted;
};

struct DenseRows {
  __device__ __forceinline__ int operator()(int r) const { return r; }
};

template <int TI, int TJ>
struct WarpGram {
  double acc[TI][TJ][2];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
      for (int j = 0; j < TJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }

  // Accumulate rows [r0, r1) (multiple of 4 apart) of a staged chunk.
  // base: stage base pointer; rowoff(r) maps a logical row to its smem row
  // index (identity for dense chunks); d: staged weights (may be null when no
  // column is weighted); mask bit (i*TJ+j) set => tile needed.
  template <class RowMap>
  __device__ __forceinline__ void run(const double* base, const LaneCol (&a)[TI],
                                      const LaneCol (&b)[TJ], const double* d, int r0,
                                      int r1, unsigned mask, RowMap rowmap) {
    const int q = threadIdx.x & 3;
#pragma unroll 2
    for (int r = r0; r < r1; r += 4) {
      const int rr = rowmap(r + q);
      double av[TI], bv[TJ];
      // branch free: a lane whose column lies beyond the Gram (ok = false)
      // reads the valid element its {off, str} = {0, 0} points at, and its
      // products land only in accumulator rows / columns the caller never
      // writes out; every tile is accumulated (unneeded ones are never read),
      // so no predicated mma (a WARPSYNC per DMMA) is emitted
#pragma unroll
      for (int i = 0; i < TI; ++i) av[i] = base[a[i].off + rr * a[i].str];
      const double w = d ? d[r + q] : 1.0;
#pragma unroll
      for (int j = 0; j < TJ; ++j) {
        const double v = base[b[j].off + rr * b[j].str];
        bv[j] = b[j].weighted ? __dmul_rn(w, v) : v;
      }
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
};

}  // namespace b2l
