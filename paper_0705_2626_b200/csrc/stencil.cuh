// Shared geometry of the z-streaming stencil kernels (stencil.cu,
// stencil_gram.cu).
#pragma once

#include "common.cuh"

namespace b2l {

struct StencilGeom {
  int nx, ny, nz;  // local grid (nz = owned planes)
  int ld;          // doubles per point (row stride), even
  int TX, TY;      // interior tile
  int tiles_x;
  int zchunk;
  int nelem;       // TX*TY*ld
  int has_lo, has_hi;
  double scale;
  uint32_t stage_bytes;  // (TX+2)(TY+2) ld 8
  uint32_t stage_stride; // stage_bytes rounded to 128
  uint32_t out_stride;   // TX TY ld 8 rounded to 128
};

struct StencilPlan {
  StencilGeom g;
  int ept, nst;
  size_t smem;
  dim3 grid;
};

int plan_stencil(int nx, int ny, int nz, int ld, StencilPlan* p);
int choose_zchunk(int tiles, int nz, int slots);

}  // namespace b2l
