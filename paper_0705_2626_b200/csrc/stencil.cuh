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
  int zbeg, zend;  // planes [zbeg, zend) processed by this launch
  int zedge;       // 1: only the slab's edge planes 0 and nz-1 (one CTA row each)
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
  int nob = 3;      // output tiles of the stencil + Gram ring (with nst)
  size_t smem;
  dim3 grid;
};

int plan_stencil(int nx, int ny, int nz, int ld, StencilPlan* p);

// Which planes a launch covers (z-slab overlap): all of them, the
// interior [1, nz-1) that needs no halo, or the two edge planes that do.
enum ZMode { Z_ALL = 0, Z_INTERIOR = 1, Z_EDGE = 2 };
// Sets zbeg/zend/zedge/zchunk and the grid's y extent; false if the mode
// selects no plane (an interior of a slab of <= 2 planes).
bool apply_zmode(StencilGeom& g, dim3& grid, int tiles, int mode, int slots);

// The planes [z0, z1) of this CTA.
__device__ __forceinline__ void stencil_zrange(const StencilGeom& g, int& z0, int& z1) {
  if (g.zedge) {
    z0 = (blockIdx.y == 0) ? 0 : g.nz - 1;
    z1 = z0 + 1;
  } else {
    z0 = g.zbeg + blockIdx.y * g.zchunk;
    z1 = min(g.zend, z0 + g.zchunk);
  }
}
int choose_zchunk(int tiles, int nz, int slots);

// K1+K5b geometry (stencil_gram.cu)
struct SGramGeom {
  int m, ldx, kw;   // X columns / leading dim, W columns used
  int ldxp;         // pitch of the X tile in shared memory (sgram_pitch(ldx))
  int a, b;         // m + kw, kw
  int npts;         // points per tile (TX*TY)
  int ngroups;      // ceil(npts / 8)
  uint32_t x_bytes, x_stride;
  double* partial;  // [grid][a*b]
};

// One planned launch of the stencil + Gram pass over a z-mode's planes
// (tensor maps encoded once).  twopass: ld > 16, K1 then a K5 Gram.
struct SGramPlan {
  StencilPlan p;
  SGramGeom G;
  size_t smem;
  int gpw, twopass, nparts, zmode;
  const double *in, *x, *halo;
  double* out;
  int nx, ny, nz, ld, ldx, has_lo, has_hi;
  double scale;
  CUtensorMap tin, thalo, tout, txm;
};
int sgram_plan(const double* in, double* out, int nx, int ny, int nz, int ld, const double* halo,
               int has_lo, int has_hi, double scale, const double* x, int ldx, int m, int kw,
               int zmode, SGramPlan* P);
int sgram_launch(SGramPlan& P, double* partial, cudaStream_t st);
int sgram_finish(const SGramPlan& P, const double* partial, int nparts, double* gram_out,
                 cudaStream_t st);

}  // namespace b2l
