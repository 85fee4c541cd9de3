// z-slab domain decomposition over GPUs, one process per GPU:
// NCCL over NVLink / NVSwitch for the one-plane halo and the sum of every
// small reduction, with the halo exchange overlapped with the interior
// planes of the stencil pass.
//
// The reference is single-process; the paper ran the same
// decomposition through MPI inside hypre.  Rank r owns
// planes [floor(r N/P), floor((r+1) N/P)): a contiguous row range of every
// point-major block (z varies slowest, operators.py:63-67), so a boundary
// plane is nx*ny*ld contiguous doubles and travels as one ncclSend.
//
// NCCL is bound at run time (dlopen + dlsym) to the library the process
// already uses -- PyTorch's bundled libnccl.so.2 -- so the one communicator
// stack is shared with torch.distributed; nccl.h supplies the types only.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "../../include/b200lobpcg.h"
#include "stencil.cuh"

namespace b2l {

int stencil7(const double* in, double* out, int nx, int ny, int nz, int ld, const double* halo,
             int has_lo, int has_hi, double scale, cudaStream_t st, int zmode = 0);
int stencil7_gram(const double* in, double* out, int nx, int ny, int nz, int ld,
                  const double* halo, int has_lo, int has_hi, double scale, const double* x,
                  int ldx, int m, int kw, double* gram_out, cudaStream_t st);
int stencil7_gram_split(const double* in, double* out, int nx, int ny, int nz, int ld,
                        const double* halo, int has_lo, int has_hi, double scale,
                        const double* x, int ldx, int m, int kw, double* gram_out,
                        cudaStream_t st, double** part_buf, size_t* part_cap,
                        cudaEvent_t before_edges);

namespace {
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

template <class F>
bool bind(F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(g_nccl.handle, name));
  return f != nullptr;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const char* msg = g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?";
  return fail(-B2L_ENCCL, std::string("nccl: ") + what + ": " + msg);
}
}  // namespace

#define B2L_NCCL(expr)                                   \
  do {                                                   \
    ncclResult_t r_ = (expr);                            \
    if (r_ != ncclSuccess) return nccl_fail(r_, #expr);  \
  } while (0)

}  // namespace b2l

using namespace b2l;

struct b2l_slab {
  int world = 1, rank = 0, nx = 0, ny = 0, nz = 0;
  int device = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;           // communication stream
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr, ev_f1 = nullptr, ev_red = nullptr,
              ev_sg = nullptr, ev_g2 = nullptr;
  double* halo = nullptr;              // [lo plane | hi plane], (2 nx ny, ld)
  size_t halo_cap = 0;
  double* part = nullptr;              // CTA partials of the split stencil + Gram
  size_t part_cap = 0;
};

namespace b2l {
// Accessors for iterate.cu (the struct stays private to this file).
cudaStream_t slab_comm_stream(b2l_slab* s) { return s->cs; }
bool slab_multi(const b2l_slab* s) { return s && s->comm; }
cudaEvent_t slab_event(b2l_slab* s, int which) {
  switch (which) {
    case 0: return s->ev_f1;
    case 1: return s->ev_red;
    case 2: return s->ev_sg;
    default: return s->ev_g2;
  }
}

static int grow(double** buf, size_t* cap, size_t doubles) {
  if (*cap >= doubles) return 0;
  if (*buf) B2L_CUDA(cudaFree(*buf));
  *buf = nullptr;
  *cap = 0;
  B2L_CUDA(cudaMalloc(buf, doubles * sizeof(double)));
  B2L_CUDA(cudaMemset(*buf, 0, doubles * sizeof(double)));
  *cap = doubles;
  return 0;
}

// Post the boundary-plane exchange of `in` (ld doubles per point) on the
// communication stream, ordered after everything queued on `st`: send the
// first owned plane down and the last one up, receive the neighbours' planes
// into halo[lo | hi].  ev_halo marks completion.
int slab_halo_start(b2l_slab* s, const double* in, int ld, cudaStream_t st) {
  const size_t plane = (size_t)s->nx * s->ny * ld;
  if (int rc = grow(&s->halo, &s->halo_cap, 2 * plane)) return rc;
  B2L_CUDA(cudaEventRecord(s->ev_in, st));
  B2L_CUDA(cudaStreamWaitEvent(s->cs, s->ev_in, 0));
  const bool lo = s->rank > 0, hi = s->rank < s->world - 1;
  if (!lo && !hi) {   // one rank: nothing to exchange, keep the ordering
    B2L_CUDA(cudaEventRecord(s->ev_halo, s->cs));
    return 0;
  }
  B2L_NCCL(g_nccl.GroupStart());
  if (lo) {
    B2L_NCCL(g_nccl.Send(in, plane, ncclFloat64, s->rank - 1, s->comm, s->cs));
    B2L_NCCL(g_nccl.Recv(s->halo, plane, ncclFloat64, s->rank - 1, s->comm, s->cs));
  }
  if (hi) {
    B2L_NCCL(g_nccl.Send(in + (size_t)(s->nz - 1) * plane, plane, ncclFloat64, s->rank + 1,
                         s->comm, s->cs));
    B2L_NCCL(g_nccl.Recv(s->halo + plane, plane, ncclFloat64, s->rank + 1, s->comm, s->cs));
  }
  B2L_NCCL(g_nccl.GroupEnd());
  B2L_CUDA(cudaEventRecord(s->ev_halo, s->cs));
  return 0;
}

int slab_allreduce(b2l_slab* s, double* buf, size_t count, cudaStream_t st) {
  if (!s->comm || count == 0) return 0;
  B2L_NCCL(g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, s->comm, st));
  return 0;
}

// A W on the slab with [X ; W]^T A W (this rank's part): the interior planes
// run while the halo travels, the two edge planes after it lands.
int slab_stencil7_gram(b2l_slab* s, const double* in, double* out, int ld, double scale,
                       const double* x, int ldx, int m, int kw, double* gram_out,
                       cudaStream_t st) {
  if (!slab_multi(s) || s->world == 1)
    return stencil7_gram(in, out, s->nx, s->ny, s->nz, ld, nullptr, 0, 0, scale, x, ldx, m, kw,
                         gram_out, st);
  if (int rc = slab_halo_start(s, in, ld, st)) return rc;
  return stencil7_gram_split(in, out, s->nx, s->ny, s->nz, ld, s->halo, s->rank > 0,
                             s->rank < s->world - 1, scale, x, ldx, m, kw, gram_out, st,
                             &s->part, &s->part_cap, s->ev_halo);
}

// The compute half of slab_stencil7_gram, for callers that posted the halo
// exchange themselves (b2l_fast_iteration queues reductions in between).
int slab_sgram_after_halo(b2l_slab* s, const double* in, double* out, int ld, double scale,
                          const double* x, int ldx, int m, int kw, double* gram_out,
                          cudaStream_t st) {
  if (s->world == 1)   // no halo: the one-launch pass (same sums as one GPU)
    return stencil7_gram(in, out, s->nx, s->ny, s->nz, ld, nullptr, 0, 0, scale, x, ldx, m, kw,
                         gram_out, st);
  return stencil7_gram_split(in, out, s->nx, s->ny, s->nz, ld, s->halo, s->rank > 0,
                             s->rank < s->world - 1, scale, x, ldx, m, kw, gram_out, st,
                             &s->part, &s->part_cap, s->ev_halo);
}

int slab_stencil7(b2l_slab* s, const double* in, double* out, int ld, double scale,
                  cudaStream_t st) {
  if (!slab_multi(s) || s->world == 1)
    return stencil7(in, out, s->nx, s->ny, s->nz, ld, nullptr, 0, 0, scale, st);
  if (int rc = slab_halo_start(s, in, ld, st)) return rc;
  const int lo = s->rank > 0, hi = s->rank < s->world - 1;
  if (int rc = stencil7(in, out, s->nx, s->ny, s->nz, ld, s->halo, lo, hi, scale, st, Z_INTERIOR))
    return rc;
  B2L_CUDA(cudaStreamWaitEvent(st, s->ev_halo, 0));
  return stencil7(in, out, s->nx, s->ny, s->nz, ld, s->halo, lo, hi, scale, st, Z_EDGE);
}
}  // namespace b2l

extern "C" {

int b2l_nccl_load(const char* path) {
  if (g_nccl.handle) return 0;
  // prefer the copy already in the process (torch's), then the given path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(-B2L_ENCCL, std::string("nccl: cannot load libnccl.so.2: ") + dlerror());
  g_nccl.handle = h;
  bool ok = bind(g_nccl.GetUniqueId, "ncclGetUniqueId") &&
            bind(g_nccl.CommInitRank, "ncclCommInitRank") &&
            bind(g_nccl.CommDestroy, "ncclCommDestroy") &&
            bind(g_nccl.AllReduce, "ncclAllReduce") && bind(g_nccl.Send, "ncclSend") &&
            bind(g_nccl.Recv, "ncclRecv") && bind(g_nccl.GroupStart, "ncclGroupStart") &&
            bind(g_nccl.GroupEnd, "ncclGroupEnd") &&
            bind(g_nccl.GetErrorString, "ncclGetErrorString");
  if (!ok) {
    g_nccl = NcclApi{};
    return fail(-B2L_ENCCL, "nccl: missing symbols in libnccl.so.2");
  }
  return 0;
}

int b2l_nccl_unique_id(unsigned char* out, int len) {
  B2L_CHECK(out && len >= (int)sizeof(ncclUniqueId), -B2L_EINVAL, "nccl_unique_id: buffer");
  if (int rc = b2l_nccl_load(nullptr)) return rc;
  ncclUniqueId id;
  B2L_NCCL(g_nccl.GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int b2l_slab_create(const unsigned char* nccl_id, int world, int rank, int nx, int ny,
                    int nz_local, b2l_slab** out) {
  B2L_CHECK(out && world >= 1 && rank >= 0 && rank < world && nx > 0 && ny > 0 && nz_local > 0,
            -B2L_EINVAL, "slab_create: bad arguments");
  B2L_CHECK(nccl_id || world == 1, -B2L_EINVAL, "slab_create: world > 1 needs an NCCL id");
  b2l_slab* s = new b2l_slab;
  s->world = world;
  s->rank = rank;
  s->nx = nx;
  s->ny = ny;
  s->nz = nz_local;
  cudaGetDevice(&s->device);
  auto bad = [&](int rc) {
    b2l_slab_destroy(s);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&s->cs, cudaStreamNonBlocking) != cudaSuccess)
    return bad(fail(-B2L_EINVAL, "slab_create: stream"));
  cudaEvent_t* evs[] = {&s->ev_in, &s->ev_halo, &s->ev_f1, &s->ev_red, &s->ev_sg, &s->ev_g2};
  for (cudaEvent_t* e : evs)
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
      return bad(fail(-B2L_EINVAL, "slab_create: event"));
  if (nccl_id) {
    if (int rc = b2l_nccl_load(nullptr)) return bad(rc);
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = g_nccl.CommInitRank(&s->comm, world, id, rank);
    if (r != ncclSuccess) {
      s->comm = nullptr;
      return bad(nccl_fail(r, "ncclCommInitRank"));
    }
  }
  *out = s;
  return 0;
}

int b2l_slab_destroy(b2l_slab* s) {
  if (!s) return 0;
  if (s->cs) cudaStreamSynchronize(s->cs);
  if (s->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(s->comm);
  cudaEvent_t evs[] = {s->ev_in, s->ev_halo, s->ev_f1, s->ev_red, s->ev_sg, s->ev_g2};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (s->cs) cudaStreamDestroy(s->cs);
  if (s->halo) cudaFree(s->halo);
  if (s->part) cudaFree(s->part);
  delete s;
  return 0;
}

int b2l_slab_info(const b2l_slab* s, int* world, int* rank, int* has_comm) {
  B2L_CHECK(s, -B2L_EINVAL, "slab_info: null");
  if (world) *world = s->world;
  if (rank) *rank = s->rank;
  if (has_comm) *has_comm = s->comm != nullptr;
  return 0;
}

int b2l_slab_allreduce(b2l_slab* s, double* buf, long long count, void* stream) {
  B2L_CHECK(s && (buf || count == 0) && count >= 0, -B2L_EINVAL, "slab_allreduce: bad args");
  return slab_allreduce(s, buf, (size_t)count, static_cast<cudaStream_t>(stream));
}

int b2l_slab_stencil7(b2l_slab* s, const double* in, double* out, int ld, double scale,
                      void* stream) {
  B2L_CHECK(s && in && out, -B2L_EINVAL, "slab_stencil7: null");
  return slab_stencil7(s, in, out, ld, scale, static_cast<cudaStream_t>(stream));
}

int b2l_slab_stencil7_gram(b2l_slab* s, const double* in, double* out, int ld, double scale,
                           const double* x, int ldx, int m, int kw, double* gram_out,
                           void* stream) {
  B2L_CHECK(s && in && out && gram_out, -B2L_EINVAL, "slab_stencil7_gram: null");
  return slab_stencil7_gram(s, in, out, ld, scale, x, ldx, m, kw, gram_out,
                            static_cast<cudaStream_t>(stream));
}

int b2l_stencil7_gram_split(const double* in, double* out, int nx, int ny, int nz, int ld,
                            const double* halo, int has_lo, int has_hi, double scale,
                            const double* x, int ldx, int m, int kw, double* gram_out,
                            void* stream) {
  return stencil7_gram_split(in, out, nx, ny, nz, ld, halo, has_lo, has_hi, scale, x, ldx, m, kw,
                             gram_out, static_cast<cudaStream_t>(stream), nullptr, 0, nullptr);
}

}  // extern "C"
