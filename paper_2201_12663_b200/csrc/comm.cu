// comm.cpp - collectives for the R-sharded RHOSVD path.
//
// Every R-dependent quantity on the path is a sum over canonical terms
// (T_l, G_l, the b x b Grams of W, Uhat X, rho, beta), so the only collective
// is an fp64 SUM all-reduce.  Two backends behind one handle:
//   * NCCL (NVLink 5 / NVSwitch), loaded with dlopen so the library has no
//     link-time NCCL dependency (torch's bundled libnccl.so.2 is picked up
//     when already loaded);
//   * a host callback (e.g. torch.distributed gloo), used by the multi-rank
//     tests that run world_size 2 on one GPU or on CPU.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "comm.h"

namespace rhosvd {

namespace {
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, NcclUid, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*reduce)(const void*, void*, size_t, int, int, int, void*, cudaStream_t) = nullptr;
  int (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  bool ok = false;
};
NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (a.h) {
      a.getUniqueId = (int (*)(void*))dlsym(a.h, "ncclGetUniqueId");
      a.commInitRank = (int (*)(void**, int, NcclUid, int))dlsym(a.h, "ncclCommInitRank");
      a.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(a.h, "ncclAllReduce");
      a.reduce = (int (*)(const void*, void*, size_t, int, int, int, void*, cudaStream_t))dlsym(a.h, "ncclReduce");
      a.broadcast = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(a.h, "ncclBroadcast");
      a.commDestroy = (int (*)(void*))dlsym(a.h, "ncclCommDestroy");
      a.getErrorString = (const char* (*)(int))dlsym(a.h, "ncclGetErrorString");
      a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.reduce && a.broadcast && a.commDestroy;
    }
  }
  return a;
}
constexpr int kNcclFloat64 = 8, kNcclSum = 0;
}  // namespace

int comm_allreduce(rhosvd_comm* c, double* p, int64_t count, cudaStream_t st) {
  if (!c || !c->active() || count <= 0) return RHOSVD_OK;
  if (c->kind == rhosvd_comm::NCCL) {
    int r = api().allReduce(p, p, (size_t)count, kNcclFloat64, kNcclSum, c->nccl, st);
    if (r != 0)
      return fail(RHOSVD_ENCCL, std::string("ncclAllReduce: ") +
                                    (api().getErrorString ? api().getErrorString(r) : std::to_string(r)));
    return RHOSVD_OK;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, cudaGetErrorString(e));
  int r = c->fn(p, count, (rhosvd_stream)st, c->user);
  if (r != 0) return fail(RHOSVD_ENCCL, "callback all-reduce failed: " + std::to_string(r));
  // the callback may copy back with a synchronous cudaMemcpy from pageable memory, which can
  // return before the DMA lands and is ordered only on the legacy stream: make the result
  // visible to work queued on `st` (a non-blocking stream) before continuing
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, cudaGetErrorString(e));
  return RHOSVD_OK;
}

static int nccl_status(int r, const char* what) {
  if (r == 0) return RHOSVD_OK;
  return fail(RHOSVD_ENCCL, std::string(what) + ": " +
                                (api().getErrorString ? api().getErrorString(r) : std::to_string(r)));
}

int comm_reduce_root(rhosvd_comm* c, double* p, int64_t count, cudaStream_t st) {
  if (!c || !c->active() || count <= 0) return RHOSVD_OK;
  if (c->kind == rhosvd_comm::NCCL)
    return nccl_status(api().reduce(p, p, (size_t)count, kNcclFloat64, kNcclSum, 0, c->nccl, st), "ncclReduce");
  return comm_allreduce(c, p, count, st);  // callback backend: every rank gets the sum
}

int comm_broadcast(rhosvd_comm* c, double* p, int64_t count, int root, cudaStream_t st) {
  if (!c || !c->active() || count <= 0) return RHOSVD_OK;
  if (c->kind == rhosvd_comm::NCCL)
    return nccl_status(api().broadcast(p, p, (size_t)count, kNcclFloat64, root, c->nccl, st), "ncclBroadcast");
  // callback backend (sum only): the non-root ranks contribute zeros; x + 0 = x exactly
  if (c->rank != root) {
    cudaError_t e = cudaMemsetAsync(p, 0, (size_t)count * sizeof(double), st);
    if (e != cudaSuccess) return fail(RHOSVD_ECUDA, cudaGetErrorString(e));
  }
  return comm_allreduce(c, p, count, st);
}

}  // namespace rhosvd

using namespace rhosvd;

extern "C" int rhosvd_nccl_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(RHOSVD_EINVAL, "null id");
  if (!api().ok) return fail(RHOSVD_ENCCL, "libnccl.so.2 not loadable");
  NcclUid u;
  int r = api().getUniqueId(&u);
  if (r != 0) return fail(RHOSVD_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(id, u.b, 128);
  return RHOSVD_OK;
}

extern "C" int rhosvd_comm_init_nccl(const uint8_t id[128], int world, int rank, rhosvd_comm** out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return fail(RHOSVD_EINVAL, "bad comm args");
  *out = nullptr;
  if (!api().ok) return fail(RHOSVD_ENCCL, "libnccl.so.2 not loadable");
  auto* c = new rhosvd_comm();
  c->kind = rhosvd_comm::NCCL;
  c->world = world;
  c->rank = rank;
  c->force = getenv("RHOSVD_COMM_FORCE") && getenv("RHOSVD_COMM_FORCE")[0] == '1';
  NcclUid u;
  std::memcpy(u.b, id, 128);
  int r = api().commInitRank(&c->nccl, world, u, rank);
  if (r != 0) {
    delete c;
    return fail(RHOSVD_ENCCL, "ncclCommInitRank failed: " + std::to_string(r));
  }
  *out = c;
  return RHOSVD_OK;
}

extern "C" int rhosvd_comm_init_callback(rhosvd_allreduce_fn fn, void* user, int world, int rank,
                                         rhosvd_comm** out) {
  if (!out || !fn || world < 1 || rank < 0 || rank >= world) return fail(RHOSVD_EINVAL, "bad comm args");
  auto* c = new rhosvd_comm();
  c->kind = rhosvd_comm::CALLBACK;
  c->fn = fn;
  c->user = user;
  c->world = world;
  c->rank = rank;
  c->force = getenv("RHOSVD_COMM_FORCE") && getenv("RHOSVD_COMM_FORCE")[0] == '1';
  *out = c;
  return RHOSVD_OK;
}

extern "C" void rhosvd_comm_destroy(rhosvd_comm* c) {
  if (!c) return;
  if (c->kind == rhosvd_comm::NCCL && c->nccl && api().ok) api().commDestroy(c->nccl);
  delete c;
}
