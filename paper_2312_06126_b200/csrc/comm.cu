// comm.cu -- NCCL for the in-group gradient exchange (north_star "NCCL allreduce
// of the small gradient buffers over NVLink").
//
// NCCL is resolved at run time with dlopen (the copy torch ships, or any libnccl.so.2 on the
// loader path), so the single-GPU library has no link-time NCCL dependency and multi-rank
// learners fail loudly with SPZ_ENCCL if it is missing.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "comm.h"
#include "internal.h"

namespace spz {

namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* cands[] = {"/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
    for (const char* c : cands)
      if ((h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
  }
  if (!h) {
    g_nccl.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
    return;
  }
  g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.AllReduce = reinterpret_cast<decltype(g_nccl.AllReduce)>(dlsym(h, "ncclAllReduce"));
  g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  g_nccl.Broadcast = reinterpret_cast<decltype(g_nccl.Broadcast)>(dlsym(h, "ncclBroadcast"));
  g_nccl.CommSplit = reinterpret_cast<decltype(g_nccl.CommSplit)>(dlsym(h, "ncclCommSplit"));
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce && g_nccl.GetErrorString &&
              g_nccl.Broadcast && g_nccl.CommSplit;
  if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks required symbols";
}

spz_status nccl_fail(const char* what, ncclResult_t r) {
  return fail(SPZ_ENCCL, std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
}
}  // namespace

spz_status nccl_available() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) return fail(SPZ_ENCCL, g_nccl.why);
  return SPZ_OK;
}

spz_status comm_init(Comm* c, const uint8_t* uid, int world, int rank) {
  spz_status s = nccl_available();
  if (s != SPZ_OK) return s;
  ncclUniqueId id;
  std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm;
  ncclResult_t r = g_nccl.CommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  c->handle = comm;
  c->world = world;
  c->rank = rank;
  return SPZ_OK;
}

spz_status comm_split(const Comm& world, int color, int key, Comm* out) {
  ncclComm_t nc;
  ncclResult_t r = g_nccl.CommSplit(static_cast<ncclComm_t>(world.handle), color, key, &nc, nullptr);
  if (r != ncclSuccess) return nccl_fail("ncclCommSplit", r);
  out->handle = nc;
  out->rank = key;
  out->world = -1;
  return SPZ_OK;
}

cudaError_t comm_broadcast_f32(const Comm& c, float* buf, size_t count, int root, cudaStream_t st) {
  ncclResult_t r = g_nccl.Broadcast(buf, buf, count, ncclFloat32, root, static_cast<ncclComm_t>(c.handle), st);
  if (r != ncclSuccess) {
    set_error(std::string("ncclBroadcast: ") + g_nccl.GetErrorString(r));
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

void comm_destroy(Comm* c) {
  if (c->handle && g_nccl.ok) g_nccl.CommDestroy(static_cast<ncclComm_t>(c->handle));
  c->handle = nullptr;
}

cudaError_t comm_allreduce_sum(const Comm& c, void* buf, size_t count, bool f64, cudaStream_t st) {
  ncclResult_t r = g_nccl.AllReduce(buf, buf, count, f64 ? ncclFloat64 : ncclFloat32, ncclSum,
                                    static_cast<ncclComm_t>(c.handle), st);
  if (r != ncclSuccess) {
    set_error(std::string("ncclAllReduce: ") + g_nccl.GetErrorString(r));
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace spz

extern "C" spz_status spz_nccl_unique_id(uint8_t out[128]) {
  if (!out) return spz::fail(SPZ_EINVAL, "spz_nccl_unique_id: NULL out");
  spz_status s = spz::nccl_available();
  if (s != SPZ_OK) return s;
  ncclUniqueId id;
  ncclResult_t r = spz::g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return spz::nccl_fail("ncclGetUniqueId", r);
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return SPZ_OK;
}
