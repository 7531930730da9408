// Row-partitioned feature exchange through NCCL for non-Python callers of the
// C ABI (SURVEY 8(b) hg_allgather_features, 8(e)): an exact-count all-gather
// of each rank's feature rows [s_p, s_{p+1}) into the [N, F] buffer every
// rank's SpMM reads in place -- one NCCL group of P broadcasts (the
// all-gather-v idiom), so no rank is padded to the largest partition.
//
// libnccl is bound at run time (dlopen: the copy already loaded in the
// process, e.g. torch's, else libnccl.so.2), so libhalfgnn.so carries no link
// dependency on NCCL; only nccl.h's types are used at compile time.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "hg_common.cuh"

namespace hg {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.group_start &&
             api.group_end && api.broadcast && api.error_string;
  });
  return api;
}

#define HG_NCCL(call)                                                                    \
  do {                                                                                   \
    ncclResult_t hg_r_ = (call);                                                         \
    if (hg_r_ != ncclSuccess) {                                                          \
      ::hg::set_error("NCCL error '%s' at %s:%d", nccl().error_string(hg_r_), __FILE__, \
                      __LINE__);                                                         \
      return HG_ECUDA;                                                                   \
    }                                                                                    \
  } while (0)

}  // namespace hg

using namespace hg;

extern "C" int hg_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int hg_nccl_unique_id(void* id_out) {
  HG_REQUIRE(nccl().ok, "hg_nccl_unique_id: libnccl.so.2 not found");
  HG_REQUIRE(id_out, "hg_nccl_unique_id: null output");
  ncclUniqueId id;
  HG_NCCL(nccl().get_unique_id(&id));
  memcpy(id_out, &id, sizeof(id));
  return HG_OK;
}

extern "C" int hg_nccl_comm_init(void** comm_out, int32_t nranks, const void* id, int32_t rank) {
  HG_REQUIRE(nccl().ok, "hg_nccl_comm_init: libnccl.so.2 not found");
  HG_REQUIRE(comm_out && id && nranks >= 1 && rank >= 0 && rank < nranks,
             "hg_nccl_comm_init: bad arguments");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  HG_NCCL(nccl().comm_init_rank(&comm, nranks, uid, rank));
  *comm_out = comm;
  return HG_OK;
}

extern "C" int hg_nccl_comm_destroy(void* comm) {
  HG_REQUIRE(nccl().ok, "hg_nccl_comm_destroy: libnccl.so.2 not found");
  if (comm) HG_NCCL(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
  return HG_OK;
}

extern "C" int hg_allgather_features(void* comm, const void* x_local, void* x_full,
                                     const int64_t* splits, int32_t parts, int32_t rank,
                                     int64_t row_bytes, void* stream) {
  HG_REQUIRE(nccl().ok, "hg_allgather_features: libnccl.so.2 not found");
  HG_REQUIRE(comm && splits && parts >= 1 && rank >= 0 && rank < parts && row_bytes > 0,
             "hg_allgather_features: bad arguments");
  HG_REQUIRE(splits[0] == 0, "hg_allgather_features: splits must start at 0");
  for (int q = 0; q < parts; ++q)
    HG_REQUIRE(splits[q + 1] >= splits[q], "hg_allgather_features: splits must not decrease");
  HG_REQUIRE(x_full && (x_local || splits[rank + 1] == splits[rank]),
             "hg_allgather_features: null buffer");
  char* full = static_cast<char*>(x_full);
  cudaStream_t st = as_stream(stream);
  HG_NCCL(nccl().group_start());
  for (int q = 0; q < parts; ++q) {
    const size_t bytes = (size_t)(splits[q + 1] - splits[q]) * (size_t)row_bytes;
    char* dst = full + (size_t)splits[q] * (size_t)row_bytes;
    const void* src = q == rank ? x_local : dst;
    ncclResult_t r = nccl().broadcast(src, dst, bytes, ncclUint8, q, static_cast<ncclComm_t>(comm), st);
    if (r != ncclSuccess) {
      nccl().group_end();
      HG_NCCL(r);
    }
  }
  HG_NCCL(nccl().group_end());
  return HG_OK;
}
