// In-library NCCL transport of the column-sharded engine:
// one process per GPU, the global-level exchanges as ncclAllGather inside
// each rank group, all enqueued by one C call per run (no Python, no host
// sync).  libnccl.so.2 is opened at run time (dlopen): a process that
// already loaded NCCL -- torch does -- shares that copy; the library itself
// has no link-time NCCL dependency.  Declarations come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/blockinv_b200.h"
#include "bi_common.cuh"
#include "bi_shard_internal.cuh"

namespace bi {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not found: ") + (dlerror() ? dlerror() : "");
      return a;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommSplit && a.CommDestroy && a.AllGather && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks ncclCommSplit/ncclAllGather (NCCL >= 2.18 required)";
    return a;
  }();
  return api;
}

int nccl_fail(const char* what, ncclResult_t r) {
  set_error(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
  return BI_ENCCL;
}

}  // namespace
}  // namespace bi

void bi::shard_destroy_comms(bi_engine* e) {
  auto& comms = shard_group_comms(e);
  if (nccl().ok)
    for (auto& kv : comms) nccl().CommDestroy(static_cast<ncclComm_t>(kv.second));
  comms.clear();
}

using namespace bi;

#define BI_NCCL_TRY(expr)                                        \
  do {                                                           \
    ncclResult_t _r = (expr);                                    \
    if (_r != ncclSuccess) return ::bi::nccl_fail(#expr, _r);    \
  } while (0)

extern "C" int bi_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int bi_nccl_unique_id(unsigned char* id) {
  BI_REQUIRE(id != nullptr, "null argument");
  if (!nccl().ok) {
    set_error(nccl().why);
    return BI_ENCCL;
  }
  ncclUniqueId u;
  BI_NCCL_TRY(nccl().GetUniqueId(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

extern "C" int bi_nccl_comm_init(int nranks, const unsigned char* id, int rank, void** comm) {
  BI_REQUIRE(id && comm && nranks >= 1 && rank >= 0 && rank < nranks, "bad communicator arguments");
  if (!nccl().ok) {
    set_error(nccl().why);
    return BI_ENCCL;
  }
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  BI_NCCL_TRY(nccl().CommInitRank(&c, nranks, u, rank));
  *comm = c;
  return 0;
}

extern "C" int bi_nccl_comm_destroy(void* comm) {
  if (!comm) return 0;
  if (!nccl().ok) return BI_ENCCL;
  BI_NCCL_TRY(nccl().CommDestroy(static_cast<ncclComm_t>(comm)));
  return 0;
}

// The engine's group communicators: one ncclCommSplit of the world
// communicator per power-of-two group size (color = the group, key = rank).
// Collective over the world communicator: every rank calls it, same order.
extern "C" int bi_engine_shard_set_comm(bi_engine* e, void* world) {
  BI_REQUIRE(e && world, "null argument");
  BI_REQUIRE(shard_staging(e), "engine created without BI_SHARD_STAGING");
  if (!nccl().ok) {
    set_error(nccl().why);
    return BI_ENCCL;
  }
  shard_destroy_comms(e);
  auto& comms = shard_group_comms(e);
  const int P = shard_nranks(e), r = shard_rank(e);
  for (int gs = 2; gs <= P; gs *= 2) {
    ncclComm_t sub = nullptr;
    BI_NCCL_TRY(nccl().CommSplit(static_cast<ncclComm_t>(world), r / gs, r, &sub, nullptr));
    comms[gs] = sub;
  }
  return 0;
}

// Steps [first, last] of this rank: segments (CUDA graphs) and, at every
// global-level exchange, pack -> ncclAllGather in the group -> unpack, all
// on `stream`.
extern "C" int bi_engine_run_nccl(bi_engine* e, int first_step, int last_step, int use_graph, void* stream) {
  BI_REQUIRE(e, "null engine");
  const int n = bi_engine_shard_segments(e, first_step, last_step, nullptr, nullptr, nullptr, 0);
  if (n < 0) return n;
  std::vector<int> b(n), en(n), x(n);
  bi_engine_shard_segments(e, first_step, last_step, b.data(), en.data(), x.data(), n);
  auto& comms = shard_group_comms(e);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (first_step == 1) {
    int rc = shard_zero_minv(e, s);
    if (rc) return rc;
  }
  for (int k = 0; k < n; ++k) {
    int rc = bi_engine_run_ops(e, b[k], en[k], use_graph, stream);
    if (rc) return rc;
    if (x[k] < 0) continue;
    int64_t d[8];
    bi_engine_xchg_desc(e, x[k], d);
    const int gs = (int)d[1];
    if ((rc = bi_engine_xchg_pack(e, x[k], stream)) != 0) return rc;
    if (gs > 1) {  // (a group of one packs straight into the receive area)
      auto it = comms.find(gs);
      BI_REQUIRE(it != comms.end(), "group communicators missing: call bi_engine_shard_set_comm first");
      double *send = nullptr, *recv = nullptr;
      bi_engine_shard_buffers(e, &send, &recv);
      BI_NCCL_TRY(nccl().AllGather(send, recv, (size_t)(d[2] * d[3]), ncclDouble,
                                   static_cast<ncclComm_t>(it->second), s));
    }
    if ((rc = bi_engine_xchg_unpack(e, x[k], stream)) != 0) return rc;
  }
  return 0;
}
