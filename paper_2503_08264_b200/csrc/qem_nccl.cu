// qem_nccl.cu -- the in-library plate-sum all-reduce (north star "a tiny
// NCCL all-reduce (in log-sum-exp-safe form) over NVLink").
//
// Groups shard contiguously over ranks (qem_shard_range); each rank's forward leaves its local
// plate sum [G_r(0..K-1), sum_i c_i] (fp64, K+1 entries) in the reduce buffer, and one SUM
// all-reduce of that buffer is the only exchange of a QEM iteration: the plate product is a plain
// sum of centred log-messages (Eq. 7c; elimination PAPER.md:393), so nothing is
// exponentiated before the reduction.  Every rank then runs the root softmax redundantly on the
// identical reduced bytes.
//
// NCCL is resolved at run time (dlopen): the process normally has torch's libnccl.so.2 loaded
// already (RTLD_NOLOAD finds it, so libqem and torch share one NCCL), else QEM_NCCL_LIB or the
// default search path.  A process that never asks for a communicator never touches NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "qem_internal.h"

namespace qem {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*comm_count)(const ncclComm_t, int*);
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*get_version)(int*);
  const char* (*error_string)(ncclResult_t);
};

namespace {
NcclApi g_api;
int g_state = 0;  // 0 = not tried, 1 = loaded, -1 = failed
char g_why[256] = "";
std::mutex g_mu;

void* open_nccl() {
  const char* env = getenv("QEM_NCCL_LIB");
  if (env && *env) return dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  // torch links libnccl.so.2; prefer the copy already in the process
  if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD)) return h;
  if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL)) return h;
  return dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
}
}  // namespace

const NcclApi* nccl_api(const char** why) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_state == 0) {
    void* h = open_nccl();
    if (!h) {
      snprintf(g_why, sizeof g_why, "cannot load NCCL (libnccl.so.2; set QEM_NCCL_LIB): %s", dlerror());
      g_state = -1;
    } else {
#define SYM(field, name)                                                            \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));            \
  if (!g_api.field) {                                                               \
    snprintf(g_why, sizeof g_why, "NCCL library lacks %s", name);                   \
    g_state = -1;                                                                   \
  }
      g_state = 1;
      SYM(get_unique_id, "ncclGetUniqueId")
      SYM(comm_init_rank, "ncclCommInitRank")
      SYM(comm_destroy, "ncclCommDestroy")
      SYM(comm_count, "ncclCommCount")
      SYM(comm_user_rank, "ncclCommUserRank")
      SYM(all_reduce, "ncclAllReduce")
      SYM(get_version, "ncclGetVersion")
      SYM(error_string, "ncclGetErrorString")
#undef SYM
    }
  }
  if (g_state != 1) {
    if (why) *why = g_why;
    return nullptr;
  }
  return &g_api;
}

const char* nccl_error_string(int r) {
  const char* why = "";
  const NcclApi* api = nccl_api(&why);
  return api ? api->error_string((ncclResult_t)r) : why;
}

// SUM all-reduce of the context's reduce buffer (K+1 fp64) in place on `st` over the bound
// communicator.  Returns the ncclResult_t (0 = success); a context without a communicator is a
// no-op (single rank).
int ctx_allreduce(qem_ctx* c, cudaStream_t st) {
  if (!c->nccl_comm) return 0;
  const NcclApi* api = nccl_api(nullptr);
  if (!api) return (int)ncclSystemError;
  double* buf = c->bufs.plate_sum ? c->bufs.plate_sum : c->tw.red;
  return (int)api->all_reduce(buf, buf, (size_t)c->desc.K + 1, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, st);
}

// One eager all-reduce over the context's own reduce buffer (its contents are scratch until the
// next forward): NCCL sets up its connections on the first collective of a communicator, which
// must not happen inside a stream capture.
int nccl_warmup(qem_ctx* c, cudaStream_t st) {
  const NcclApi* api = nccl_api(nullptr);
  if (!api) return (int)ncclSystemError;
  double* buf = c->tw.red;
  return (int)api->all_reduce(buf, buf, (size_t)c->desc.K + 1, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, st);
}

int nccl_unique_id(void* out128) {
  const NcclApi* api = nccl_api(nullptr);
  if (!api) return (int)ncclSystemError;
  return (int)api->get_unique_id(reinterpret_cast<ncclUniqueId*>(out128));
}

int nccl_comm_init(void** comm, const void* id128, int rank, int world) {
  const NcclApi* api = nccl_api(nullptr);
  if (!api) return (int)ncclSystemError;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclComm_t cm = nullptr;
  const ncclResult_t r = api->comm_init_rank(&cm, world, id, rank);
  *comm = cm;
  return (int)r;
}

int nccl_comm_shape(void* comm, int* rank, int* world) {
  const NcclApi* api = nccl_api(nullptr);
  if (!api) return (int)ncclSystemError;
  ncclResult_t r = api->comm_count((ncclComm_t)comm, world);
  if (r == ncclSuccess) r = api->comm_user_rank((ncclComm_t)comm, rank);
  return (int)r;
}

void nccl_comm_destroy(void* comm) {
  const NcclApi* api = nccl_api(nullptr);
  if (api && comm) api->comm_destroy((ncclComm_t)comm);
}

int nccl_version() {
  const NcclApi* api = nccl_api(nullptr);
  int v = 0;
  if (api) api->get_version(&v);
  return v;
}

}  // namespace qem
