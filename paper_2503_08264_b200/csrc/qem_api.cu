// qem_api.cu -- the C-ABI (include/qem.h): validation, context/workspace,
// phase orchestration and the CUDA-graph QEM loop.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "qem_internal.h"

namespace {
thread_local char g_err[512] = "";

qem_status fail(qem_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

qem_status cuda_fail(cudaError_t e, const char* where) {
  return fail(QEM_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
}

bool sharded(const qem_ctx* c) { return c->g_begin != 0 || c->g_end != c->desc.n; }

qem_status nccl_fail(int r, const char* where) {
  return fail(QEM_NCCL_ERROR, "%s: %s", where, qem::nccl_error_string(r));
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int pad4(int x) { return (x + 3) & ~3; }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

qem_status validate(const qem_model_desc* d, char* msg, size_t cap) {
  char buf[256] = "";
  qem_status s = QEM_OK;
#define BAD(...)                                \
  do {                                          \
    snprintf(buf, sizeof buf, __VA_ARGS__);     \
    s = QEM_INVALID_MODEL;                      \
    goto done;                                  \
  } while (0)
  if (!d) BAD("null model description");
  if (d->K < 1 || d->K > QEM_MAX_K) BAD("K=%d out of range [1, %d]", d->K, QEM_MAX_K);
  if (d->n < 1) BAD("n=%lld must be >= 1", (long long)d->n);
  if (d->n_obs < 0) BAD("n_obs=%d must be >= 0", d->n_obs);
  if (!(d->prior_var > 0)) BAD("prior_var must be > 0");
  if (d->family == QEM_FAMILY_TWO_LEVEL) {
    if (d->d < 1 || d->d > QEM_MAX_D) BAD("d=%d out of range [1, %d]", d->d, QEM_MAX_D);
    if (!qem::tl_supported_d(d->d)) BAD("d=%d has no compiled kernel (QEM_D_MENU: 1-8, 10, 12, 14, 16, 18, 20, 24, 32)", d->d);
    if (d->scale_kind < QEM_SCALE_FIXED || d->scale_kind > QEM_SCALE_LOGVAR) BAD("unknown scale_kind %d", d->scale_kind);
    if (d->scale_kind == QEM_SCALE_FIXED && !(d->fixed_var > 0)) BAD("fixed_var must be > 0");
    if (d->obs_kind == QEM_OBS_GAUSS) {
      if (d->d != 1) BAD("OBS_GAUSS requires d == 1 (got %d)", d->d);
      if (!(d->obs_var > 0)) BAD("obs_var must be > 0");
    } else if (d->obs_kind != QEM_OBS_BERNOULLI_LOGIT) {
      BAD("obs_kind %d not valid for the two-level family", d->obs_kind);
    }
  } else if (d->family == QEM_FAMILY_THREE_LEVEL) {
    if (d->obs_kind != QEM_OBS_POISSON_LOG) BAD("three-level family requires OBS_POISSON_LOG");
    if (d->n_sub < 1) BAD("n_sub=%d must be >= 1", d->n_sub);
    if (d->n_cov < 0 || d->n_cov > QEM_MAX_D) BAD("n_cov=%d out of range", d->n_cov);
    if (!(d->top_var > 0) || !(d->sub_var > 0)) BAD("top_var and sub_var must be > 0");
    if (d->n > (1 << 20) || (int64_t)d->n * d->n_sub * d->K * d->K > (int64_t)1 << 31)
      BAD("three-level model too large for the replicated fp64 tables");
  } else {
    BAD("unknown family %d", d->family);
  }
#undef BAD
done:
  if (msg && cap) {
    strncpy(msg, buf, cap - 1);
    msg[cap - 1] = 0;
  }
  if (s != QEM_OK) fail(s, "%s", buf);
  return s;
}

// Carve the workspace; with base == nullptr only measures.
size_t carve(qem_ctx* c, char* base) {
  const qem_model_desc& d = c->desc;
  const int K = d.K;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  c->cnt = reinterpret_cast<qem::Counters*>(take(sizeof(qem::Counters)));
  if (d.family == QEM_FAMILY_TWO_LEVEL) {
    const int D = d.d;
    c->tw.fwd_coef = reinterpret_cast<float*>(take(sizeof(float) * K * (D + 2)));
    c->tw.bwd_table = reinterpret_cast<float*>(take(sizeof(float) * K * pad4(D + 3)));
    c->tw.f_root = reinterpret_cast<double*>(take(sizeof(double) * K));
    c->tw.ref = reinterpret_cast<qem::RefInfo*>(take(sizeof(qem::RefInfo)));
    // per-CTA plate-sum partials: fp64 (tensor-core forward) or 16-byte split sums (FFMA forward, Fx2)
    c->tw.partial = reinterpret_cast<double*>(take(2 * sizeof(double) * (size_t)c->grid_fwd * (K + 1)));
    c->tw.red = reinterpret_cast<double*>(take(sizeof(double) * (K + 1)));
    c->tw.dg = reinterpret_cast<float*>(take(sizeof(float) * (size_t)c->n_local * K));
    const size_t kp = (size_t)((K + 15) / 16 * 16);  // >= FwdLayout::kpad(K) for any column chunk <= 16
    if (!c->tc)
      c->tw.colrec =  // per group: the column records + a trailer of 4 + pad4(D) floats (FwdLayout::GH)
          reinterpret_cast<float*>(take(sizeof(float) * (size_t)c->n_local * (kp * pad4(D + 3) + 4 + pad4(D))));
    if (c->tc) {
      c->tw.rowop = take((size_t)K * 96);
      c->tw.rowop_x = take((size_t)K * 32);
      c->tw.colop = take((size_t)c->n_local * K * (D == 1 ? 64 : 128));  // TcGeo<D>::COL
      c->tw.colaux = reinterpret_cast<float*>(take((size_t)c->n_local * K * 8));
      c->tw.rowop_b = take((size_t)K * 96);
      c->tw.bgam = reinterpret_cast<float*>(take(sizeof(float) * K));
    }
    c->tw.gstat = reinterpret_cast<float*>(take(sizeof(float) * (size_t)c->n_local));
    c->tw.gmode = reinterpret_cast<int*>(take(sizeof(int) * (size_t)c->n_local));  // TC forward tile modes
    c->tw.gtb = reinterpret_cast<float*>(take(sizeof(float) * (size_t)c->n_local));  // FFMA d = 1 bounds
    c->tw.cvec = reinterpret_cast<double*>(take(sizeof(double) * (size_t)c->n_local));
    c->tw.perm = reinterpret_cast<int*>(take(sizeof(int) * K));
    c->tw.alpha_d = reinterpret_cast<double*>(take(sizeof(double) * K));
    c->tw.coef_d = reinterpret_cast<double*>(take(sizeof(double) * K * (D + 1)));
    c->tw.hmsg = reinterpret_cast<float*>(take(sizeof(float) * (size_t)c->n_local * K));
    c->tw.tA = reinterpret_cast<double*>(take(sizeof(double) * (size_t)c->n_local * K));
    c->tw.bwd_coef = reinterpret_cast<float*>(take(sizeof(float) * K * (D + 1)));
  } else {
    const int64_t A = d.n, AB = d.n * d.n_sub, KK = (int64_t)K * K;
    c->th.f_root = reinterpret_cast<double*>(take(sizeof(double) * K));
    c->th.Lab = reinterpret_cast<double*>(take(sizeof(double) * AB * KK));
    c->th.Mab = reinterpret_cast<double*>(take(sizeof(double) * AB * KK));
    c->th.Fab = reinterpret_cast<double*>(take(sizeof(double) * AB * KK));
    c->th.Ta = reinterpret_cast<double*>(take(sizeof(double) * A * KK));
    c->th.ha = reinterpret_cast<double*>(take(sizeof(double) * A * K));
    c->th.red = reinterpret_cast<double*>(take(sizeof(double) * (K + 1)));
  }
  return off;
}

bool level_ok(const qem_level& l) { return l.q_mean && l.q_var && l.ema_m1 && l.ema_v && l.z && l.w && l.m1 && l.v; }

qem_status need_bound(qem_ctx* c) {
  if (!c) return fail(QEM_INVALID_ARGUMENT, "null context");
  if (!c->bound) return fail(QEM_INVALID_ARGUMENT, "no buffers bound (call qem_bind first)");
  return QEM_OK;
}

}  // namespace

extern "C" {

qem_status qem_model_validate(const qem_model_desc* desc, char* msg, size_t cap) { return validate(desc, msg, cap); }

qem_status qem_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
  if (!begin || !end) return fail(QEM_INVALID_ARGUMENT, "null output pointer");
  if (n < 0 || world < 1 || rank < 0 || rank >= world)
    return fail(QEM_INVALID_ARGUMENT, "bad shard request n=%lld rank=%d world=%d", (long long)n, rank, world);
  *begin = (int64_t)((__int128)n * rank / world);
  *end = (int64_t)((__int128)n * (rank + 1) / world);
  return QEM_OK;
}

// Shared by qem_create / qem_create_in / qem_workspace_bytes: validate, fill the context, size the
// workspace; then (unless measure_only) carve it from `ws` (caller-owned) or a cudaMalloc.
static qem_status create_impl(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin,
                              int64_t group_end, void* ws, size_t ws_cap, size_t* bytes, qem_ctx** out) {
  if (out) *out = nullptr;
  qem_status s = validate(desc, nullptr, 0);
  if (s != QEM_OK) return s;
  if (group_begin < 0 || group_end > desc->n || group_begin >= group_end)
    return fail(QEM_INVALID_ARGUMENT, "bad local group range [%lld, %lld) of n=%lld", (long long)group_begin,
                (long long)group_end, (long long)desc->n);
  if (desc->family == QEM_FAMILY_THREE_LEVEL && (group_begin != 0 || group_end != desc->n))
    return fail(QEM_UNSUPPORTED, "three-level models run as replicas only (no group sharding)");
  if (desc->family == QEM_FAMILY_TWO_LEVEL) {  // shared memory that grows with K and J
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && optin > 0) {
      const size_t need = qem::tl_max_smem(desc);
      if (need > (size_t)optin)
        return fail(QEM_INVALID_MODEL, "K=%d, J=%d needs %zu bytes of shared memory per block (device limit %d)",
                    desc->K, desc->n_obs, need, optin);
    }
  }
  qem_ctx* c = new (std::nothrow) qem_ctx();
  if (!c) return fail(QEM_INVALID_ARGUMENT, "out of host memory");
  c->desc = *desc;
  c->opts.new_weight = 0.3;
  c->opts.schedule_p = 0.0;
  c->opts.var_floor = 1e-8;
  if (opts) c->opts = *opts;
  if (!(c->opts.var_floor > 0) || !(c->opts.new_weight > 0 && c->opts.new_weight <= 1) || c->opts.schedule_p < 0 ||
      c->opts.schedule_p >= 1) {
    delete c;
    return fail(QEM_INVALID_ARGUMENT, "bad options (need 0<new_weight<=1, 0<=schedule_p<1, var_floor>0)");
  }
  if (c->opts.fresh_denominator && desc->family != QEM_FAMILY_TWO_LEVEL) {
    delete c;
    return fail(QEM_UNSUPPORTED, "fresh denominator: two-level family only");
  }
  c->g_begin = group_begin;
  c->g_end = group_end;
  c->n_local = group_end - group_begin;
  c->R = desc->family == QEM_FAMILY_TWO_LEVEL ? desc->d + (desc->scale_kind != QEM_SCALE_FIXED) : 1 + desc->n_cov;
  c->grid_fwd = c->grid_bwd = 1;
  c->tc = desc->family == QEM_FAMILY_TWO_LEVEL && qem::tl_use_tc(desc);
  if (desc->family == QEM_FAMILY_TWO_LEVEL) qem::tl_grids(desc, c->n_local, sm_count(), &c->grid_fwd, &c->grid_bwd, &c->grid_prep);
  c->grid_stage = (int)(c->n_local < sm_count() ? c->n_local : sm_count());
  c->ws_bytes = carve(c, nullptr);
  if (bytes) *bytes = c->ws_bytes;
  if (!out) {  // measure only
    delete c;
    return QEM_OK;
  }
  cudaError_t e = cudaSuccess;
  if (ws) {
    if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0 || ws_cap < c->ws_bytes) {
      const size_t need = c->ws_bytes;
      delete c;
      return fail(QEM_INVALID_ARGUMENT, "caller workspace: need %zu bytes at 256-byte alignment (got %zu)", need, ws_cap);
    }
    c->ws = ws;
    c->ws_owned = false;
  } else {
    e = cudaMalloc(&c->ws, c->ws_bytes);
    if (e != cudaSuccess) {
      delete c;
      return cuda_fail(e, "cudaMalloc(workspace)");
    }
    c->ws_owned = true;
  }
  carve(c, reinterpret_cast<char*>(c->ws));
  e = cudaMemset(c->cnt, 0, sizeof(qem::Counters));
  if (e != cudaSuccess) {
    if (c->ws_owned) cudaFree(c->ws);
    delete c;
    return cuda_fail(e, "cudaMemset");
  }
  *out = c;
  return QEM_OK;
}

qem_status qem_create(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin, int64_t group_end,
                      qem_ctx** out) {
  if (!out) return fail(QEM_INVALID_ARGUMENT, "null output pointer");
  return create_impl(desc, opts, group_begin, group_end, nullptr, 0, nullptr, out);
}

qem_status qem_workspace_bytes(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin,
                               int64_t group_end, size_t* bytes) {
  if (!bytes) return fail(QEM_INVALID_ARGUMENT, "null output pointer");
  return create_impl(desc, opts, group_begin, group_end, nullptr, 0, bytes, nullptr);
}

qem_status qem_create_in(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin, int64_t group_end,
                         void* d_workspace, size_t ws_bytes, qem_ctx** out) {
  if (!out || !d_workspace) return fail(QEM_INVALID_ARGUMENT, "null output or workspace pointer");
  return create_impl(desc, opts, group_begin, group_end, d_workspace, ws_bytes, nullptr, out);
}

void qem_destroy(qem_ctx* c) {
  if (!c) return;
  if (c->graph_valid) cudaGraphExecDestroy(c->graph);
  if (c->nccl_owned) qem::nccl_comm_destroy(c->nccl_comm);
  if (c->ws && c->ws_owned) cudaFree(c->ws);
  delete c;
}

// ---- communicator (SURVEY.md §8(b) qem_set_nccl_comm, §8(e)) ----

qem_status qem_nccl_unique_id(void* h_id) {
  if (!h_id) return fail(QEM_INVALID_ARGUMENT, "null id buffer");
  const int r = qem::nccl_unique_id(h_id);
  return r == 0 ? QEM_OK : nccl_fail(r, "ncclGetUniqueId");
}

// The communicator's (rank, world) must own exactly this context's group block.
static qem_status adopt_comm(qem_ctx* c, void* comm, int owned) {
  int rank = -1, world = 0;
  const int r = qem::nccl_comm_shape(comm, &rank, &world);
  if (r != 0) return nccl_fail(r, "ncclCommCount / ncclCommUserRank");
  int64_t b = 0, e = 0;
  qem_shard_range(c->desc.n, rank, world, &b, &e);
  if (b != c->g_begin || e != c->g_end)
    return fail(QEM_INVALID_ARGUMENT, "communicator rank %d of %d owns groups [%lld, %lld), the context [%lld, %lld)",
                rank, world, (long long)b, (long long)e, (long long)c->g_begin, (long long)c->g_end);
  if (c->nccl_owned) qem::nccl_comm_destroy(c->nccl_comm);
  c->nccl_comm = comm;
  c->nccl_owned = owned;
  c->nccl_rank = rank;
  c->nccl_world = world;
  c->nccl_warm = 0;
  if (c->graph_valid) {  // a captured loop without (or with another) all-reduce is stale
    cudaGraphExecDestroy(c->graph);
    c->graph_valid = 0;
  }
  return QEM_OK;
}

qem_status qem_nccl_init(qem_ctx* c, const void* h_id, int32_t rank, int32_t world) {
  if (!c || !h_id) return fail(QEM_INVALID_ARGUMENT, "null argument");
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "three-level models run as replicas only");
  if (world < 1 || rank < 0 || rank >= world) return fail(QEM_INVALID_ARGUMENT, "bad rank %d of %d", rank, world);
  int64_t b = 0, e = 0;
  qem_shard_range(c->desc.n, rank, world, &b, &e);
  if (b != c->g_begin || e != c->g_end)
    return fail(QEM_INVALID_ARGUMENT, "rank %d of %d owns groups [%lld, %lld), the context [%lld, %lld)", rank, world,
                (long long)b, (long long)e, (long long)c->g_begin, (long long)c->g_end);
  void* comm = nullptr;
  int r = qem::nccl_comm_init(&comm, h_id, rank, world);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  qem_status s = adopt_comm(c, comm, 1);
  if (s != QEM_OK) {
    qem::nccl_comm_destroy(comm);
    return s;
  }
  cudaStream_t st;
  cudaError_t ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return cuda_fail(ce, "qem_nccl_init: stream");
  r = qem::nccl_warmup(c, st);  // connect now (collective, like the init), so later captures see a live comm
  ce = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (r != 0) return nccl_fail(r, "qem_nccl_init: warm-up all-reduce");
  if (ce != cudaSuccess) return cuda_fail(ce, "qem_nccl_init: warm-up sync");
  c->nccl_warm = 1;
  return QEM_OK;
}

qem_status qem_set_nccl_comm(qem_ctx* c, void* nccl_comm) {
  if (!c) return fail(QEM_INVALID_ARGUMENT, "null context");
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "three-level models run as replicas only");
  if (!nccl_comm) {  // detach
    if (c->nccl_owned) qem::nccl_comm_destroy(c->nccl_comm);
    c->nccl_comm = nullptr;
    c->nccl_owned = 0;
    c->nccl_rank = 0;
    c->nccl_world = 1;
    if (c->graph_valid) {
      cudaGraphExecDestroy(c->graph);
      c->graph_valid = 0;
    }
    return QEM_OK;
  }
  return adopt_comm(c, nccl_comm, 0);
}

qem_status qem_nccl_info(const qem_ctx* c, int32_t* rank, int32_t* world, int32_t* version) {
  if (!c) return fail(QEM_INVALID_ARGUMENT, "null context");
  if (rank) *rank = c->nccl_comm ? c->nccl_rank : 0;
  if (world) *world = c->nccl_comm ? c->nccl_world : 1;
  if (version) *version = c->nccl_comm ? qem::nccl_version() : 0;
  return QEM_OK;
}

qem_status qem_bind(qem_ctx* c, const qem_buffers* b) {
  if (!c || !b) return fail(QEM_INVALID_ARGUMENT, "null argument");
  const int nlev = c->desc.family == QEM_FAMILY_TWO_LEVEL ? 2 : 3;
  for (int l = 0; l < nlev; ++l)
    if (!level_ok(b->level[l])) return fail(QEM_INVALID_ARGUMENT, "level %d has a null buffer", l);
  if (!b->x || !b->log_pe) return fail(QEM_INVALID_ARGUMENT, "null observation or log_pe buffer");
  if ((c->desc.obs_kind == QEM_OBS_BERNOULLI_LOGIT || c->desc.obs_kind == QEM_OBS_POISSON_LOG) && !b->y)
    return fail(QEM_INVALID_ARGUMENT, "null label buffer y");
  if (c->opts.fresh_denominator && !b->log_pe_fresh)
    return fail(QEM_INVALID_ARGUMENT, "opts.fresh_denominator needs bufs.log_pe_fresh");
  if (b->eps_bank[0]) {
    for (int l = 1; l < nlev; ++l)
      if (!b->eps_bank[l]) return fail(QEM_INVALID_ARGUMENT, "eps_bank: level %d is NULL", l);
    if (b->eps_bank_len < 1) return fail(QEM_INVALID_ARGUMENT, "eps_bank_len must be >= 1");
  }
  c->bufs = *b;
  c->bound = 1;
  if (c->graph_valid) {
    cudaGraphExecDestroy(c->graph);
    c->graph_valid = 0;
  }
  return QEM_OK;
}

qem_status qem_sample_q(qem_ctx* c, uint64_t seed, int32_t iter, const float* const* d_eps, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (iter < 1 && !d_eps) return fail(QEM_INVALID_ARGUMENT, "iter must be >= 1 in Philox mode");
  c->launches = 0;
  cudaError_t e = qem::launch_sample(c, seed, iter < 1 ? 1 : iter, d_eps, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_q");
}

// Sampler + forward; on the tensor-core path the level-1 draws are fused into the column prep
// (k_colprep_tc: the same Philox counters and transform as k_sample, bit-identical samples), so z is
// written once and never re-read by the prep.  iter 0 = the device iteration counter (graph mode).
static cudaError_t sample_forward(qem_ctx* c, uint64_t seed, int32_t iter, cudaStream_t st) {
  if (!(c->tc && c->desc.family == QEM_FAMILY_TWO_LEVEL)) {
    cudaError_t e = qem::launch_sample(c, seed, iter, nullptr, st);
    if (e != cudaSuccess) return e;
    return c->desc.family == QEM_FAMILY_TWO_LEVEL ? qem::tl_forward(c, st) : qem::th_forward(c, st);
  }
  cudaError_t e = qem::launch_sample(c, seed, iter, nullptr, st, 0, /*root_only=*/1);
  if (e != cudaSuccess) return e;
  c->fuse_sample = 1;
  c->fuse_iter = iter;
  c->fuse_seed = seed;
  e = qem::tl_forward(c, st);
  c->fuse_sample = 0;
  return e;
}

qem_status qem_sample_estep_forward(qem_ctx* c, uint64_t seed, int32_t iter, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (iter < 1) return fail(QEM_INVALID_ARGUMENT, "iter must be >= 1");
  c->launches = 0;
  const cudaError_t e = sample_forward(c, seed, iter, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_estep_forward");
}

qem_status qem_estep_forward(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  c->launches = 0;
  cudaError_t e = c->desc.family == QEM_FAMILY_TWO_LEVEL ? qem::tl_forward(c, (cudaStream_t)stream)
                                                         : qem::th_forward(c, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_forward");
}

qem_status qem_reduce_buffer(qem_ctx* c, double** d_buf, int64_t* count) {
  if (!c || !d_buf || !count) return fail(QEM_INVALID_ARGUMENT, "null argument");
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "three-level has no sharded reduction");
  *d_buf = c->bufs.plate_sum ? c->bufs.plate_sum : c->tw.red;
  *count = c->desc.K + 1;
  return QEM_OK;
}

qem_status qem_estep_backward(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  c->launches = 0;
  cudaError_t e = c->desc.family == QEM_FAMILY_TWO_LEVEL ? qem::tl_backward(c, (cudaStream_t)stream)
                                                         : qem::th_backward(c, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_backward");
}

qem_status qem_estep_reduce(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "three-level has no sharded reduction");
  if (!c->nccl_comm) {
    if (sharded(c)) return fail(QEM_UNSUPPORTED, "sharded context without a communicator (qem_nccl_init / qem_set_nccl_comm)");
    return QEM_OK;  // single rank: the local plate sum is the global one
  }
  const int r = qem::ctx_allreduce(c, (cudaStream_t)stream);
  return r == 0 ? QEM_OK : nccl_fail(r, "qem_estep_reduce");
}

qem_status qem_estep(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (sharded(c) && !c->nccl_comm)
    return fail(QEM_UNSUPPORTED, "qem_estep on a sharded context needs a communicator (qem_nccl_init / "
                                 "qem_set_nccl_comm), or the phase calls with a caller all-reduce");
  s = qem_estep_forward(c, stream);
  if (s) return s;
  const int64_t l = c->launches;
  if (c->nccl_comm) {
    s = qem_estep_reduce(c, stream);
    if (s) return s;
  }
  s = qem_estep_backward(c, stream);
  c->launches += l;
  return s;
}

static cudaError_t evidence_root(qem_ctx* c, cudaStream_t st) {
  c->evidence_only = 1;
  const cudaError_t e = qem::tl_backward(c, st);
  c->evidence_only = 0;
  return e;
}

qem_status qem_evidence_root(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "fresh denominator: two-level family only");
  if (!c->bufs.log_pe_fresh) return fail(QEM_INVALID_ARGUMENT, "bufs.log_pe_fresh is NULL");
  c->launches = 0;
  const cudaError_t e = evidence_root(c, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_evidence_root");
}

qem_status qem_estep_evidence(qem_ctx* c, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "fresh denominator: two-level family only");
  if (!c->bufs.log_pe_fresh) return fail(QEM_INVALID_ARGUMENT, "bufs.log_pe_fresh is NULL");
  if (sharded(c) && !c->nccl_comm)
    return fail(QEM_UNSUPPORTED, "qem_estep_evidence on a sharded context needs a communicator");
  s = qem_estep_forward(c, stream);
  if (s) return s;
  const int64_t l = c->launches;
  if (c->nccl_comm) {
    s = qem_estep_reduce(c, stream);
    if (s) return s;
  }
  s = qem_evidence_root(c, stream);
  c->launches += l;
  return s;
}

qem_status qem_mstep_family(int32_t family, int64_t n, int32_t C, double lam, const double* d_m_new,
                            double* d_m_ema, double* d_params, int32_t* d_status, void* stream) {
  if (family < QEM_QFAMILY_GAMMA || family > QEM_QFAMILY_MULTINOMIAL)
    return fail(QEM_INVALID_ARGUMENT, "unknown Q family %d", family);
  const bool needs_c = family == QEM_QFAMILY_CATEGORICAL || family == QEM_QFAMILY_DIRICHLET ||
                       family == QEM_QFAMILY_BINOMIAL || family == QEM_QFAMILY_MULTINOMIAL;
  if (n < 0 || (needs_c && C < 1) || (family == QEM_QFAMILY_DIRICHLET && C > 16))
    return fail(QEM_INVALID_ARGUMENT, "bad n or C");
  if (n > 0 && (!d_m_new || !d_m_ema || !d_params)) return fail(QEM_INVALID_ARGUMENT, "null array");
  if (!(lam >= 0.0 && lam < 1.0)) return fail(QEM_INVALID_ARGUMENT, "lam must be in [0, 1)");
  const cudaError_t e =
      qem::launch_mstep_family(family, n, C, lam, d_m_new, d_m_ema, d_params, d_status, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_mstep_family");
}

qem_status qem_estep_tables(int64_t n, int32_t K, const double* d_f_root, const double* d_f, double* d_g,
                            double* d_log_pe, double* d_w_root, double* d_w, void* stream) {
  if (n < 0 || K < 1 || K > QEM_TABLES_MAX_K) return fail(QEM_INVALID_ARGUMENT, "need n >= 0 and 1 <= K <= %d", QEM_TABLES_MAX_K);
  if ((int64_t)n * K > ((int64_t)1 << 40)) return fail(QEM_INVALID_ARGUMENT, "tables too large");
  if (!d_f_root || !d_log_pe || !d_w_root || (n > 0 && (!d_f || !d_g || !d_w)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_estep_tables(n, K, d_f_root, d_f, d_g, d_log_pe, d_w_root, d_w, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_tables");
}

qem_status qem_estep_separable(int64_t n, int32_t K, int32_t R, const double* d_f_root, const double* d_rows,
                               const double* d_cols, double* d_g, double* d_log_pe, double* d_w_root, double* d_w,
                               void* stream) {
  if (n < 0 || K < 1 || K > QEM_MAX_K || R < 0 || R > 3)
    return fail(QEM_INVALID_ARGUMENT, "need n >= 0, 1 <= K <= %d, 0 <= R <= 3", QEM_MAX_K);
  if (!d_f_root || !d_rows || !d_log_pe || !d_w_root || (n > 0 && (!d_cols || !d_g || !d_w)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_estep_separable(n, K, R, d_f_root, d_rows, d_cols, d_g, d_log_pe, d_w_root, d_w,
                                                    (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_separable");
}

qem_status qem_cols_gamma_poisson(int64_t n, int32_t K, int32_t J, double alpha, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                  const double* d_q, const double* d_z, double* d_f_root, double* d_rows,
                                  double* d_cols, void* stream) {
  if (n < 0 || K < 1 || J < 0 || !(alpha > 0.0)) return fail(QEM_INVALID_ARGUMENT, "bad sizes or alpha");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || !d_rows ||
      (n > 0 && (!d_q || !d_z || !d_cols || (J > 0 && !d_y))))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_gamma_cols(n, K, J, alpha, d_root_z, d_root_mean, d_root_var, d_y, d_q, d_z,
                                               d_f_root, d_rows, d_cols, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_cols_gamma_poisson");
}

qem_status qem_cols_qmp_gaussian(int64_t n, int32_t K, int32_t J, int32_t scheme, double prior_var, double group_var,
                                 double obs_var, const float* d_root_z, const float* d_root_mean,
                                 const float* d_root_var, const double* d_q, const int32_t* d_copy, const float* d_eps,
                                 const float* d_x, double* d_z, double* d_f_root, double* d_rows, double* d_cols,
                                 void* stream) {
  if (n < 0 || n > 0x7fffffffLL || K < 1 || K > QEM_MAX_K || J < 0 || (scheme != QEM_QMP_PERMUTATION && scheme != QEM_QMP_MIXTURE) ||
      !(prior_var > 0.0) || !(group_var > 0.0) || !(obs_var > 0.0))
    return fail(QEM_INVALID_ARGUMENT, "need 0 <= n < 2^31, 1 <= K <= %d, J >= 0, a scheme and positive variances",
                QEM_MAX_K);
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || !d_rows ||
      (n > 0 && (!d_q || !d_copy || !d_eps || !d_z || !d_cols || (J > 0 && !d_x))))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_qmp_cols(n, K, J, scheme, prior_var, group_var, obs_var, d_root_z, d_root_mean,
                                             d_root_var, d_q, d_copy, d_eps, d_x, d_z, d_f_root, d_rows, d_cols,
                                             (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_cols_qmp_gaussian");
}

qem_status qem_moments_qmp(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z, const double* d_w,
                           const double* d_z, double* d_root_m, double* d_gm, void* stream) {
  if (n < 0 || K < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_w_root || !d_root_z || !d_root_m || (n > 0 && (!d_w || !d_z || !d_gm)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_qmp_moments(n, K, d_w_root, d_root_z, d_w, d_z, d_root_m, d_gm, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_moments_qmp");
}

qem_status qem_cols_beta_binomial(int64_t n, int32_t K, double kappa, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                  const int32_t* d_N, const double* d_q, const double* d_z, double* d_f_root,
                                  double* d_rows, double* d_cols, void* stream) {
  if (n < 0 || K < 1 || !(kappa > 0.0)) return fail(QEM_INVALID_ARGUMENT, "bad sizes or kappa");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || !d_rows ||
      (n > 0 && (!d_y || !d_N || !d_q || !d_z || !d_cols)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_beta_cols(n, K, kappa, d_root_z, d_root_mean, d_root_var, d_y, d_N, d_q, d_z,
                                              d_f_root, d_rows, d_cols, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_cols_beta_binomial");
}

qem_status qem_backward_resample(qem_ctx* c, int32_t S, uint64_t seed, int32_t* d_idx_root, int32_t* d_idx,
                                 void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "backward resampling: two-level family only");
  if (S < 1 || !d_idx_root || !d_idx) return fail(QEM_INVALID_ARGUMENT, "need S >= 1 and output arrays");
  const cudaError_t e = qem::launch_resample(c, S, seed, d_idx_root, d_idx, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_backward_resample");
}

qem_status qem_predictive_loglik(qem_ctx* c, int32_t S, const int32_t* d_idx, int32_t J_test, const void* d_x_test,
                                 const uint8_t* d_y_test, double* d_ll_part, double* d_ll_s, double* d_pll,
                                 void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "predictive log-likelihood: two-level family only");
  if (S < 1 || J_test < 0 || !d_idx || !d_ll_part || !d_ll_s || (J_test > 0 && !d_x_test) ||
      (J_test > 0 && c->desc.obs_kind == QEM_OBS_BERNOULLI_LOGIT && !d_y_test))
    return fail(QEM_INVALID_ARGUMENT, "need S >= 1, J_test >= 0 and the arrays");
  const cudaError_t e = qem::launch_predict(c, S, d_idx, J_test, d_x_test, d_y_test, d_ll_part, d_ll_s, d_pll,
                                            (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_predictive_loglik");
}

qem_status qem_global_iw(qem_ctx* c, double* d_diag, double* d_scratch, double* d_log_pe, double* d_w,
                         double* d_m1, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "global IW: two-level family only");
  if (c->g_begin != 0 || c->g_end != c->desc.n) return fail(QEM_UNSUPPORTED, "global IW: world == 1 only");
  if (!d_diag || !d_scratch || !d_log_pe || !d_w) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_global_iw(c, d_diag, d_scratch, d_log_pe, d_w, d_m1, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_global_iw");
}

qem_status qem_logmeanexp(int64_t n, const double* d_x, double* d_out, void* stream) {
  if (n < 1 || !d_x || !d_out) return fail(QEM_INVALID_ARGUMENT, "need n >= 1 and arrays");
  const cudaError_t e = qem::launch_logmeanexp(n, d_x, d_out, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_logmeanexp");
}

qem_status qem_sample_gamma(int64_t n, int32_t K, uint64_t seed, int32_t iter, const double* d_q, double* d_z,
                            void* stream) {
  if (n < 0 || n > 0xffffffffLL || K < 1 || iter < 1)
    return fail(QEM_INVALID_ARGUMENT, "need 0 <= n < 2^32, K >= 1, iter >= 1");
  if (n > 0 && (!d_q || !d_z)) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_gamma_sample(n, K, seed, iter, d_q, d_z, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_gamma");
}

qem_status qem_tables_gamma_poisson(int64_t n, int32_t K, int32_t J, double alpha, const float* d_root_z,
                                    const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                    const double* d_q, const double* d_z, double* d_f_root, double* d_f,
                                    void* stream) {
  if (n < 0 || K < 1 || J < 0 || !(alpha > 0.0)) return fail(QEM_INVALID_ARGUMENT, "bad sizes or alpha");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || (n > 0 && (!d_q || !d_z || !d_f || (J > 0 && !d_y))))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_gamma_tables(n, K, J, alpha, d_root_z, d_root_mean, d_root_var, d_y, d_q, d_z,
                                                 d_f_root, d_f, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_tables_gamma_poisson");
}

qem_status qem_moments_gamma(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z, const double* d_w,
                             const double* d_z, double* d_root_m, double* d_gm, void* stream) {
  if (n < 0 || K < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_w_root || !d_root_z || !d_root_m || (n > 0 && (!d_w || !d_z || !d_gm)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_gamma_moments(n, K, d_w_root, d_root_z, d_w, d_z, d_root_m, d_gm, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_moments_gamma");
}

qem_status qem_sample_beta(int64_t n, int32_t K, uint64_t seed, int32_t iter, const double* d_q, double* d_z,
                           void* stream) {
  if (n < 0 || n > 0xffffffffLL || K < 1 || iter < 1)
    return fail(QEM_INVALID_ARGUMENT, "need 0 <= n < 2^32, K >= 1, iter >= 1");
  if (n > 0 && (!d_q || !d_z)) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_beta_sample(n, K, seed, iter, d_q, d_z, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_beta");
}

qem_status qem_tables_beta_binomial(int64_t n, int32_t K, double kappa, const float* d_root_z,
                                    const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                    const int32_t* d_N, const double* d_q, const double* d_z, double* d_f_root,
                                    double* d_f, void* stream) {
  if (n < 0 || K < 1 || !(kappa > 0.0)) return fail(QEM_INVALID_ARGUMENT, "bad sizes or kappa");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || (n > 0 && (!d_y || !d_N || !d_q || !d_z || !d_f)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_beta_tables(n, K, kappa, d_root_z, d_root_mean, d_root_var, d_y, d_N, d_q, d_z,
                                                d_f_root, d_f, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_tables_beta_binomial");
}

qem_status qem_moments_beta(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z, const double* d_w,
                            const double* d_z, double* d_root_m, double* d_gm, void* stream) {
  if (n < 0 || K < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_w_root || !d_root_z || !d_root_m || (n > 0 && (!d_w || !d_z || !d_gm)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_beta_moments(n, K, d_w_root, d_root_z, d_w, d_z, d_root_m, d_gm, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_moments_beta");
}

qem_status qem_tables_crossed(int64_t n, int32_t K, int32_t J, int32_t C, int32_t T, const float* d_root_z,
                              const float* d_root_mean, const float* d_root_var, const float* d_z, const float* d_q_mean,
                              const float* d_q_var, const int32_t* d_comp, const int32_t* d_jtype, const uint8_t* d_y,
                              double* d_f_root, double* d_f, void* stream) {
  if (n < 0 || K < 1 || J < 0 || C < 1 || T < 1 || J > 4096) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  {  // the crossed-table kernel stages 8 warps x J offsets (fp64) in shared memory
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && optin > 0 &&
        (size_t)8 * J * sizeof(double) > (size_t)optin)
      return fail(QEM_INVALID_ARGUMENT, "J=%d needs %zu bytes of shared memory per block (device limit %d)", J,
                  (size_t)8 * J * sizeof(double), optin);
  }
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root ||
      (n > 0 && (!d_z || !d_q_mean || !d_q_var || !d_f || (J > 0 && (!d_comp || !d_jtype || !d_y)))))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_crossed_tables(n, K, J, C, T, d_root_z, d_root_mean, d_root_var, d_z, d_q_mean,
                                                   d_q_var, d_comp, d_jtype, d_y, d_f_root, d_f, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_tables_crossed");
}

qem_status qem_estep_crossed(int64_t n, int32_t K, int32_t J, int32_t C, int32_t T, const float* d_root_z,
                             const float* d_root_mean, const float* d_root_var, const float* d_z, const float* d_q_mean,
                             const float* d_q_var, const int32_t* d_comp, const int32_t* d_jtype, const uint8_t* d_y,
                             double* d_f_root, double* d_g, double* d_log_pe, double* d_w_root, double* d_w,
                             void* stream) {
  if (n < 0 || K < 1 || K > QEM_MAX_K || J < 0 || C < 1 || T < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || !d_log_pe || !d_w_root ||
      (n > 0 && (!d_z || !d_q_mean || !d_q_var || !d_g || !d_w || (J > 0 && (!d_comp || !d_jtype || !d_y)))))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  {  // the backward stages K x J row offsets (fp64) per group in shared memory
    int dev = 0, optin = 0;
    const size_t need = (size_t)(2 * K + (size_t)K * J) * sizeof(double) + J + 8;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && optin > 0 &&
        need > (size_t)optin)
      return fail(QEM_INVALID_ARGUMENT, "K=%d, J=%d needs %zu bytes of shared memory per block (device limit %d)", K, J,
                  need, optin);
  }
  const cudaError_t e = qem::launch_crossed_estep(n, K, J, C, T, d_root_z, d_root_mean, d_root_var, d_z, d_q_mean,
                                                  d_q_var, d_comp, d_jtype, d_y, d_f_root, d_g, d_log_pe, d_w_root, d_w,
                                                  (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_crossed");
}

qem_status qem_moments_gaussian(int64_t n, int32_t K, int32_t R, const double* d_w_root, const float* d_root_z,
                                const double* d_w, const float* d_z, double* d_root_m, double* d_gm, void* stream) {
  if (n < 0 || K < 1 || R < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_w_root || !d_root_z || !d_root_m || (n > 0 && (!d_w || !d_z || !d_gm)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_crossed_moments(n, K, R, d_w_root, d_root_z, d_w, d_z, d_root_m, d_gm, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_moments_gaussian");
}

qem_status qem_sample_normal(int64_t rows, int32_t K, int32_t level, uint64_t seed, int32_t iter,
                             const float* d_mean, const float* d_var, const float* d_eps, float* d_z, void* stream) {
  if (rows < 0 || K < 1 || iter < 1 || level < 0 || level > 255)
    return fail(QEM_INVALID_ARGUMENT, "need rows >= 0, K >= 1, iter >= 1, 0 <= level < 256");
  if (rows > 0 && (!d_mean || !d_var || !d_z)) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_sample_rows(rows, K, level, seed, iter, d_mean, d_var, d_eps, d_z, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_normal");
}

qem_status qem_sample_categorical(int64_t n, int32_t C, int32_t K, uint64_t seed, int32_t iter, const double* d_p,
                                  int32_t* d_z, void* stream) {
  if (n < 0 || n > 0xffffffffLL || C < 1 || C > QEM_CAT_MAX_C || K < 1 || iter < 1)
    return fail(QEM_INVALID_ARGUMENT, "need 0 <= n < 2^32, 1 <= C <= %d, K >= 1, iter >= 1", QEM_CAT_MAX_C);
  if (n > 0 && (!d_p || !d_z)) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_sample(n, C, K, seed, iter, d_p, d_z, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_sample_categorical");
}

qem_status qem_tables_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const double* d_x,
                                  const double* d_loglik, const double* d_p, const int32_t* d_z, double* d_f_root,
                                  double* d_f, void* stream) {
  if (n < 0 || C < 1 || C > QEM_CAT_MAX_C || K < 1 || d < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root ||
      (n > 0 && (!d_x || !d_loglik || !d_p || !d_z || !d_f)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_tables(n, C, K, d, d_root_z, d_root_mean, d_root_var, d_x, d_loglik, d_p,
                                               d_z, d_f_root, d_f, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_tables_categorical");
}

qem_status qem_estep_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const float* d_root_z,
                                 const float* d_root_mean, const float* d_root_var, const double* d_x,
                                 const double* d_loglik, const double* d_p, const int32_t* d_z, double* d_f_root,
                                 double* d_g, double* d_log_pe, double* d_w_root, double* d_w, void* stream) {
  if (n < 0 || C < 1 || C > QEM_CAT_MAX_C || K < 1 || K > QEM_TABLES_MAX_K || d < 1)
    return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_root_z || !d_root_mean || !d_root_var || !d_f_root || !d_log_pe || !d_w_root ||
      (n > 0 && (!d_x || !d_loglik || !d_p || !d_z || !d_g || !d_w)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_estep(n, C, K, d, d_root_z, d_root_mean, d_root_var, d_x, d_loglik, d_p, d_z,
                                              d_f_root, d_g, d_log_pe, d_w_root, d_w, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_estep_categorical");
}

qem_status qem_moments_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const double* d_w_root,
                                   const float* d_root_z, const double* d_w, const int32_t* d_z, double* d_root_m,
                                   double* d_pm, void* stream) {
  if (n < 0 || C < 1 || C > QEM_CAT_MAX_C || K < 1 || d < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!d_w_root || !d_root_z || !d_root_m || (n > 0 && (!d_w || !d_z || !d_pm)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e =
      qem::launch_cat_moments(n, C, K, d, d_w_root, d_root_z, d_w, d_z, d_root_m, d_pm, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_moments_categorical");
}

qem_status qem_mstep_categorical(int64_t n, int32_t C, int32_t d, double lam, double var_floor,
                                 const double* d_root_m, double* d_root_ema, float* d_root_mean, float* d_root_var,
                                 const double* d_pm, double* d_p_ema, double* d_p, int64_t* d_clamps, void* stream) {
  if (n < 0 || C < 1 || C > QEM_CAT_MAX_C || d < 1) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (!(lam >= 0.0 && lam < 1.0) || !(var_floor > 0.0)) return fail(QEM_INVALID_ARGUMENT, "need 0 <= lam < 1, var_floor > 0");
  if (!d_root_m || !d_root_ema || !d_root_mean || !d_root_var || (n > 0 && (!d_pm || !d_p_ema || !d_p)))
    return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_mstep(n, C, d, lam, var_floor, d_root_m, d_root_ema, d_root_mean, d_root_var,
                                              d_pm, d_p_ema, d_p, d_clamps, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_mstep_categorical");
}

qem_status qem_mstep_gaussian(int64_t rows, double lam, double var_floor, const double* d_m, double* d_ema,
                              float* d_mean, float* d_var, int64_t* d_clamps, void* stream) {
  if (rows < 0 || rows > 0x7fffffffLL) return fail(QEM_INVALID_ARGUMENT, "bad rows");
  if (!(lam >= 0.0 && lam < 1.0) || !(var_floor > 0.0)) return fail(QEM_INVALID_ARGUMENT, "need 0 <= lam < 1, var_floor > 0");
  if (rows == 0) return QEM_OK;
  if (!d_m || !d_ema || !d_mean || !d_var) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_mstep(0, 1, (int)rows, lam, var_floor, d_m, d_ema, d_mean, d_var, nullptr,
                                              nullptr, nullptr, d_clamps, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_mstep_gaussian");
}

double qem_history_weight(int32_t t, double new_weight, double schedule_p) {
  return schedule_p > 0.0 ? 1.0 - pow((double)(t < 1 ? 1 : t), -schedule_p) : 1.0 - new_weight;
}

qem_status qem_loglik_bernoulli_states(int64_t n, int32_t C, int32_t R, const uint8_t* d_y, const double* d_logit,
                                       double* d_L, void* stream) {
  if (n < 0 || C < 1 || C > QEM_CAT_MAX_C || R < 0) return fail(QEM_INVALID_ARGUMENT, "bad sizes");
  if (n > 0 && (!d_L || (R > 0 && (!d_y || !d_logit)))) return fail(QEM_INVALID_ARGUMENT, "null array");
  const cudaError_t e = qem::launch_cat_loglik(n, C, R, d_y, d_logit, d_L, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_loglik_bernoulli_states");
}

qem_status qem_mstep(qem_ctx* c, int32_t t, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (t < 1) return fail(QEM_INVALID_ARGUMENT, "t must be >= 1");
  c->launches = 0;
  cudaError_t e = qem::launch_mstep(c, t, (cudaStream_t)stream);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_mstep");
}

static cudaError_t iterate_body(qem_ctx* c, uint64_t seed, cudaStream_t st) {
  struct Guard {
    qem_ctx* c;
    ~Guard() { c->in_iterate = 0; }
  } guard{c};
  c->in_iterate = 1;
  cudaError_t e;
  if (c->opts.fresh_denominator) {  // z_new from the independent Philox stream, its evidence first
    e = qem::launch_sample(c, seed, 0, nullptr, st, 0x800000u);
    if (e != cudaSuccess) return e;
    e = qem::tl_forward(c, st);
    if (e != cudaSuccess) return e;
    const int nr = qem::ctx_allreduce(c, st);
    if (nr != 0) {
      c->nccl_last = nr;
      return cudaErrorUnknown;
    }
    e = evidence_root(c, st);
    if (e != cudaSuccess) return e;
  }
  if (c->bufs.eps_bank[0]) {  // parity mode: the bank's draws, then the forward
    e = qem::launch_sample(c, seed, 0, nullptr, st);
    if (e != cudaSuccess) return e;
    e = c->desc.family == QEM_FAMILY_TWO_LEVEL ? qem::tl_forward(c, st) : qem::th_forward(c, st);
  } else {
    e = sample_forward(c, seed, 0, st);
  }
  if (e != cudaSuccess) return e;
  // the only exchange of a sharded iteration: SUM of the (K+1) fp64 plate sums (no-op at one rank)
  const int nr = qem::ctx_allreduce(c, st);
  if (nr != 0) {
    c->nccl_last = nr;
    return cudaErrorUnknown;
  }
  e = c->desc.family == QEM_FAMILY_TWO_LEVEL ? qem::tl_backward(c, st) : qem::th_backward(c, st);
  if (e != cudaSuccess) return e;
  return qem::launch_mstep(c, 0, st);
}

qem_status qem_iterate(qem_ctx* c, int32_t t0, int32_t T, uint64_t seed, int32_t use_graph, void* stream) {
  qem_status s = need_bound(c);
  if (s) return s;
  if (t0 < 1 || T < 0) return fail(QEM_INVALID_ARGUMENT, "need t0 >= 1 and T >= 0");
  if (c->bufs.eps_bank[0] && T > c->bufs.eps_bank_len)
    return fail(QEM_INVALID_ARGUMENT, "T=%d exceeds the bound eps bank (%lld iterations)", T,
                (long long)c->bufs.eps_bank_len);
  if (sharded(c) && !c->nccl_comm)
    return fail(QEM_UNSUPPORTED, "qem_iterate on a sharded context needs a communicator (qem_nccl_init / "
                                 "qem_set_nccl_comm)");
  if (c->nccl_comm && !c->nccl_warm) {  // NCCL connects lazily: one eager collective before any capture
    const int r = qem::nccl_warmup(c, (cudaStream_t)stream);
    if (r != 0) return nccl_fail(r, "qem_iterate: NCCL warm-up");
    c->nccl_warm = 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // device iteration counter and trace base
  int32_t hdr[2] = {t0, t0};
  cudaError_t e = cudaMemcpyAsync(&c->cnt->iter, hdr, sizeof hdr, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "qem_iterate: counter upload");
  e = cudaStreamSynchronize(st);  // hdr is a host stack buffer
  if (e != cudaSuccess) return cuda_fail(e, "qem_iterate: sync");
  int64_t per_iter = 0;
  if (!use_graph) {
    for (int j = 0; j < T; ++j) {
      c->launches = 0;
      c->nccl_last = 0;
      e = iterate_body(c, seed, st);
      if (c->nccl_last) return nccl_fail(c->nccl_last, "qem_iterate (eager): all-reduce");
      if (e != cudaSuccess) return cuda_fail(e, "qem_iterate (eager)");
      per_iter = c->launches;
    }
    c->launches = per_iter * T;
    return QEM_OK;
  }
  if (!c->graph_valid || c->graph_seed_ != seed) {
    if (c->graph_valid) {
      cudaGraphExecDestroy(c->graph);
      c->graph_valid = 0;
    }
    cudaStream_t cap;
    e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "stream create");
    cudaGraph_t g;
    e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      c->launches = 0;
      c->nccl_last = 0;
      cudaError_t eb = iterate_body(c, seed, cap);
      e = cudaStreamEndCapture(cap, &g);
      if (eb != cudaSuccess) e = eb;
      if (c->nccl_last) {
        if (e == cudaSuccess) cudaGraphDestroy(g);
        cudaStreamDestroy(cap);
        return nccl_fail(c->nccl_last, "qem_iterate: graph capture of the all-reduce");
      }
    }
    if (e == cudaSuccess) {
      e = cudaGraphInstantiate(&c->graph, g, 0);
      cudaGraphDestroy(g);
    }
    cudaStreamDestroy(cap);
    if (e != cudaSuccess) return cuda_fail(e, "qem_iterate: graph capture");
    c->graph_valid = 1;
    c->graph_seed_ = seed;
    c->graph_launches_ = c->launches;
  }
  for (int j = 0; j < T; ++j) {
    e = cudaGraphLaunch(c->graph, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
  }
  c->launches = c->graph_launches_ * T;
  return QEM_OK;
}

qem_status qem_read_flags(qem_ctx* c, void* stream, uint32_t* flags, int64_t* clamps) {
  if (!c || !flags) return fail(QEM_INVALID_ARGUMENT, "null argument");
  qem::Counters h;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaMemcpy(&h, c->cnt, sizeof h, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "qem_read_flags");
  *flags = h.flags;
  if (clamps) *clamps = (int64_t)h.clamps;
  uint32_t z = 0;
  unsigned long long zc = 0;
  cudaMemcpy(&c->cnt->flags, &z, sizeof z, cudaMemcpyHostToDevice);
  cudaMemcpy(&c->cnt->clamps, &zc, sizeof zc, cudaMemcpyHostToDevice);
  return QEM_OK;
}

qem_status qem_read_mode_hist(qem_ctx* c, void* stream, uint64_t* h) {
  if (!c || !h) return fail(QEM_INVALID_ARGUMENT, "null argument");
  unsigned long long tmp[8];
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaMemcpy(tmp, c->cnt->mode_hist, sizeof tmp, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(c->cnt->mode_hist, 0, sizeof tmp);
  if (e != cudaSuccess) return cuda_fail(e, "qem_read_mode_hist");
  for (int m = 0; m < 8; ++m) h[m] = tmp[m];
  return QEM_OK;
}

int64_t qem_kernel_launches(const qem_ctx* c) { return c ? c->launches : 0; }

int32_t qem_pair_path(const qem_ctx* c) { return c ? (c->tc ? 1 : 0) : -1; }

qem_status qem_set_kernel_events(qem_ctx* c, void* fwd_start, void* fwd_end, void* bwd_start, void* bwd_end) {
  if (!c) return fail(QEM_INVALID_ARGUMENT, "null context");
  if (c->graph_valid) {  // the captured loop baked the previous events in
    cudaGraphExecDestroy(c->graph);
    c->graph_valid = 0;
  }
  c->ev[0] = fwd_start;
  c->ev[1] = fwd_end;
  c->ev[2] = bwd_start;
  c->ev[3] = bwd_end;
  return QEM_OK;
}

qem_status qem_copy_messages(qem_ctx* c, float* d_dg, double* d_c, void* stream) {
  if (!c || !d_dg || !d_c) return fail(QEM_INVALID_ARGUMENT, "null argument");
  if (c->desc.family != QEM_FAMILY_TWO_LEVEL) return fail(QEM_UNSUPPORTED, "messages are two-level only");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_dg, c->tw.dg, sizeof(float) * c->n_local * c->desc.K, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_c, c->tw.cvec, sizeof(double) * c->n_local, cudaMemcpyDeviceToDevice, st);
  return e == cudaSuccess ? QEM_OK : cuda_fail(e, "qem_copy_messages");
}

const char* qem_status_str(qem_status s) {
  switch (s) {
    case QEM_OK: return "QEM_OK";
    case QEM_INVALID_ARGUMENT: return "QEM_INVALID_ARGUMENT";
    case QEM_INVALID_MODEL: return "QEM_INVALID_MODEL";
    case QEM_UNSUPPORTED: return "QEM_UNSUPPORTED";
    case QEM_CUDA_ERROR: return "QEM_CUDA_ERROR";
    case QEM_NCCL_ERROR: return "QEM_NCCL_ERROR";
  }
  return "QEM_UNKNOWN_STATUS";
}

const char* qem_last_error(void) { return g_err; }

const char* qem_version(void) { return "qem-b200 0.1 (sm_100a)"; }

}  // extern "C"
