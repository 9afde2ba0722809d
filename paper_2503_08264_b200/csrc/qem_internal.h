// qem_internal.h -- context layout and launcher prototypes shared by the
// library's translation units (not part of the public C-ABI, include/qem.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qem.h"

namespace qem {

// Reference-row data for the differenced forward.
struct RefInfo {
  float mu_ref[QEM_MAX_D];  // parent mean of the reference root sample
  double e_ref;             // 1 / V_ref
  double bref_const;        // -(d/2)(ln 2pi + ln V_ref)
  int k_ref;
  int k_star;               // backward reference: argmax_k w_root(k) (tensor-core path)
  float mu_star[QEM_MAX_D]; // parent mean of root sample k_star
  double e_star;            // 1 / V_star
  double bstar_const;       // -(d/2)(ln 2pi + ln V_star)
};

// Two-level workspace (device pointers, carved out of one allocation).
struct TwoLevelWs {
  float* fwd_coef;    // [K][D+2]   alpha, gamma, c[0..D-1]
  float* bwd_table;   // [K][RS]    alpha*log2e, gamma*log2e, c*log2e, w_root (RS = pad4(D+3))
  double* f_root;     // [K]        log p(root^k) - log q(root^k)
  RefInfo* ref;       // [1]
  double* partial;    // [grid][K+1] per-CTA plate sums
  double* red;        // [K+1]      local plate sum (all-reduce buffer)
  float* dg;          // [n_local][K] Delta g_i(k)
  float* colrec;      // [n_local][Kp][pad4(D+3)] column records u[D], |u|^2, P_i, ln P_i
  float* gstat;       // [n_local]  max_k' |u|^2 (forward mode bound)
  double* cvec;       // [n_local]  c_i = g_i(k_ref)
  int* perm;          // [K]        forward row order (rows sorted by coefficient magnitude)
  double* alpha_d;    // [K]        alpha_k in fp64
  double* coef_d;     // [K][D+1]   gamma_k, c_k[D]: the fp32 row coefficients held as fp64 (the TC
                      //            forward's aux merge evaluates alpha'_ik without conversions)
  // tensor-core path (d = 16, K % 256 == 0): bf16x3 operands, DESIGN.md "Tensor cores"
  void* rowop;        // [K] x 96 B  log2e c_k split in 3 bf16 (K-major canonical layout)
  void* rowop_x;      // [K] x 32 B  forward row extra slab (log2e gamma_k pattern, lP switch)
  void* colop;        // [n_local][K] x 128 B  u = z - mu_ref split + column extra slab
  float* colaux;      // [n_local][2][K] SoA {P, ln P}
  int* gmode;         // [n_local]  forward tile mode of the group (decided in k_colprep_tc)
  float* gtb;         // [n_local]  FFMA d = 1: the forward's bound on |D'| over the group (k_forward), 2x bounds the backward's |E|
  double* tA;         // [n_local][K] t_ref(k') = B(k_ref,k') + A_i(k'), A = sum_j log p(x_ij|z^k') - log q(z^k') (fp64)
  void* rowop_b;      // [K] x 96 B  backward rows: log2e (e_k mu_k - e_* mu_*) split (k_star-differenced)
  float* bgam;        // [K]        backward log2e gamma*_k = -log2e (e_k - e_*) / 2
  float* bwd_coef;    // [K][D+1]   FFMA backward rows: Eb_k = e_k mu_k - e_* mu_* (D), Eg_k = -(e_k - e_*)/2
  float* hmsg;        // [n_local][K] h_i(k) = dg_i(k) - alpha'_ik (re-centred message)
};

struct ThreeLevelWs {
  double* f_root;  // [K]
  double* Lab;     // [AB][K kab][K kr]  Poisson table
  double* Mab;     // [AB][K ka][K kr]
  double* Fab;     // [AB][K ka][K kab]  F_ab = lnN(v; u_a, sub_var) - log q(v)
  double* Ta;      // [A][K kr][K ka]
  double* ha;      // [A][K]
  double* red;     // [K+1]
};

struct Counters {
  uint32_t ticket_fwd;
  uint32_t ticket_mstep;
  uint32_t flags;
  uint32_t pad;
  unsigned long long clamps;
  int32_t iter;        // current iteration t (graph mode)
  int32_t trace_base;  // t0 of the running qem_iterate
  unsigned long long mode_hist[8];  // forward tile modes, counted per (warp, group)
  uint32_t claim_fwd;  // k_forward's dynamic group queue (groups past the first wave); reset by its last CTA
  uint32_t claim_bwd;  // k_backward's dynamic group queue; reset by k_root (which always runs just before it)
};

}  // namespace qem

struct qem_ctx {
  qem_model_desc desc;
  qem_opts opts;
  int64_t g_begin, g_end, n_local;
  int R;  // root dims
  int grid_fwd;
  int grid_bwd;
  int grid_prep;
  int grid_stage;  // one CTA per SM, capped by the groups (TMA-staged per-group kernels)
  void* ws;
  size_t ws_bytes;
  bool ws_owned;  // false: caller-owned workspace (qem_create_in)
  qem::TwoLevelWs tw;
  qem::ThreeLevelWs th;
  qem::Counters* cnt;
  qem_buffers bufs;
  int bound;
  int64_t launches;
  cudaGraphExec_t graph;
  int graph_valid;
  int in_iterate;
  int tc;  // d=16 tensor-core pair kernels in use
  int evidence_only;  // the next tl_backward runs the root evidence only (fresh-denominator pass)
  void* ev[4];  // optional caller events around the pair-tile kernels (fwd start/end, bwd start/end)
  uint64_t graph_seed_;
  int64_t graph_launches_;
  // in-library plate-sum all-reduce (qem_nccl.cu): ncclComm_t, NULL = single rank
  void* nccl_comm;
  int nccl_owned;  // created by qem_nccl_init (destroyed with the context)
  int nccl_rank, nccl_world;
  int fuse_sample;     // the next tl_forward's column prep draws the level-1 samples (tensor-core path)
  int fuse_iter;       // ... for this iteration (0: the device counter)
  uint64_t fuse_seed;  // ... with this Philox key
  int nccl_warm;   // one eager collective has run on the communicator
  int nccl_last;   // ncclResult_t of a failed all-reduce inside iterate_body
};

namespace qem {
// two-level launchers (qem_two_level.cu)
cudaError_t tl_forward(qem_ctx* c, cudaStream_t s);
cudaError_t tl_backward(qem_ctx* c, cudaStream_t s);
int tl_supported_d(int d);
int tl_use_tc(const qem_model_desc* d);
size_t tl_max_smem(const qem_model_desc* d);
void tl_grids(const qem_model_desc* d, int64_t n_local, int sms, int* grid_fwd, int* grid_bwd, int* grid_prep);
// three-level launchers (qem_three_level.cu)
cudaError_t th_forward(qem_ctx* c, cudaStream_t s);
cudaError_t th_backward(qem_ctx* c, cudaStream_t s);
// common (qem_common.cu)
cudaError_t launch_sample(qem_ctx* c, uint64_t seed, int32_t iter, const float* const* d_eps,
                          cudaStream_t s, uint32_t iter_or = 0, int root_only = 0);
cudaError_t launch_mstep(qem_ctx* c, int32_t t, cudaStream_t s);
// NCCL, resolved at run time (qem_nccl.cu); int results are ncclResult_t (0 = success)
int ctx_allreduce(qem_ctx* c, cudaStream_t st);
int nccl_warmup(qem_ctx* c, cudaStream_t st);
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, const void* id128, int rank, int world);
int nccl_comm_shape(void* comm, int* rank, int* world);
void nccl_comm_destroy(void* comm);
const char* nccl_error_string(int r);
int nccl_version();
// non-Gaussian Q families (qem_expfam.cu)
cudaError_t launch_estep_tables(int64_t n, int K, const double* f_root, const double* f, double* g, double* log_pe,
                                double* w_root, double* w, cudaStream_t st);
cudaError_t launch_estep_separable(int64_t n, int K, int R, const double* f_root, const double* rows,
                                   const double* cols, double* g, double* log_pe, double* w_root, double* w,
                                   cudaStream_t st);
cudaError_t launch_qmp_cols(int64_t n, int K, int J, int scheme, double pv, double gv, double ov, const float* mu,
                            const float* rm, const float* rv, const double* q, const int32_t* copy, const float* eps,
                            const float* x, double* z, double* f_root, double* rows, double* cols, cudaStream_t st);
cudaError_t launch_qmp_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                               const double* z, double* root_m, double* gm, cudaStream_t st);
cudaError_t launch_gamma_cols(int64_t n, int K, int J, double alpha, const float* mu, const float* rm, const float* rv,
                              const int32_t* y, const double* q, const double* z, double* f_root, double* rows,
                              double* cols, cudaStream_t st);
cudaError_t launch_beta_cols(int64_t n, int K, double kappa, const float* mu, const float* rm, const float* rv,
                             const int32_t* y, const int32_t* N, const double* q, const double* z, double* f_root,
                             double* rows, double* cols, cudaStream_t st);
cudaError_t launch_plate_root(int64_t n, int K, const double* f_root, const double* g, double* scratch,
                              double* log_pe, double* w_root, cudaStream_t st);
cudaError_t launch_cat_estep(int64_t n, int C, int K, int d, const float* rz, const float* rm, const float* rv,
                             const double* x, const double* L, const double* p, const int32_t* z, double* f_root,
                             double* g, double* log_pe, double* w_root, double* w, cudaStream_t st);
cudaError_t launch_gamma_sample(int64_t n, int K, uint64_t seed, int32_t iter, const double* q, double* z,
                                cudaStream_t st);
cudaError_t launch_gamma_tables(int64_t n, int K, int J, double alpha, const float* mu, const float* rm, const float* rv,
                                const int32_t* y, const double* q, const double* z, double* f_root, double* f,
                                cudaStream_t st);
cudaError_t launch_gamma_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                                 const double* z, double* root_m, double* gm, cudaStream_t st);
cudaError_t launch_beta_sample(int64_t n, int K, uint64_t seed, int32_t iter, const double* q, double* z,
                               cudaStream_t st);
cudaError_t launch_beta_tables(int64_t n, int K, double kappa, const float* mu, const float* rm, const float* rv,
                               const int32_t* y, const int32_t* N, const double* q, const double* z, double* f_root,
                               double* f, cudaStream_t st);
cudaError_t launch_beta_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                                const double* z, double* root_m, double* gm, cudaStream_t st);
cudaError_t launch_crossed_tables(int64_t n, int K, int J, int C, int T, const float* rz, const float* rm,
                                  const float* rv, const float* z, const float* qm, const float* qv, const int32_t* comp,
                                  const int32_t* jtype, const uint8_t* y, double* f_root, double* f, cudaStream_t st);
cudaError_t launch_crossed_estep(int64_t n, int K, int J, int C, int T, const float* rz, const float* rm,
                                 const float* rv, const float* z, const float* qm, const float* qv,
                                 const int32_t* comp, const int32_t* jtype, const uint8_t* y, double* f_root,
                                 double* g, double* log_pe, double* w_root, double* w, cudaStream_t st);
cudaError_t launch_crossed_moments(int64_t n, int K, int R, const double* w_root, const float* rz, const double* w,
                                   const float* z, double* root_m, double* gm, cudaStream_t st);
cudaError_t launch_sample_rows(int64_t rows, int K, int level, uint64_t seed, int32_t iter, const float* qm,
                               const float* qv, const float* eps, float* z, cudaStream_t st);
cudaError_t launch_cat_sample(int64_t n, int C, int K, uint64_t seed, int32_t iter, const double* p, int32_t* z,
                              cudaStream_t st);
cudaError_t launch_cat_tables(int64_t n, int C, int K, int d, const float* rz, const float* rm, const float* rv,
                              const double* x, const double* L, const double* p, const int32_t* z, double* f_root,
                              double* f, cudaStream_t st);
cudaError_t launch_cat_mstep(int64_t n, int C, int d, double lam, double floor, const double* root_m, double* root_ema,
                             float* root_mean, float* root_var, const double* pm, double* p_ema, double* p,
                             int64_t* clamps, cudaStream_t st);
cudaError_t launch_cat_loglik(int64_t n, int C, int R, const uint8_t* y, const double* logit, double* L,
                              cudaStream_t st);
cudaError_t launch_cat_moments(int64_t n, int C, int K, int d, const double* w_root, const float* rz, const double* w,
                               const int32_t* z, double* root_m, double* pm, cudaStream_t st);
cudaError_t launch_resample(qem_ctx* c, int S, uint64_t seed, int32_t* idx_root, int32_t* idx, cudaStream_t st);
cudaError_t launch_predict(qem_ctx* c, int S, const int32_t* idx, int J, const void* x, const uint8_t* y,
                           double* ll_part, double* ll_s, double* pll, cudaStream_t st);
cudaError_t launch_global_iw(qem_ctx* c, double* diag, double* scratch, double* log_pe, double* w, double* m1,
                             cudaStream_t st);
cudaError_t launch_logmeanexp(int64_t n, const double* x, double* out, cudaStream_t st);
cudaError_t launch_mstep_family(int family, int64_t n, int C, double lam, const double* m_new, double* m_ema,
                                double* params, int32_t* status, cudaStream_t st);
}  // namespace qem
