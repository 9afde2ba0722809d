/*
 * qem.h -- C-ABI of the B200-native QEM MPIW E-step library (libqem.so).
 *
 * Implements the data-parallel hot path of QEM (arXiv 2503.08264): sample K
 * copies of every latent from the factorised Gaussian Q, evaluate every
 * (parent sample k, child sample k') log-factor of every plate instance,
 * reduce them by max-shifted log-sum-exp along the plate tree into the
 * log-marginal estimate log Pe over all K^n index tuples, run the backward
 * (marginal) pass for each latent's per-sample weights, form first/second
 * moments, and apply the EMA + closed-form Gaussian M-step.
 *
 * Citations are PAPER.md:<line> (section / equation) of the paper text:
 *   Eq. 7a-c  (Sec. 3.2)  MPIW moment, weight, evidence
 *   Alg. 1            QEM loop
 *   Eq. 9     (Sec. 4)    EMA over mean parameters
 *   PAPER.md:393-394 (Limitations)          elimination over the plate tree,
 *                                           grouping, chunking
 * Readings of ambiguous points (R1..R43) are listed in DESIGN.md.
 *
 * ENTRY POINTS
 *  - the hot path (context-based, two- and three-level Gaussian models):
 *    qem_model_validate, qem_shard_range, qem_create / qem_workspace_bytes + qem_create_in,
 *    qem_bind, qem_sample_q, qem_estep (= qem_estep_forward + qem_estep_reduce (the NCCL
 *    all-reduce of qem_reduce_buffer) + qem_estep_backward), qem_mstep, qem_iterate (CUDA graph),
 *    the communicator (qem_nccl_unique_id, qem_nccl_init, qem_set_nccl_comm, qem_nccl_info),
 *    qem_read_flags, diagnostics (qem_read_mode_hist, qem_set_kernel_events,
 *    qem_copy_messages, qem_kernel_launches, qem_pair_path);
 *  - NEXT rows: qem_estep_evidence / qem_evidence_root (fresh-sample
 *    denominator), qem_mstep_family (Gamma, Beta, Dirichlet, Bernoulli, Binomial,
 *    Multinomial, Categorical M-steps), qem_estep_tables (the E-step on explicit log-factor
 *    tables), discrete latents (qem_sample_categorical, qem_estep_categorical,
 *    qem_tables_categorical, qem_moments_categorical, qem_mstep_categorical,
 *    qem_loglik_bernoulli_states, qem_sample_normal), Gamma / Beta Q (qem_sample_gamma,
 *    qem_tables_gamma_poisson, qem_moments_gamma, qem_sample_beta, qem_tables_beta_binomial,
 *    qem_moments_beta), crossed effects (qem_tables_crossed, qem_moments_gaussian), the
 *    non-factorised Q_MP with parent-copy schemes (qem_cols_qmp_gaussian, qem_moments_qmp), the
 *    predictive log-likelihood (qem_backward_resample, qem_predictive_loglik,
 *    qem_logmeanexp) and the global-IW baseline (qem_global_iw).
 *
 * CONVENTIONS (all entry points)
 *  - Plain C types only.  Pointers named d_* are DEVICE pointers owned by the
 *    caller (e.g. torch tensors); h_* are host pointers.  The library never
 *    frees caller memory; it performs no cudaMalloc except inside
 *    qem_create (its own device workspace, freed by qem_destroy; qem_create_in
 *    takes a caller-owned workspace instead).
 *  - `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 *    All device work is stream-ordered; no call synchronises the host except
 *    qem_read_flags and the h_* readbacks documented below.
 *  - Status codes are returned, never thrown.  On error, qem_last_error()
 *    returns a NUL-terminated description (thread-local).
 *  - Numerical conditions never abort: degenerate evidence (all terms -inf),
 *    NaN, and variance clamps are recorded in device flags (qem_read_flags).
 *  - Determinism: identical inputs, launch configuration and world size give
 *    bit-identical outputs (fixed-order reductions, no float atomics).
 *
 * LAYOUTS (row-major, k fastest)
 *  Latent levels: level 0 = root group (1 instance, R dims, one SHARED copy
 *  index, R2); level 1 = groups (two-level: n instances x d dims;
 *  three-level: A top-level groups x 1 dim); level 2 = subgroups (three-level
 *  only: A*B instances x 1 dim, instance ab = a*B + b).
 *   q_mean, q_var   float  [instances*dims]        Q_t (mean, variance)
 *   ema_m1, ema_v   double [instances*dims]        EMA state (E z, Var z)
 *   z               float  [instances][dims][K]    samples
 *   w               float  [instances][K]          marginal weights (out)
 *   m1, v           double [instances*dims]        one-step moments (out)
 *  Root dims: two-level = mu[0..d-1] then s (if scale_kind != FIXED);
 *             three-level = g then beta[0..P-1].
 *  Observations (device, per LOCAL instance):
 *   OBS_GAUSS            x float [n][J]                          (d == 1)
 *   OBS_BERNOULLI_LOGIT  x uint8 [n][J][d] in {0,1}; y uint8 [n][J]
 *   OBS_POISSON_LOG      x float [A*B][J][P];  y int32 [A*B][J]
 */
#ifndef QEM_H_
#define QEM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t qem_status;
#define QEM_OK 0
#define QEM_INVALID_ARGUMENT 1 /* null pointer, size, K or d out of range */
#define QEM_INVALID_MODEL 2    /* model description fails validation */
#define QEM_UNSUPPORTED 3      /* valid but not implemented (e.g. world>1 on three-level) */
#define QEM_CUDA_ERROR 4       /* a CUDA call failed; see qem_last_error() */
#define QEM_NCCL_ERROR 5       /* an NCCL call failed or NCCL cannot be loaded; see qem_last_error() */

#define QEM_FAMILY_TWO_LEVEL 2
#define QEM_FAMILY_THREE_LEVEL 3
#define QEM_SCALE_FIXED 0    /* group prior variance = fixed_var                  */
#define QEM_SCALE_LOGSIGMA 1 /* group prior variance = exp(2 s)  (config 4)       */
#define QEM_SCALE_LOGVAR 2   /* group prior variance = exp(s)    (psi, configs 2,5) */
#define QEM_OBS_GAUSS 1
#define QEM_OBS_BERNOULLI_LOGIT 2
#define QEM_OBS_POISSON_LOG 3

/* Device flag bits (qem_read_flags). */
#define QEM_FLAG_DEGENERATE 1u /* log-evidence is -inf       */
#define QEM_FLAG_NAN 2u        /* a NaN reached a weight or moment          */
#define QEM_FLAG_CLAMP 4u      /* an M-step variance hit the floor (R8)     */

/* Q families of qem_mstep_family (NEXT row f1) and its per-instance status. */
#define QEM_QFAMILY_GAMMA 1       /* mean params (E z, E ln z)          -> (shape k, rate th)   */
#define QEM_QFAMILY_BETA 2        /* mean params (E ln z, E ln(1-z))    -> (a, b)               */
#define QEM_QFAMILY_BERNOULLI 3   /* mean param  E z                    -> p                    */
#define QEM_QFAMILY_CATEGORICAL 4 /* mean params E onehot(z) [C]        -> p [C] (normalised)   */
#define QEM_QFAMILY_DIRICHLET 5   /* mean params E ln z [C]             -> a [C] (C <= 16)      */
#define QEM_QFAMILY_BINOMIAL 6    /* mean param  E z, C = trials N      -> p = E z / N          */
#define QEM_QFAMILY_MULTINOMIAL 7 /* mean params E z [C]                -> p [C] (normalised)   */
#define QEM_EXPFAM_OK 0
#define QEM_EXPFAM_INFEASIBLE 1      /* moments outside the family's mean-parameter space        */
#define QEM_EXPFAM_NO_CONVERGENCE 2  /* the Newton iteration did not reach its tolerance          */

#define QEM_MAX_K 1024
#define QEM_MAX_D 32
/* The two-level family's latent dimensions d with compiled kernels (one translation unit each):
   1-8, 10, 12, 14, 16, 18, 20, 24, 32 (= QEM_MAX_D); any other d is QEM_INVALID_MODEL.  Shared
   memory that grows with d, K and J is checked against the device at context creation. */
#define QEM_D_MENU_STR "1,2,3,4,5,6,7,8,10,12,14,16,18,20,24,32"

/*
 * Plate-structured model description (a fixed menu).
 * Two-level (PAPER.md:1245-1262 Radon-like / 1002-1029 MovieLens-like):
 *   root mu[d] ~ N(prior_mean, prior_var), s ~ N(prior_mean, prior_var) (if scaled)
 *   z_i ~ N(mu, V I), V by scale_kind;   obs by obs_kind (GAUSS: x ~ N(z, obs_var))
 * Three-level (PAPER.md:847-851 nesting):
 *   g, beta[P] ~ N(prior_mean, prior_var); u_a ~ N(g, top_var);
 *   v_ab ~ N(u_a, sub_var); y_abj ~ Poisson(exp(v_ab + beta . x_abj))
 * n = GLOBAL number of level-1 instances; K samples per latent (1..QEM_MAX_K).
 */
typedef struct {
  int32_t family;
  int32_t d;          /* two-level latent dim (1..QEM_MAX_D); 1 for three-level */
  int32_t scale_kind;
  int32_t obs_kind;
  int64_t n;          /* groups (two-level) or top-level groups A (three-level) */
  int32_t n_sub;      /* B (three-level) */
  int32_t n_obs;      /* J observations per group / subgroup */
  int32_t n_cov;      /* P covariates (three-level) */
  int32_t K;
  double fixed_var, obs_var, top_var, sub_var, prior_mean, prior_var;
} qem_model_desc;

/* EMA / M-step options (Eq. 9, Theorem 1, R5, R8). */
typedef struct {
  double new_weight; /* w in (0,1]: m_t = (1-w) m_{t-1} + w m_one  (history lambda = 1-w) */
  double schedule_p; /* if > 0: lambda_t = 1 - t^{-p} (Theorem 1) overrides new_weight   */
  double var_floor;  /* Gaussian M-step variance floor (> 0), default 1e-8              */
  int32_t fresh_denominator; /* 1: fresh-sample denominator (R28):
                                the one-step moments are sum_k r_k(z) m(z^k) / Pe(z_new) for an
                                independent draw z_new, i.e. qem_mstep scales the self-normalised
                                ones by Pe(z)/Pe(z_new) = exp(log_pe - log_pe_fresh).  Needs
                                bufs.log_pe_fresh; two-level family only.  0 (default): Eq. 7a. */
  int32_t reserved;
} qem_opts;

typedef struct {
  float* q_mean;
  float* q_var;
  double* ema_m1;
  double* ema_v;
  float* z;
  float* w;
  double* m1;
  double* v;
} qem_level;

/* Device buffers bound to a context (all caller-owned).  Unused levels may be
   zeroed.  x/y are the observation arrays of the LOCAL shard. */
typedef struct {
  qem_level level[3];
  const void* x;
  const void* y;
  double* log_pe;      /* [1] log Pe of the last E-step (replicated on every rank) */
  double* trace;       /* [trace_len] optional: log Pe of iteration t0+j at [j],
                          written by qem_iterate only (never by the eager calls) */
  int64_t trace_len;
  double* plate_sum;   /* [K+1] optional caller-owned plate-sum / all-reduce buffer;
                          NULL = the context's own (see qem_reduce_buffer)          */
  double* log_pe_fresh; /* [1] log Pe(z_new) of the fresh-denominator pass (qem_estep_evidence);
                          required when opts.fresh_denominator, else may be NULL    */
  const float* eps_bank[3]; /* optional parity mode of qem_iterate: per bound level, host-generated
                          N(0,1) draws [eps_bank_len][instances*dims][K] (fp32, device); iteration
                          t0+j samples with slice j instead of Philox (the fresh-denominator z_new
                          still comes from Philox).  eps_bank[0] == NULL: Philox (default). */
  int64_t eps_bank_len;
} qem_buffers;

typedef struct qem_ctx qem_ctx;

/* Validate a model description.  Returns QEM_OK or QEM_INVALID_MODEL with a
   one-line reason in msg (truncated to cap bytes, always NUL-terminated). */
qem_status qem_model_validate(const qem_model_desc* desc, char* msg, size_t cap);

/* Shard of level-1 instances owned by `rank` of `world`: a contiguous block
   [r*n/world, (r+1)*n/world).  Integer-exact. */
qem_status qem_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end);

/* Create a context for LOCAL level-1 instances [group_begin, group_end) of the
   model (global indices key the Philox counters, so samples do not depend on
   the world size).  world > 1 is supported for the two-level family only.
   Device workspace is allocated here (O(n_local*K) floats) and freed by
   qem_destroy.  opts may be NULL (w=0.3, no schedule, floor 1e-8).
   Errors: QEM_INVALID_MODEL as qem_model_validate; QEM_INVALID_ARGUMENT for an
   empty, reversed or out-of-range block (a rank of a world larger than n owns no
   groups and creates no context) or bad opts; QEM_UNSUPPORTED for a proper
   sub-block of a three-level model; QEM_CUDA_ERROR if the allocation fails. */
qem_status qem_create(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin,
                      int64_t group_end, qem_ctx** out);
/* Caller-owned workspace variant (serving deployments that pool device memory):
   qem_workspace_bytes reports the bytes qem_create_in needs for the same
   (desc, opts, group range) -- host-only arithmetic, no device call except the
   SM-count query that sizes the per-CTA partial buffers; qem_create_in carves
   the context's buffers from d_workspace (device memory, 256-byte aligned,
   >= that many bytes, owned by the caller and not freed by qem_destroy; it
   must outlive the context).  Errors: QEM_INVALID_ARGUMENT on a null pointer,
   misalignment or a short workspace; otherwise as qem_create. */
qem_status qem_workspace_bytes(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin,
                               int64_t group_end, size_t* bytes);
qem_status qem_create_in(const qem_model_desc* desc, const qem_opts* opts, int64_t group_begin,
                         int64_t group_end, void* d_workspace, size_t ws_bytes, qem_ctx** out);
void qem_destroy(qem_ctx* ctx);

/* Bind the caller's device buffers.  Must precede every compute call; may be
   called again to re-bind (invalidates a captured qem_iterate graph). */
qem_status qem_bind(qem_ctx* ctx, const qem_buffers* bufs);

/* K1 -- Q sampler (Alg. 1 line 4 "z ~ Q_t"; location-scale sampling,
   PAPER.md:708-719).  For every bound level: z = fmaf(sqrtf(q_var), eps, q_mean)
   (fp32, R22).  eps comes from d_eps[level] ([instances*dims][K]
   float, host-generated parity mode) when d_eps != NULL and d_eps[level] !=
   NULL, else from Philox4x32-10 keyed by (seed, iter, level, GLOBAL instance,
   dim, k) + Box-Muller. */
qem_status qem_sample_q(qem_ctx* ctx, uint64_t seed, int32_t iter, const float* const* d_eps,
                        void* stream);

/* ---- Group sharding over ranks (PAPER.md:393-394 plate-wise elimination) ----
   One process per GPU; rank r's context owns groups qem_shard_range(n, r, world).  The only
   exchange of a QEM iteration is a SUM all-reduce of the (K+1) fp64 plate sums
   [G_r(0..K-1), sum_i c_i] the local forward leaves in the reduce buffer (qem_reduce_buffer):
   log-sum-exp-safe because the plate product is a plain sum of centred log-messages (Eq. 7c,
   PAPER.md:148), so nothing is exponentiated before the reduction.  Every rank then computes the
   root weights redundantly from the identical reduced bytes (root samples come from Philox keyed
   by global indices: no broadcast).  The library runs that all-reduce itself (ncclAllReduce,
   fp64 SUM, in place, on the call's stream, so qem_iterate captures it in its CUDA graph) once a
   communicator is attached.  NCCL is loaded at run time (the process's libnccl.so.2, e.g. torch's,
   else QEM_NCCL_LIB); processes that attach none never load it.  Two-level family only
   (QEM_UNSUPPORTED for three-level contexts, which run as replicas).

   qem_nccl_unique_id: writes a fresh ncclUniqueId (QEM_NCCL_ID_BYTES bytes) to h_id (host); rank 0
     calls it and the caller distributes the bytes (e.g. over torch.distributed).
   qem_nccl_init: COLLECTIVE over the `world` ranks: ncclCommInitRank(world, id, rank) plus one
     warm-up all-reduce (NCCL connects on its first collective, which must not be captured).  The
     context owns the communicator (destroyed by qem_destroy or a later attach).  Errors:
     QEM_INVALID_ARGUMENT if qem_shard_range(n, rank, world) is not the context's group block;
     QEM_NCCL_ERROR if NCCL fails or cannot be loaded.
   qem_set_nccl_comm: attach a caller-owned ncclComm_t (passed as void*; NULL detaches); its
     (ncclCommUserRank, ncclCommCount) must own the context's group block (else
     QEM_INVALID_ARGUMENT).  Attaching invalidates a captured qem_iterate graph.
   qem_nccl_info: the attached communicator's rank / world (0 / 1 without one) and NCCL version
     (ncclGetVersion code, 0 without one); any output pointer may be NULL.
   qem_estep_reduce: the all-reduce between qem_estep_forward and qem_estep_backward (a no-op on an
     unsharded context without a communicator; QEM_UNSUPPORTED on a sharded one without). */
#define QEM_NCCL_ID_BYTES 128
qem_status qem_nccl_unique_id(void* h_id);
qem_status qem_nccl_init(qem_ctx* ctx, const void* h_id, int32_t rank, int32_t world);
qem_status qem_set_nccl_comm(qem_ctx* ctx, void* nccl_comm);
qem_status qem_nccl_info(const qem_ctx* ctx, int32_t* rank, int32_t* world, int32_t* version);

/* K2..K4 -- one MPIW E-step on the bound samples (Eq. 7a-c):
   log Pe -> bufs.log_pe, weights -> level[*].w, moments (E z, Var z) ->
   level[*].m1 / .v.  = qem_estep_forward + qem_estep_reduce + qem_estep_backward.  A sharded
   context needs a communicator (QEM_UNSUPPORTED otherwise); callers that reduce the plate sums
   themselves use the phases with their own all-reduce of qem_reduce_buffer in between. */
qem_status qem_estep(qem_ctx* ctx, void* stream);
/* Phase 1: sample prep, unary terms, pair-tile forward log-sum-exp; leaves the
   local plate sum [G(0..K-1), sum_i c_i] (fp64) in the reduce buffer. */
qem_status qem_estep_forward(qem_ctx* ctx, void* stream);
/* qem_sample_q (Philox mode, iter >= 1) + qem_estep_forward in one call: on the tensor-core path the
   level-1 draws are made inside the column prep (the same Philox counters and transform as the
   sampler, so the bound z is bit-identical to qem_sample_q's), saving the prep's read of z; other
   paths run the two calls.  qem_iterate uses it unless an eps bank is bound. */
qem_status qem_sample_estep_forward(qem_ctx* ctx, uint64_t seed, int32_t iter, void* stream);
/* Device pointer + count of the plate-sum buffer (fp64, K+1 entries). */
qem_status qem_reduce_buffer(qem_ctx* ctx, double** d_buf, int64_t* count);
/* SUM all-reduce of that buffer over the attached communicator (see "Group sharding" above). */
qem_status qem_estep_reduce(qem_ctx* ctx, void* stream);
/* Phase 2: root softmax + log Pe (from the reduced buffer), backward weights,
   moments. */
qem_status qem_estep_backward(qem_ctx* ctx, void* stream);

/* Fresh-denominator evidence pass: forward + root evidence on the
   currently bound samples (drawn independently of the E-step's: Philox with bit 23 of `iter`
   set, or a second host eps draw), log Pe(z_new) -> bufs.log_pe_fresh.  Weights, moments and
   bufs.log_pe are not touched.  world == 1; sharded runs call qem_estep_forward, all-reduce
   the reduce buffer, then qem_evidence_root.  Two-level family only (else QEM_UNSUPPORTED). */
qem_status qem_estep_evidence(qem_ctx* ctx, void* stream);
qem_status qem_evidence_root(qem_ctx* ctx, void* stream);

/* K5 -- EMA over mean parameters + Gaussian M-step for every bound level
   (Alg. 1 lines 3 and 6; Eq. 9): with lambda = history weight of iteration t,
     m1 <- lam m1 + (1-lam) m1_new
     v  <- lam v + (1-lam) v_new + lam (1-lam) (m1_old - m1_new)^2
   (exactly the EMA of (E z, E z^2), R19), then
     q_mean = (float) m1,  q_var = (float) max(v, var_floor).
   With opts.fresh_denominator the one-step mean parameters (m1_new, v_new + m1_new^2) are
   first multiplied by exp(log_pe - log_pe_fresh) (read on the device).                */
qem_status qem_mstep(qem_ctx* ctx, int32_t t, void* stream);

/* ---- Gamma approximate posteriors (NEXT row f1, E-step side; R32) ----
   Gamma-Poisson hierarchy under a Gaussian root: mu ~ N(0, 1), Q_root = N(m, v) (1-dim root);
   lambda_i | mu ~ Gamma(shape alpha, rate alpha e^-mu); y_ij | lambda_i ~ Poisson(lambda_i);
   Q_i = Gamma(shape k_i, rate th_i).  One QEM iteration = qem_sample_normal (root) +
   qem_sample_gamma + qem_cols_gamma_poisson + qem_estep_separable (or qem_tables_gamma_poisson +
   qem_estep_tables) + qem_moments_gamma + qem_mstep_family(QEM_QFAMILY_GAMMA) for the groups and
   qem_mstep_gaussian for the root.  Device arrays, caller-owned, asynchronous on `stream`; QEM_INVALID_ARGUMENT on bad
   sizes / null arrays. */
/* d_z [n][K] fp64 Gamma(shape, rate) draws, d_q [n][2] = Q_i's (shape, rate) (qem_mstep_family's
   QEM_QFAMILY_GAMMA parameter layout): Marsaglia-Tsang (shape < 1: boosted), attempt
   a of (i, k) from Philox4x32-10 at counter (k, a, i, 6 << 24 | iter), key = seed: normal
   sqrt(-2 ln u0) cos(2 pi u1), acceptance u2, boost u3^(1/shape), u_j = (word_j + 1/2) 2^-32
   (fp64); NaN after 64 rejected attempts.  iter >= 1. */
qem_status qem_sample_gamma(int64_t n, int32_t K, uint64_t seed, int32_t iter, const double* d_q, double* d_z,
                            void* stream);
/* Log-factor tables (fp64): d_f_root [K] = log N(mu^k; 0, 1) - log N(mu^k; m, v) (mu^k =
   d_root_z[k], fp32; d_root_mean/var [1] fp32); d_f [n][K][K] = log Gamma(l; alpha, alpha e^-mu^k)
   + sum_j log Pois(y_ij; l) - log Gamma(l; k_i, th_i), l = d_z[i][k'] (d_y [n][J] int32 counts,
   d_q [n][2] fp64 = Q_i's (shape, rate)).  Feed to qem_estep_tables. */
qem_status qem_tables_gamma_poisson(int64_t n, int32_t K, int32_t J, double alpha, const float* d_root_z,
                                    const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                    const double* d_q, const double* d_z, double* d_f_root, double* d_f,
                                    void* stream);
/* Mean parameters under qem_estep_tables' weights: d_gm [n][2] = (E lambda_i, E ln lambda_i),
   d_root_m [2] = (E mu, E mu^2). */
qem_status qem_moments_gamma(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z,
                             const double* d_w, const double* d_z, double* d_root_m, double* d_gm,
                             void* stream);

/* ---- Beta approximate posteriors (NEXT row f1, E-step side; R32) ----
   Beta-Binomial hierarchy under a Gaussian root: mu ~ N(0, 1), Q_root = N(m, v); p_i | mu ~
   Beta(kappa s, kappa (1 - s)), s = sigmoid(mu); y_i ~ Binomial(N_i, p_i); Q_i = Beta(a_i, b_i).
   One QEM iteration = qem_sample_normal (root) + qem_sample_beta + qem_tables_beta_binomial +
   qem_estep_tables + qem_moments_beta + qem_mstep_family(QEM_QFAMILY_BETA) +
   qem_mstep_categorical(n = 0) for the root.  d_q [n][2] = (a, b) (fp64, the BETA parameter
   layout of qem_mstep_family).
   qem_sample_beta: z = X / (X + Y), X ~ Gamma(a), Y ~ Gamma(b) by Marsaglia-Tsang as
   qem_sample_gamma on the Philox streams 7 << 24 (X) and 8 << 24 (Y).
   qem_tables_beta_binomial: d_f_root [K] as qem_tables_gamma_poisson; d_f [n][K][K] =
   log Beta(p; kappa s_k, kappa (1 - s_k)) + log Binomial(y_i; N_i, p) - log Beta(p; a_i, b_i),
   p = d_z[i][k'], d_y / d_N [n] int32.
   qem_moments_beta: d_gm [n][2] = (E ln p_i, E ln(1 - p_i)), d_root_m [2] = (E mu, E mu^2). */
qem_status qem_sample_beta(int64_t n, int32_t K, uint64_t seed, int32_t iter, const double* d_q, double* d_z,
                           void* stream);
qem_status qem_tables_beta_binomial(int64_t n, int32_t K, double kappa, const float* d_root_z,
                                    const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                    const int32_t* d_N, const double* d_q, const double* d_z, double* d_f_root,
                                    double* d_f, void* stream);
qem_status qem_moments_beta(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z,
                            const double* d_w, const double* d_z, double* d_root_m, double* d_gm, void* stream);

/* ---- Crossed effects (NEXT row f4; R33) ----
   Bus-Breakdown-shaped: root group (shared index k) = (mu, C company weights, T journey-type
   weights), all N(0, 1), samples d_root_z [R][K] fp32 with R = 1 + C + T and Q_root
   d_root_mean / d_root_var [R]; n groups (year x borough) with w_i ~ N(mu, 1), Q_i =
   N(d_q_mean[i], d_q_var[i]), samples d_z [n][K] fp32; J observations per group with company
   index d_comp [n][J] in [0, C), journey type d_jtype [n][J] in [0, T) and label d_y [n][J] in
   {0, 1}: delay ~ Bernoulli(sigmoid(w_i + cw_c + jw_t)).  One QEM iteration = qem_sample_normal
   (root rows, level 0) + qem_sample_normal (group rows, level 1) + qem_tables_crossed +
   qem_estep_tables + qem_moments_gaussian + qem_mstep_gaussian for the root dims and again for the
   group latents.
   qem_tables_crossed: d_f_root [K] = sum_r log N(r^k; 0, 1) - log q(r^k); d_f [n][K][K] =
   log N(w_i^k'; mu^k, 1) + sum_j [y eta - softplus(eta)] - log q_i(w_i^k'),
   eta = w_i^k' + cw^k_{comp_ij} + jw^k_{jtype_ij} (fp64).  J <= 4096.
   qem_moments_gaussian: d_root_m [R][2] = (E r, E r^2) under d_w_root; d_gm [n][2] = (E w_i,
   E w_i^2) under d_w [n][K]. */
qem_status qem_tables_crossed(int64_t n, int32_t K, int32_t J, int32_t C, int32_t T, const float* d_root_z,
                              const float* d_root_mean, const float* d_root_var, const float* d_z,
                              const float* d_q_mean, const float* d_q_var, const int32_t* d_comp,
                              const int32_t* d_jtype, const uint8_t* d_y, double* d_f_root, double* d_f,
                              void* stream);
/* The crossed-effects E-step on chip (no n x K x K table; R37): the factor above is
   evaluated per pair inside the forward (one block per group, online log-sum-exp over k') and again
   inside the backward, fp64 as qem_tables_crossed + qem_estep_tables, same outputs (d_f_root [K],
   d_g [n][K], d_log_pe [1], d_w_root [K], d_w [n][K]).  K <= QEM_MAX_K; K x J row offsets must fit in
   shared memory (else QEM_INVALID_ARGUMENT). */
qem_status qem_estep_crossed(int64_t n, int32_t K, int32_t J, int32_t C, int32_t T, const float* d_root_z,
                             const float* d_root_mean, const float* d_root_var, const float* d_z, const float* d_q_mean,
                             const float* d_q_var, const int32_t* d_comp, const int32_t* d_jtype, const uint8_t* d_y,
                             double* d_f_root, double* d_g, double* d_log_pe, double* d_w_root, double* d_w,
                             void* stream);
qem_status qem_moments_gaussian(int64_t n, int32_t K, int32_t R, const double* d_w_root, const float* d_root_z,
                                const double* d_w, const float* d_z, double* d_root_m, double* d_gm,
                                void* stream);

/* ---- Predictive log-likelihood (NEXT row f3; R31) ----
   qem_backward_resample: after qem_estep (or qem_estep_forward + the all-reduce + the root pass
   of qem_estep_backward) on a two-level context, draw S index tuples from the MPIW posterior
   over index tuples (r_k / sum r, Eq. 7a-c) by ancestral sampling in reverse elimination order:
   k_root ~ w_root, then k_i ~ P_i(k' | k_root) = exp(B_i(k_root,k') + A_i(k') - ln K - g_i(k_root))
   for every LOCAL instance i, by inverse CDF (fp64 prefix in k' order) on 24-bit Philox
   uniforms: word 0 of Philox4x32-10 at counter (s, 0, 0, 5 << 24) for the root and
   (s, 1 + global i, 0, 5 << 24) for instance i, key = seed -- identical across world sizes.
   d_idx_root [S], d_idx [S][n_local] int32 (device, caller-owned).
   qem_predictive_loglik: ll_part[s][i] = sum_j log p(x_test_ij | z_i^{idx[s][i]}) (fp64;
   test data laid out as the training data: Gaussian float [n_local][J_test], Bernoulli
   uint8 x [n_local][J_test][d] + y [n_local][J_test]), d_ll_s[s] = sum_i ll_part[s][i] (local
   instances, fixed order) and, when d_pll != NULL, d_pll = log (1/S) sum_s exp(ll_s) -- valid
   at world == 1; sharded runs SUM-all-reduce d_ll_s and call qem_logmeanexp.  Errors:
   QEM_UNSUPPORTED for the three-level family, QEM_INVALID_ARGUMENT for S < 1 or null arrays. */
qem_status qem_backward_resample(qem_ctx* ctx, int32_t S, uint64_t seed, int32_t* d_idx_root, int32_t* d_idx,
                                 void* stream);
qem_status qem_predictive_loglik(qem_ctx* ctx, int32_t S, const int32_t* d_idx, int32_t J_test,
                                 const void* d_x_test, const uint8_t* d_y_test, double* d_ll_part,
                                 double* d_ll_s, double* d_pll, void* stream);
/* Global importance weighting (App. A, Eq. glob_iw; the baseline MPIW improves
   on): after qem_estep_forward on a world-1 two-level context, the K joint draws with every
   latent at the same index k: d_diag [n][K] = B_i(k, z_i^k) + A_i(z_i^k) (fp64),
   d_log_pe [1] = lse_k (f_root(k) + sum_i d_diag[i][k]) - ln K, d_w [K] = the normalised
   weights, and (when d_m1 != NULL) d_m1 [n][d] = sum_k w_k z_i^k.  d_scratch: >= n*K doubles.
   QEM_UNSUPPORTED for the three-level family or a sharded context. */
qem_status qem_global_iw(qem_ctx* ctx, double* d_diag, double* d_scratch, double* d_log_pe, double* d_w,
                         double* d_m1, void* stream);
/* d_out[0] = log (1/n) sum_i exp(d_x[i]) (fp64, fixed order), n >= 1. */
qem_status qem_logmeanexp(int64_t n, const double* d_x, double* d_out, void* stream);

/* ---- Discrete latents under a continuous root (NEXT row f1, E-step side; R30) ----
   Occupancy-shaped model: root r in R^d, prior N(0, I), Q_root =
   N(m, diag v); per instance i a categorical z_i in {0..C-1}, prior logits eta_ic(r) = x_ic . r,
   Q_i = Categorical(p_i), observations through the per-state log-likelihood table
   L_i(c) = log p(y_i | z_i = c).  One QEM iteration = qem_sample_normal (root) +
   qem_sample_categorical + qem_tables_categorical + qem_estep_tables +
   qem_moments_categorical + qem_mstep_categorical.  All arrays device-resident and caller-owned; calls are asynchronous on `stream`;
   QEM_INVALID_ARGUMENT on bad sizes / null arrays. */
#define QEM_CAT_MAX_C 8

/* Gaussian samples z[row][k] = fmaf(sqrtf(var[row]), eps, mean[row]) (fp32, R22) for `rows`
   latent rows: eps from d_eps [rows][K] when non-NULL, else Philox4x32-10 at counter
   (k/4, 0, row, level << 24 | iter) + Box-Muller, as qem_sample_q.  iter >= 1, 0 <= level < 256. */
qem_status qem_sample_normal(int64_t rows, int32_t K, int32_t level, uint64_t seed, int32_t iter,
                             const float* d_mean, const float* d_var, const float* d_eps, float* d_z,
                             void* stream);
/* Categorical samples z[i][k] in [0, C): the smallest c with u < p_i(0) + ... + p_i(c) (fp64
   sequential prefix; C-1 if none), u = ((w >> 8) + 1/2) 2^-24 from word k%4 of Philox4x32-10 at
   counter (k/4, 0, i, 3 << 24 | iter), key = seed.  d_p [n][C] fp64 (rows summing to 1),
   d_z [n][K] int32.  1 <= C <= QEM_CAT_MAX_C, iter >= 1. */
qem_status qem_sample_categorical(int64_t n, int32_t C, int32_t K, uint64_t seed, int32_t iter,
                                  const double* d_p, int32_t* d_z, void* stream);
/* Log-factor tables of the model above (fp64):
     d_f_root [K]      log N(r^k; 0, I) - log q(r^k)          (r^k = d_root_z[.][k], fp32 [d][K])
     d_f [n][K][K]     log softmax_c(x_i . r^k)[z_i^k'] + L_i(z_i^k') - log p_i(z_i^k')
   d_root_mean/var [d] fp32 (Q_root), d_x [n][C][d], d_loglik [n][C], d_p [n][C] fp64,
   d_z [n][K] int32.  Feed d_f_root / d_f to qem_estep_tables. */
qem_status qem_tables_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const double* d_x,
                                  const double* d_loglik, const double* d_p, const int32_t* d_z,
                                  double* d_f_root, double* d_f, void* stream);
/* The same E-step without materialising the tables (O(n K C) instead of O(n K^2)): f_i(k,k')
   depends on k' only through the state z_i^k', so with n_i(c) = #{k' : z_i^k' = c},
   g_i(k) = log sum_c n_i(c) exp(h_i(k,c)) - ln K and w_i(k') = W_i(z_i^k'), W_i(c) =
   sum_k w_root(k) exp(h_i(k,c) - ln K - g_i(k)), h_i(k,c) the table entry of state c.  Outputs
   as qem_tables_categorical + qem_estep_tables (d_f_root [K], d_g [n][K], d_log_pe [1],
   d_w_root [K], d_w [n][K]; d_w doubles as the plate-sum scratch).  K <= QEM_TABLES_MAX_K. */
qem_status qem_estep_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const float* d_root_z,
                                 const float* d_root_mean, const float* d_root_var, const double* d_x,
                                 const double* d_loglik, const double* d_p, const int32_t* d_z,
                                 double* d_f_root, double* d_g, double* d_log_pe, double* d_w_root,
                                 double* d_w, void* stream);
/* Moments (Eq. 7a) from qem_estep_tables' weights: d_root_m [d][2] = (E r_e, E r_e^2) under
   d_w_root [K]; d_pm [n][C] = E onehot(z_i) = sum_k' w_i(k') [z_i^k' = c] under d_w [n][K]. */
qem_status qem_moments_categorical(int64_t n, int32_t C, int32_t K, int32_t d, const double* d_w_root,
                                   const float* d_root_z, const double* d_w, const int32_t* d_z,
                                   double* d_root_m, double* d_pm, void* stream);
/* EMA over mean parameters (history weight lam in [0, 1), Eq. 9 / DESIGN.md R5) + M-step:
   root  d_root_ema [d][2] <- lam ema + (1-lam) d_root_m;  Q_root mean = E r, var =
         max(E r^2 - (E r)^2, var_floor), written fp32 to d_root_mean / d_root_var (R22);
   inst  d_p_ema [n][C] <- lam ema + (1-lam) d_pm;  d_p = d_p_ema / sum_c d_p_ema (fp64).
   Variance-floor clamps are added to *d_clamps (int64, device) when non-NULL. */
qem_status qem_mstep_categorical(int64_t n, int32_t C, int32_t d, double lam, double var_floor,
                                 const double* d_root_m, double* d_root_ema, float* d_root_mean,
                                 float* d_root_var, const double* d_pm, double* d_p_ema, double* d_p,
                                 int64_t* d_clamps, void* stream);
/* EMA + Gaussian M-step of `rows` Gaussian latent dimensions (the root groups of the NEXT-row models,
   the crossed effects' group latents): d_ema [rows][2] <- lam d_ema + (1 - lam) d_m, both holding the
   mean parameters (E z, E z^2) (Eq. 9); then mean = E z, var = max(E z^2 - (E z)^2, var_floor) written
   fp32 to d_mean / d_var (R22); variance-floor clamps added to *d_clamps when non-NULL.  The same
   kernel as qem_mstep_categorical's root part, under its own name. */
qem_status qem_mstep_gaussian(int64_t rows, double lam, double var_floor, const double* d_m, double* d_ema,
                              float* d_mean, float* d_var, int64_t* d_clamps, void* stream);
/* History weight lambda of iteration t (R5): 1 - new_weight, or 1 - t^-p when
   schedule_p > 0 (Theorem 1) -- the value k_mstep uses; host arithmetic. */
double qem_history_weight(int32_t t, double new_weight, double schedule_p);

/* Per-state log-likelihood of R Bernoulli observations per instance (the data table L of
   qem_tables_categorical): d_L[i][c] = sum_r y_ir l_irc - softplus(l_irc), softplus(l) =
   max(l, 0) + log1p(exp(-|l|)) (fp64); d_y [n][R] uint8 in {0,1}, d_logit [n][R][C] fp64. */
qem_status qem_loglik_bernoulli_states(int64_t n, int32_t C, int32_t R, const uint8_t* d_y,
                                       const double* d_logit, double* d_L, void* stream);

/* MPIW E-step on EXPLICIT log-factor tables (Eq. 7a-c; plate elimination,
   PAPER.md:393) for a root with K samples and n plate instances below it:
     d_f_root [K]        f_root(k)   = log p(root^k) - log q(root^k)
     d_f      [n][K][K]  f_i(k, k')  = log p(z_i^k', x_i | root^k) - log q(z_i^k')  (k' fastest)
   Outputs (device, fp64, caller-owned): d_g [n][K] messages g_i(k) = lse_k' f_i(k,k') - ln K;
   d_log_pe [1] = lse_k (f_root(k) + sum_i g_i(k)) - ln K; d_w_root [K] root weights;
   d_w [n][K] per-instance marginal weights w_i(k') (each row sums to 1; also the scratch of the plate
   sum before the backward writes it).  Any factor kind the
   caller can tabulate runs here (discrete latents, crossed effects); it also pins the reduction
   of the fused kernels independently of their factor arithmetic.  Degenerate evidence (every
   root sample at -inf) gives log Pe = -inf and NaN weights, as data.  n may be 0 (d_f, d_g, d_w
   then unused).  Errors: QEM_INVALID_ARGUMENT for n < 0, K outside [1, QEM_TABLES_MAX_K] or a
   null array.  Asynchronous on `stream`. */
#define QEM_TABLES_MAX_K 8192
qem_status qem_estep_tables(int64_t n, int32_t K, const double* d_f_root, const double* d_f, double* d_g,
                            double* d_log_pe, double* d_w_root, double* d_w, void* stream);

/* The same E-step for SEPARABLE log-factors, without the n x K x K table (north star: the N K^2
   tensor is never materialised in HBM; NEXT rows f1 / f4, R37):
     f_i(k, k') = a_k + sum_{r<R} b_k[r] phi_i(k')[r] + psi_i(k'),   0 <= R <= 3
     d_rows [K][1 + R]   (a_k, b_k[0..R-1])                     fp64, device
     d_cols [n][K][R + 1] (phi_i(k')[0..R-1], psi_i(k'))         fp64, device
   Each group's columns are staged in shared memory and every pair is evaluated on chip (fp64),
   once for the forward and once for the backward.  Outputs, scratch use and degenerate-evidence
   behaviour as qem_estep_tables.  Errors: QEM_INVALID_ARGUMENT for n < 0, K outside [1, QEM_MAX_K],
   R outside [0, 3] or a null array. */
qem_status qem_estep_separable(int64_t n, int32_t K, int32_t R, const double* d_f_root, const double* d_rows,
                               const double* d_cols, double* d_g, double* d_log_pe, double* d_w_root, double* d_w,
                               void* stream);
/* Separable factors of the Gamma-Poisson model (R = 1: rows [K][2], columns [n][K][2]; the same
   densities as qem_tables_gamma_poisson) and of the Beta-Binomial model (R = 2: rows [K][3],
   columns [n][K][3]; as qem_tables_beta_binomial), plus d_f_root [K]. */
qem_status qem_cols_gamma_poisson(int64_t n, int32_t K, int32_t J, double alpha, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                  const double* d_q, const double* d_z, double* d_f_root, double* d_rows,
                                  double* d_cols, void* stream);
qem_status qem_cols_beta_binomial(int64_t n, int32_t K, double kappa, const float* d_root_z,
                                  const float* d_root_mean, const float* d_root_var, const int32_t* d_y,
                                  const int32_t* d_N, const double* d_q, const double* d_z, double* d_f_root,
                                  double* d_rows, double* d_cols, void* stream);

/* ---- Non-factorised Q_MP with parent-copy schemes (App. A; NEXT row f4; R43) ----
   Conjugate two-level Gaussian hierarchy mu ~ N(0, prior_var), z_i | mu ~ N(mu, group_var),
   x_ij | z_i ~ N(z_i, obs_var) with a proposal whose child depends on its parent:
   Q(mu) = N(d_root_mean[0], d_root_var[0]), Q(z_i | mu) = N(alpha_i + beta_i mu, s_i),
   d_q [n][3] = (alpha_i, beta_i, s_i > 0) fp64.  qem_cols_qmp_gaussian draws the child copies
     d_z[i][k'] = alpha_i + beta_i mu^c + sqrt(s_i) d_eps[i][k'],  c = d_copy[i][k'] in [0, K)
   (mu^k = d_root_z[k] fp32; d_eps [n][K] fp32 standard normals, e.g. qem_sample_normal with mean 0,
   variance 1; d_copy [n][K] int32, drawn by the caller: a uniformly random permutation per group
   for QEM_QMP_PERMUTATION -- the scheme the paper used, PAPER.md:479 --, iid uniform indices for
   QEM_QMP_MIXTURE) and writes the separable factors of
     f_i(k, k') = log N(z_i^k'; mu^k, group_var) + sum_j log N(x_ij; z_i^k', obs_var) - log q_MP,i(k'),
     q_MP,i(k') = N(z_i^k'; alpha_i + beta_i mu^c, s_i)                    (permutation)
                = (1/K) sum_k N(z_i^k'; alpha_i + beta_i mu^k, s_i)        (mixture)
   as d_rows [K][2] = (a_k, b_k), d_cols [n][K][2] = (z_i^k', psi_i(k')) for qem_estep_separable
   (R = 1), plus d_f_root [K] = log N(mu^k; 0, prior_var) - log q(mu^k); d_x [n][J] fp32.  fp64.
   qem_moments_qmp: d_gm [n][2] = (E z_i, E z_i^2) under d_w [n][K], d_root_m [2] = (E mu, E mu^2)
   under d_w_root [K].  beta_i = 0 is the factorised Q of the hot path.  Device arrays,
   caller-owned, asynchronous on `stream`; QEM_INVALID_ARGUMENT on bad sizes, a bad scheme, a
   non-positive variance or a null array (indices in d_copy are not range-checked). */
#define QEM_QMP_PERMUTATION 0
#define QEM_QMP_MIXTURE 1
qem_status qem_cols_qmp_gaussian(int64_t n, int32_t K, int32_t J, int32_t scheme, double prior_var, double group_var,
                                 double obs_var, const float* d_root_z, const float* d_root_mean,
                                 const float* d_root_var, const double* d_q, const int32_t* d_copy, const float* d_eps,
                                 const float* d_x, double* d_z, double* d_f_root, double* d_rows, double* d_cols,
                                 void* stream);
qem_status qem_moments_qmp(int64_t n, int32_t K, const double* d_w_root, const float* d_root_z, const double* d_w,
                           const double* d_z, double* d_root_m, double* d_gm, void* stream);

/* EMA over mean parameters + M-step for non-Gaussian Q families (Alg. 1 lines 3, 6; Eq. 9;
   PAPER.md:218 "a Beta's parameters are recovered from expectations of log transformations",
   PAPER.md:247).  Context-free, stream-ordered, one device thread per latent instance, fp64.
   S = 2 (Gamma, Beta), 1 (Bernoulli, Binomial with C = trials), C (Categorical, Dirichlet,
   Multinomial) mean parameters per instance (PAPER.md:10's list of families):
     d_m_new  [n][S]  one-step mean parameters (input)
     d_m_ema  [n][S]  EMA state, updated in place: m <- lam m + (1 - lam) m_new
     d_params [n][S]  conventional parameters of the updated state (output): Gamma (k, th) by
                      Newton on psi(k) - ln k = m2 - ln m1, th = k/m1; Beta (a, b) by damped
                      2-d Newton in (ln a, ln b); Dirichlet a by Newton with a Sherman-Morrison
                      Hessian; Bernoulli p; Binomial p = m/N; Categorical / Multinomial p normalised
     d_status [n]     QEM_EXPFAM_* per instance (nullable)
   Errors: QEM_INVALID_ARGUMENT for a bad family / n < 0 / C < 1 / null arrays. */
qem_status qem_mstep_family(int32_t family, int64_t n, int32_t C, double lam, const double* d_m_new,
                            double* d_m_ema, double* d_params, int32_t* d_status, void* stream);

/* K6 -- T QEM iterations t = t0 .. t0+T-1 of sample (Philox, seed) ->
   E-step (forward, all-reduce over the attached communicator, backward) -> M-step, replayed
   from one captured CUDA graph, or issued eagerly when `use_graph` == 0.  A sharded context
   needs a communicator (QEM_UNSUPPORTED otherwise) and every rank calls qem_iterate with the
   same (t0, T, seed, use_graph): each iteration is one collective.  With bufs.eps_bank bound the
   samples come from the bank (QEM_INVALID_ARGUMENT if T > bufs.eps_bank_len).  With opts.fresh_denominator each
   iteration first samples z_new (Philox iteration word t | 2^23) and runs the
   evidence pass.  log Pe of iteration t0+j goes to
   bufs.trace[j] when bufs.trace != NULL. */
qem_status qem_iterate(qem_ctx* ctx, int32_t t0, int32_t T, uint64_t seed, int32_t use_graph,
                       void* stream);

/* Synchronises `stream` and returns the OR of all device flags since the last
   call (then clears them), and the number of M-step variance clamps. */
qem_status qem_read_flags(qem_ctx* ctx, void* stream, uint32_t* flags, int64_t* clamps);

/* Synchronises `stream`, copies the forward tile-mode histogram (counts of
   (CTA-warp, group) tiles evaluated in mode 0..6: 0-4 expm1 polynomial of
   degree 3/4/5/7/9, 5 online log-sum-exp; slot 6: groups whose FFMA backward ran through the
   d = 1 moment tiles (k_backward_mom1), 0 elsewhere; slot 7: tensor-core forward 64-column
   chunks (per warp) whose max-free pass came near fp32 overflow and were redone with the exact
   row max) into h_hist[8] and clears it.  Two-level only;
   diagnostics. */
qem_status qem_read_mode_hist(qem_ctx* ctx, void* stream, uint64_t* h_hist);

/* Optional cudaEvent_t handles (as void*, NULL = off) that the library
   records on the launch stream immediately before/after the two-level
   pair-tile kernels (forward K2b, backward K4) of every later E-step, so a
   caller can time exactly those kernels.  The events are caller-owned.  A captured qem_iterate
   graph is discarded (it recorded the previous events). */
qem_status qem_set_kernel_events(qem_ctx* ctx, void* fwd_start, void* fwd_end, void* bwd_start, void* bwd_end);

/* Number of kernels the last qem_* call launched (for the bench's
   gpu_launches claim). */
int64_t qem_kernel_launches(const qem_ctx* ctx);

/* Which pair-tile kernels this context runs (fixed at qem_create):
   0 = FP32 FFMA/SFU tiles (k_forward / k_backward, every d);
   1 = tcgen05 tensor-core tiles (k_forward_tc / k_backward_tc: d = 16,
       Bernoulli-logit observations, K % 256 == 0; the K x K x d cross term
       c_k . u_k' on the tensor cores in bf16x3).
   The bench uses it to name the binding pipe of its roofline.  -1 on NULL. */
int32_t qem_pair_path(const qem_ctx* ctx);

/* Copy the per-group reference-differenced messages Delta g_i(k)
   (float [n_local][K]) and per-group constants c_i (double [n_local]) of the
   last forward pass into caller buffers (stream-ordered D2D copies):
   g_i(k) = c_i + Delta g_i(k) = log (1/K) sum_k' exp(B_i(k,k') + A_i(k'))
   (DESIGN.md "Forward").  For sampled full-size parity checks; two-level only. */
qem_status qem_copy_messages(qem_ctx* ctx, float* d_dg, double* d_c, void* stream);

const char* qem_status_str(qem_status s);
const char* qem_last_error(void);
const char* qem_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QEM_H_ */
