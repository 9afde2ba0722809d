// qem_two_level.cuh -- MPIW E-step kernels for two-level plate models (root
// group -> n groups), sm_100a.  Configs 1, 2, 4, 5.  Templated on the latent dimension D; each
// D of the compiled menu is instantiated in its own translation unit (qem_tl_d<D>.cu, built in
// parallel) and qem_two_level.cu dispatches on the runtime d.
//
// Math (DESIGN.md "Forward" / "Backward"; Eq. 7a-c):
//   B_i(k,k') = log N(z_i^{k'}; mu^k, V^k I)             (parent->child factor)
//   A_i(k')   = sum_j log p(x_ij | z_i^{k'}) - log q(z_i^{k'})  (unary, fp64)
//   g_i(k)    = log (1/K) sum_k' exp(B_i(k,k') + A_i(k'))       (plate message)
// evaluated reference-differenced around one root sample k_ref:
//   t_i(k')   = B_i(k_ref,k') + A_i(k')  (fp64),  P_i = softmax(t_i),
//   c_i       = lse(t_i) - log K  = g_i(k_ref),
//   D_k(k')   = B(k,k') - B(k_ref,k') = alpha_k + gamma_k |u|^2 + c_k . u,
//               u = z - mu_ref   (coefficients differenced in fp64, H1)
//   dg_i(k)   = g_i(k) - c_i = log sum_k' P_i(k') exp(D_k(k'))
//             = log1p(sum_k' P_i(k') expm1(D_k(k')))   (small |D|: FMA-pipe polynomial)
// Root:  a(k) = f_root(k) + sum_i dg_i(k);  log Pe = sum_i c_i + lse(a) - log K.
// Backward: w_i(k') = sum_k w_root(k) exp(ln P_i(k') + D_k(k') - dg_i(k)).
#pragma once
#include <cstdio>
#include <cstdlib>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

struct TLArgs {
  int K, J, scale_kind;
  int64_t n_local;
  double fixed_var, obs_var, prior_mean, prior_var;
  const float* z_root;
  const float* qr_m;
  const float* qr_v;
  const float* z;
  const float* q_m;
  const float* q_v;
  const void* x;
  const void* y;
  float* w_root;
  double* m1_root;
  double* v_root;
  float* w;
  double* m1;
  double* v;
  double* log_pe;
  double* trace;
  int64_t trace_len;
  int t_host;
  int tc;        // tensor-core pair kernels in use (d = 16)
  int evidence_only;  // k_root: log Pe only (fresh-denominator pass)
  int prep_split;     // k_colprep_tc: warps per group (1, 2, 4, 8)
  int fuse_sample;    // k_colprep_tc draws the level-1 samples itself (qem_sample_estep_forward, qem_iterate)
  int t_sample;       // its iteration (0: the device counter, graph mode)
  uint2 skey;         // its Philox key (the seed)
  int64_t g_begin;    // global index of local group 0 (the Philox counters)
  float thr[5];  // forward tile-mode bounds for expm1 degrees 3/4/5/7/9
  float redo_thr;  // tensor-core forward: a max-free chunk whose running sum passes this is redone exactly (R41)
  TwoLevelWs ws;
  Counters* cnt;
};

// --------------------------------------------------------------- root prep
// One block.  Chooses k_ref (root sample nearest Q_root's mean in the
// Q-metric; ties -> lowest k), builds the differenced row coefficients
// (fp64 -> fp32) and the root factor f_root(k) = log p(root^k) - log q(root^k).
// phase 0: everything in one block (FFMA path: the rank sort needs every row key);
// phase 1: k_ref and RefInfo only; phase 2: the rows, split over blocks (tensor-core path, after
// phase 1 -- the row work is store-bound on one SM's LSU).
template <int D>
__global__ void __launch_bounds__(1024) k_root_prep(TLArgs a, int phase) {
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ double s_lnv_ref;
  __shared__ double s_qc[2 * (QEM_MAX_D + 1)];
  __shared__ float s_key[QEM_MAX_K];
  const int K = a.K, tid = threadIdx.x;
  const int R = D + (a.scale_kind != QEM_SCALE_FIXED);
  if (phase <= 1)  // the forward's plate-sum accumulators (Fx2 parts, added atomically by its CTAs)
    for (int k = tid; k < 2 * (K + 1); k += blockDim.x) a.ws.partial[k] = 0.0;
  if (phase == 2) {  // k_ref from phase 1
    if (tid == 0) {
      const int kr = a.ws.ref->k_ref;
      s_lnv_ref = a.scale_kind == QEM_SCALE_FIXED    ? log(a.fixed_var)
                  : a.scale_kind == QEM_SCALE_LOGSIGMA ? 2.0 * (double)a.z_root[D * K + kr]
                                                       : (double)a.z_root[D * K + kr];
    }
  } else {
  // k_ref = argmin_k sum_r (z_r^k - m_r)^2 / v_r
  double best = CUDART_INF;
  int bidx = 0x7fffffff;
  for (int k = tid; k < K; k += blockDim.x) {
    // all R loads in flight before the arithmetic (a dependent load per dimension costs ~1 us)
    float zr[D + 1], qm[D + 1], qv[D + 1];
#pragma unroll
    for (int r = 0; r < D + 1; ++r) {
      zr[r] = r < R ? a.z_root[r * K + k] : 0.f;
      qm[r] = r < R ? a.qr_m[r] : 0.f;
      qv[r] = r < R ? a.qr_v[r] : 1.f;
    }
    double q = 0.0;
#pragma unroll
    for (int r = 0; r < D + 1; ++r) {
      if (r < R) {
        const double dz = (double)zr[r] - (double)qm[r];
        q += dz * dz / (double)qv[r];
      }
    }
    if (q < best || (q == best && k < bidx)) {
      best = q;
      bidx = k;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov < best || (ov == best && oi < bidx)) {
      best = ov;
      bidx = oi;
    }
  }
  if ((tid & 31) == 0) {
    s_val[tid >> 5] = best;
    s_idx[tid >> 5] = bidx;
  }
  __syncthreads();
  if (tid == 0) {
    double bv = s_val[0];
    int bi = s_idx[0];
    for (int w = 1; w < (int)((blockDim.x + 31) >> 5); ++w)
      if (s_val[w] < bv || (s_val[w] == bv && s_idx[w] < bi)) {
        bv = s_val[w];
        bi = s_idx[w];
      }
    if (bi >= K) bi = 0;  // every distance NaN (degenerate Q, flagged by the M-step): stay in range
    RefInfo* ref = a.ws.ref;
    ref->k_ref = bi;
    float mu[D];  // loads before stores (see phase 2)
#pragma unroll
    for (int r = 0; r < D; ++r) mu[r] = a.z_root[r * K + bi];
#pragma unroll
    for (int r = 0; r < D; ++r) ref->mu_ref[r] = mu[r];
    double lnv;
    if (a.scale_kind == QEM_SCALE_FIXED)
      lnv = log(a.fixed_var);
    else if (a.scale_kind == QEM_SCALE_LOGSIGMA)
      lnv = 2.0 * (double)a.z_root[D * K + bi];
    else
      lnv = (double)a.z_root[D * K + bi];
    s_lnv_ref = lnv;
    ref->e_ref = exp(-lnv);
    ref->bref_const = -0.5 * D * (kLn2Pi + lnv);
  }
  if (phase == 1) return;
  }
  // per-dimension constants of f_root: -(ln prior_var - ln v_r)/2 and 1/v_r
  for (int r = tid; r < R; r += blockDim.x) {
    s_qc[r] = -0.5 * (log(a.prior_var) - log((double)a.qr_v[r]));
    s_qc[QEM_MAX_D + 1 + r] = 1.0 / (double)a.qr_v[r];
  }
  __syncthreads();
  const int kref = a.ws.ref->k_ref;
  const double lnv_ref = s_lnv_ref;
  const double e_ref = exp(-lnv_ref);
  constexpr int CW = D + 2;
  constexpr int RS = pad4(D + 3);
  for (int k = blockIdx.x * blockDim.x + tid; k < K; k += gridDim.x * blockDim.x) {
    double lnv, dlnv;
    if (a.scale_kind == QEM_SCALE_FIXED) {
      lnv = lnv_ref;
      dlnv = 0.0;
    } else if (a.scale_kind == QEM_SCALE_LOGSIGMA) {
      lnv = 2.0 * (double)a.z_root[D * K + k];
      dlnv = 2.0 * ((double)a.z_root[D * K + k] - (double)a.z_root[D * K + kref]);
    } else {
      lnv = (double)a.z_root[D * K + k];
      dlnv = (double)a.z_root[D * K + k] - (double)a.z_root[D * K + kref];
    }
    const double ek = exp(-lnv);
    double dd = 0.0;
    float* fc = a.ws.fwd_coef + (size_t)k * CW;
    float* bt = a.ws.bwd_table + (size_t)k * RS;
    double alpha;
    // u = z - mu_ref differenced rows D_k = alpha_k + gamma_k |u|^2 + c_k . u (both pair paths; the
    // tensor-core columns carry S = |w|^2 + 2 u0_i . w with u0_i = m_i - mu_ref, so the fp32 rounding
    // of c_k multiplies u, not z: it averages out over the groups instead of adding up coherently)
    // every load before the first store (the stores could alias z_root: interleaved, each dimension
    // would wait for a round trip -- ~12 us per launch at d = 16)
    float zkr[D], zrr[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      zkr[r] = a.z_root[r * K + k];
      zrr[r] = a.z_root[r * K + kref];
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double del = (double)zkr[r] - (double)zrr[r];
      dd += del * del;
      const double cr = ek * del;
      fc[2 + r] = (float)cr;
      bt[2 + r] = (float)(cr * kLog2eD);
    }
    alpha = -0.5 * D * dlnv - 0.5 * ek * dd;
    const double gamma = -0.5 * (ek - e_ref);
    fc[0] = (float)alpha;
    fc[1] = (float)gamma;
    a.ws.alpha_d[k] = alpha;
    bt[0] = (float)(alpha * kLog2eD);
    bt[1] = (float)(gamma * kLog2eD);
    if (a.tc) {
      // the tensor-core rows are these log2e-scaled fp32 values (one rounding from fp64, k_rowop_tc);
      // the aux merge's alpha'_ik uses exactly the same coefficients back in natural units (fp64), so
      // the MMA and the merge see one row function: a mismatch here (a second rounding of c log2e)
      // would be a fixed per-row error times the group's E_P[w] -- coherent over the groups
      double* cd = a.ws.coef_d + (size_t)k * (D + 1);
      cd[0] = (double)bt[1] * kLn2D;
#pragma unroll
      for (int r = 0; r < D; ++r) cd[1 + r] = (double)bt[2 + r] * kLn2D;
    }
    // f_root(k) = sum_r lnN(z_r; prior) - lnN(z_r; Q_root), the log-normalisers hoisted (s_qc)
    double f = 0.0;
    float zk[D + 1], qmk[D + 1];
#pragma unroll
    for (int r = 0; r < D + 1; ++r) {
      zk[r] = r < R ? a.z_root[r * K + k] : 0.f;
      qmk[r] = r < R ? a.qr_m[r] : 0.f;
    }
    const double ipv = 1.0 / a.prior_var;
#pragma unroll
    for (int r = 0; r < D + 1; ++r) {
      if (r < R) {
        const double v = (double)zk[r];
        const double dp = v - a.prior_mean, dq = v - (double)qmk[r];
        f += s_qc[r] - 0.5 * dp * dp * ipv + 0.5 * dq * dq * s_qc[QEM_MAX_D + 1 + r];
      }
    }
    a.ws.f_root[k] = f;
    // sort key: |D| bound at unit column scale
    float cn = 0.f;
    for (int r = 0; r < D; ++r) cn = fmaf(fc[2 + r], fc[2 + r], cn);
    s_key[k] = fabsf(fc[0]) + fabsf(fc[1]) + sqrtf(cn);
  }
  __syncthreads();
  if (a.tc || phase != 0) return;  // the tensor-core forward does not use the row order
  // rank sort (ties by index): perm[rank] = k
  for (int k = tid; k < K; k += blockDim.x) {
    const float kk = s_key[k];
    int rank = 0;
    for (int j = 0; j < K; ++j) {
      const float kj = s_key[j];
      rank += (kj < kk || (kj == kk && j < k)) ? 1 : 0;
    }
    a.ws.perm[rank] = k;
  }
}

// ------------------------------------------------------------ forward (K2)

__host__ __device__ constexpr double inv_fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return 1.0 / f;
}

// expm1(x) by its Taylor polynomial of degree N (Horner, FMA pipe).
template <int N>
__device__ __forceinline__ float2 expm1_poly(float2 x) {
  float2 p = f2((float)inv_fact(N));
#pragma unroll
  for (int n = N - 1; n >= 1; --n) p = fma2(p, x, f2((float)inv_fact(n)));
  return mul2(p, x);
}

// FFMA backward: rows of every kBwdUnroll whose exponentials run on the FMA pipe (exp2_poly2) instead
// of the SFU.  Narrow latents (d <= 4) take 1 of 8 (config 4, interleaved A/B: 0 1.567, 1/8 1.467,
// 2/8 1.623, 1/16 1.498, 3/16 1.529, 1/12 1.485 ms per backward); wide ones none.  QEM_BWD_SOFT
// overrides.
#ifndef QEM_BWD_UNROLL
#define QEM_BWD_UNROLL 8
#endif
constexpr int kBwdUnroll = QEM_BWD_UNROLL;
template <int D>
__host__ __device__ constexpr int bwd_soft() {
#ifdef QEM_BWD_SOFT
  return QEM_BWD_SOFT;
#else
  return D <= 4 ? 1 : 0;
#endif
}

#include "qem_forward.cuh"
#include "qem_tc.cuh"

// -------------------------------------------------------------- root (K3)
// One block: w_root = softmax(f_root + G), log Pe, root moments.
template <int D>
__global__ void __launch_bounds__(1024) k_root(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* wsh = reinterpret_cast<double*>(smem);  // [K]
  double* scratch = wsh + a.K;                    // [32]
  const int K = a.K, tid = threadIdx.x;
  const int R = D + (a.scale_kind != QEM_SCALE_FIXED);
  constexpr int RS = pad4(D + 3);
  if (tid == 0) a.cnt->claim_bwd = 0;  // the FFMA backward's group queue (stream-ordered before it)
  double mx = -CUDART_INF;
  for (int k = tid; k < K; k += blockDim.x) {
    const double av = a.ws.f_root[k] + a.ws.red[k];
    wsh[k] = av;
    mx = fmax(mx, av);
  }
  const double M = block_max(mx, scratch);
  double s = 0.0;
  for (int k = tid; k < K; k += blockDim.x) s += exp(wsh[k] - M);
  const double S = block_sum(s, scratch);
  const double L = M + log(S);
  const bool degenerate = !(L > -CUDART_INF) || isnan(L);
  if (a.evidence_only) {  // fresh-denominator pass: log Pe(z_new) only
    if (tid == 0) {
      *a.log_pe = a.ws.red[K] + L - log((double)K);
      if (degenerate) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_DEGENERATE);
      if (isnan(L)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
    }
    return;
  }
  for (int k = tid; k < K; k += blockDim.x) {
    const double w = exp(wsh[k] - L);
    wsh[k] = w;
    a.w_root[k] = (float)w;
    a.ws.bwd_table[(size_t)k * RS + 2 + D] = (float)w;
  }
  if (tid == 0) {
    const double lp = a.ws.red[K] + L - log((double)K);
    *a.log_pe = lp;
    if (a.trace) {
      const int t = resolve_iter(a.t_host, &a.cnt->iter);
      const int64_t j = (int64_t)t - a.cnt->trace_base;
      if (j >= 0 && j < a.trace_len) a.trace[j] = lp;
    }
    if (degenerate) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_DEGENERATE);
    if (isnan(L)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
  }
  __syncthreads();
  k_root_star<D>(a, wsh);  // backward reference row k* + k*-differenced rows
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int r = wid; r < R; r += nw) {
    double s1 = 0.0;
    for (int k = lane; k < K; k += 32) s1 += wsh[k] * (double)a.z_root[r * K + k];
    s1 = warp_sum(s1);
    double s2 = 0.0;
    for (int k = lane; k < K; k += 32) {
      const double dz = (double)a.z_root[r * K + k] - s1;
      s2 += wsh[k] * dz * dz;
    }
    s2 = warp_sum(s2);
    if (lane == 0) {
      a.m1_root[r] = s1;
      a.v_root[r] = s2;
    }
  }
}

// Taylor degree slot (0-4: degree 3/4/5/7/9, 5: none) for a bound on |exponent| (the forward's thresholds)
__device__ __forceinline__ int bwd_mom_mode(const TLArgs& a, float tb) {
  return tb <= a.thr[0] ? 0 : (tb <= a.thr[1] ? 1 : (tb <= a.thr[2] ? 2 : (tb <= a.thr[3] ? 3 : (tb <= a.thr[4] ? 4 : 5))));
}

// Column constants of the backward, log P(k'|k*): softmax over the group's columns of the fp64 logits
// t_ref(k') + B(k*,k') - B(k_ref,k') (t_ref from the column prep); thread t holds columns t + NT (2p + h).
template <int D, int CP>
__device__ __forceinline__ double bwd_col_logits(const TLArgs& a, int64_t i, double (&tl)[CP][2], double* red) {
  const int K = a.K, tid = threadIdx.x, NT = blockDim.x;
  double tmx = -CUDART_INF;
  {
    const double es = a.ws.ref->e_star, bs = a.ws.ref->bstar_const;
#pragma unroll
    for (int p = 0; p < CP; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kc = tid + NT * (2 * p + h);
        tl[p][h] = -CUDART_INF;
        if (kc < K) {
          double d2 = 0.0, g2 = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) {
            const double zz = (double)a.z[((size_t)i * D + r) * K + kc];
            const double dz = zz - (double)a.ws.ref->mu_star[r], gz = zz - (double)a.ws.ref->mu_ref[r];
            d2 += dz * dz;
            g2 += gz * gz;
          }
          // t_ref + B(k*,k') - B(k_ref,k')
          tl[p][h] = (bs - 0.5 * es * d2) - (a.ws.ref->bref_const - 0.5 * a.ws.ref->e_ref * g2) +
                     a.ws.tA[(size_t)i * K + kc];
          tmx = fmax(tmx, tl[p][h]);
        }
      }
  }
  tmx = block_max(tmx, red);
  double tse = 0.0;
#pragma unroll
  for (int p = 0; p < CP; ++p)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (tid + NT * (2 * p + h) < K) tse += exp(tl[p][h] - tmx);
  return tmx + log(block_sum(tse, red));
}

// Weights out + moments of one group (fp64), one pass shifted by the Q mean c = m_i (see k_backward).
template <int D, int CP>
__device__ __forceinline__ void bwd_out_moments(const TLArgs& a, int64_t i, const float2 (&acc)[CP], double* red) {
  const int K = a.K, tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = NT >> 5;
  // ---- weights out + moments (fp64), one pass shifted by the Q mean c = m_i:
  // S0 = sum w, S1 = sum w (z - c), S2 = sum w (z - c)^2, then E z = c S0 + S1 and
  // sum w (z - E z)^2 = S2 - 2 (E z - c) S1 + (E z - c)^2 S0 (exact algebra; one z conversion
  // per column and dimension instead of two, and one block reduction instead of two)
  double s0 = 0.0, s1[D], s2[D], cq[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    s1[r] = 0.0;
    s2[r] = 0.0;
    cq[r] = (double)a.q_m[i * D + r];
  }
  bool bad = false;
#pragma unroll
  for (int p = 0; p < CP; ++p)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kc = tid + NT * (2 * p + h);
      if (kc < K) {
        const float wf = h ? acc[p].y : acc[p].x;
        bad |= isnan(wf);
        a.w[(size_t)i * K + kc] = wf;
        const double wv = wf;
        s0 += wv;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          const double e = (double)a.z[((size_t)i * D + r) * K + kc] - cq[r];
          const double we = wv * e;
          s1[r] += we;
          s2[r] = fma(we, e, s2[r]);
        }
      }
    }
  if (bad) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
  s0 = warp_sum(s0);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const double v1 = warp_sum(s1[r]), v2 = warp_sum(s2[r]);
    if (lane == 0) {
      red[wid * D + r] = v1;
      red[(nw + wid) * D + r] = v2;
    }
  }
  if (lane == 0) red[32 * D + wid] = s0;  // red: [32 D] (S1, S2: 2 nw D <= 32 D, nw <= 16) + [32] (S0)
  __syncthreads();
  if (tid < D) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < nw; ++w) {
      t0 += red[32 * D + w];
      t1 += red[w * D + tid];
      t2 += red[(nw + w) * D + tid];
    }
    const double m1 = cq[tid] * t0 + t1, dm = m1 - cq[tid];
    a.m1[i * D + tid] = m1;
    a.v[i * D + tid] = t2 - 2.0 * dm * t1 + dm * dm * t0;
  }
}

// ----------------------------------------------------------- backward (K4)
// Thread t owns columns k' = t + NT*(2p+h); the row table (alpha'', gamma',
// c', w_root) is in shared memory and read as warp-broadcasts.
template <int D, int CP>
__global__ void __launch_bounds__(256) k_backward(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RS = pad4(D + 3);
  const int K = a.K, tid = threadIdx.x, NT = blockDim.x;
  constexpr int CW = D + 2;
  float* rows = reinterpret_cast<float*>(smem);          // [K][RS]
  float* spare = rows + (size_t)K * RS;                  // [K] (padded to even; unused)
  double* red = reinterpret_cast<double*>(spare + ((K + 1) & ~1));  // [32][D] + [32]
  const int lane = tid & 31, wid = tid >> 5, nw = NT >> 5;
  // groups past the first wave from a device-wide queue (claimed one group ahead; the block
  // reductions below order the claim before every thread's read of s_next)
  __shared__ int64_t s_next;

  for (int64_t i = blockIdx.x; i < a.n_local;) {
    __syncthreads();
    if (tid == 0) s_next = (int64_t)gridDim.x + atomicAdd(&a.cnt->claim_bwd, 1u);
    if constexpr (D == 1 && kMomentTiles) {
      if (bwd_mom_mode(a, 2.f * a.ws.gtb[i]) < 5) {  // k_backward_mom1's group (launched just before)
        __syncthreads();
        i = s_next;
        continue;
      }
    }
    // row table re-centred on the group's Q mean and referenced to the backward row k*
    // (DESIGN.md "Backward reference"):  log P(k'|k) = log P(k'|k*) + E_k(k') - (l_k - l_*),
    // E_k(z) = B(k,z) - B(k*,z) = E'a_ik + c''_k . w + Eg_k |w|^2 with c'' = Eb_k + 2 Eg_k m_i,
    // and E'a_ik - (l_k - l_*) = -(h_k - h_*)  (h = the forward's re-centred message)
    {
      float mi[D];
#pragma unroll
      for (int r = 0; r < D; ++r) mi[r] = a.q_m[i * D + r];
      const float hs = a.ws.hmsg[(size_t)i * K + a.ws.ref->k_star];
      for (int k = tid; k < K; k += NT) {
        const float* bc = a.ws.bwd_coef + (size_t)k * (D + 1);
        const float g = bc[D];
        float* rw = rows + (size_t)k * RS;
#pragma unroll
        for (int r = 0; r < D; ++r) rw[2 + r] = fmaf(2.f * g, mi[r], bc[r]) * kLog2e;
        rw[0] = -(a.ws.hmsg[(size_t)i * K + k] - hs) * kLog2e;
        rw[1] = g * kLog2e;
        rw[2 + D] = a.w_root[k];
      }
    }
    float2 u[CP][D], U2[CP], Lc[CP];
    constexpr int CS = pad4(D + 3);
    const int Kp = FwdLayout<D>::kpad(K);
    // column constants log P(k'|k*): softmax over the group's columns of the fp64 logits
    // B(k*,k') + A_i(k') (A from the column prep)
    double tl[CP][2];
    const double tlse = bwd_col_logits<D, CP>(a, i, tl, red);
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      float uu[2][D], u2[2], lc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        // column record (w, |w|^2, P, ln P) written by the column prep (K2a)
        const int kc = tid + NT * (2 * p + h);
        const bool ok = kc < K;
        const float* gcol = a.ws.colrec + (size_t)i * FwdLayout<D>::group_floats(K);
        float urec[D], u2rec, prec, lrec;
        load_col<D>(gcol, ok ? kc : 0, urec, u2rec, prec, lrec);
#pragma unroll
        for (int r = 0; r < D; ++r) uu[h][r] = ok ? urec[r] : 0.f;
        u2[h] = ok ? u2rec : 0.f;
        lc[h] = ok ? (float)((tl[p][h] - tlse) * kLog2eD) : -CUDART_INF_F;
      }
#pragma unroll
      for (int r = 0; r < D; ++r) u[p][r] = make_float2(uu[0][r], uu[1][r]);
      U2[p] = make_float2(u2[0], u2[1]);
      Lc[p] = make_float2(lc[0], lc[1]);
    }
    __syncthreads();
    float2 acc[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) acc[p] = f2(0.f);
    // one row of the pair tile; `soft` evaluates its exponentials on the FMA pipe (exp2_poly2)
    auto row = [&](int k, bool soft) {
      const float* rp = rows + (size_t)k * RS;
      float rb[RS];
#pragma unroll
      for (int q = 0; q < RS / 4; ++q) {
        const float4 v = reinterpret_cast<const float4*>(rp)[q];
        rb[4 * q] = v.x;
        rb[4 * q + 1] = v.y;
        rb[4 * q + 2] = v.z;
        rb[4 * q + 3] = v.w;
      }
      const float2 w2 = f2(rb[2 + D]);
#pragma unroll
      for (int p = 0; p < CP; ++p) {
        float2 t;
        if constexpr (D == 1) {
          t = add2(fma2(fma2(f2(rb[1]), u[p][0], f2(rb[2])), u[p][0], f2(rb[0])), Lc[p]);
        } else {
          t = add2(fma2(f2(rb[1]), U2[p], f2(rb[0])), Lc[p]);
#pragma unroll
          for (int r = 0; r < D; ++r) t = fma2(f2(rb[2 + r]), u[p][r], t);
        }
        acc[p] = fma2(w2, soft ? exp2_poly2(t) : make_float2(ex2(t.x), ex2(t.y)), acc[p]);
      }
    };
    int k = 0;
    for (; k + kBwdUnroll <= K; k += kBwdUnroll) {  // the last kBwdSoft rows of each block: FMA-pipe exps
#pragma unroll
      for (int kk = 0; kk < kBwdUnroll; ++kk) row(k + kk, kk >= kBwdUnroll - bwd_soft<D>());
    }
    for (; k < K; ++k) row(k, false);
    bwd_out_moments<D, CP>(a, i, acc, red);
    i = s_next;
  }
}

// ----------------------------------------------------- backward moment tiles (K4, d = 1)
// The backward for d = 1 groups whose |E| bound admits a Taylor mode (the backward twin of the forward's
// tile_moments1), one warp per group.  Per column k',
//   w(k') = P(k'|k*) sum_k a_k e^{E_k(w)},  a_k = w_root(k) 2^{rho_k},  E_k(w) = beta_k w + gamma_k w^2
// (k_backward's row table: rho_k = -log2e (h_k - h_*), in natural units for E), and with
// e^E = sum_{n<=N} E^n / n! (degree N from the bound on |E| over the group's rows and columns, with the
// forward's thresholds; the groups are those whose 2 x forward bound admits a mode, k_backward skips them):
//   sum_k a_k e^{E_k(w)} = sum_{p=0..2N} A_p w^p,  A_p = sum_{n+j=p, j<=n<=N} C(n,j)/n! sum_k a_k gamma_k^j beta_k^(n-j)
// -- the pair sum rearranged (exact algebra): O(K N^2) per group + O(N) per column in fp64 instead of
// one exponential per pair; the coefficients are reduced in a fixed order (warp butterflies).
template <int N>
__device__ __forceinline__ void bwd_mom_group(const TLArgs& a, int64_t i, float mi) {
  constexpr int NC = 2 * N + 1;
  const int K = a.K, lane = threadIdx.x & 31;
  const float hs = a.ws.hmsg[(size_t)i * K + a.ws.ref->k_star];
  double A[NC];
#pragma unroll
  for (int p = 0; p < NC; ++p) A[p] = 0.0;
  for (int k = lane; k < K; k += 32) {
    const float wr = a.w_root[k];
    if (wr == 0.f) continue;
    const float g = a.ws.bwd_coef[(size_t)k * 2 + 1];
    const double ak = (double)(wr * ex2(-(a.ws.hmsg[(size_t)i * K + k] - hs) * kLog2e));  // as the pair path
    const double ga = g, be = fmaf(2.f * g, mi, a.ws.bwd_coef[(size_t)k * 2]);
    double gp[N + 1], bp[N + 1];
    gp[0] = ak;  // a_k rides on the gamma powers
    bp[0] = 1.0;
#pragma unroll
    for (int j = 1; j <= N; ++j) {
      gp[j] = gp[j - 1] * ga;
      bp[j] = bp[j - 1] * be;
    }
    double fact = 1.0;
#pragma unroll
    for (int n = 0; n <= N; ++n) {
      if (n > 0) fact *= n;
      double bin = 1.0 / fact;  // C(n, j) / n!
#pragma unroll
      for (int j = 0; j <= n; ++j) {
        A[n + j] = fma(bin * gp[j], bp[n - j], A[n + j]);
        bin = bin * (n - j) / (j + 1);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < NC; ++p) A[p] = warp_sum(A[p]);
  // column logits t_ref + B(k*,.) - B(k_ref,.) and their softmax (fp64, as bwd_col_logits)
  const double es = a.ws.ref->e_star, bs = a.ws.ref->bstar_const;
  const double er = a.ws.ref->e_ref, br = a.ws.ref->bref_const;
  const double mus = a.ws.ref->mu_star[0], mur = a.ws.ref->mu_ref[0];
  const float* zg = a.z + (size_t)i * K;
  const double* tA = a.ws.tA + (size_t)i * K;
  auto logit = [&](int kc) {
    const double zz = zg[kc], dz = zz - mus, gz = zz - mur;
    return (bs - 0.5 * es * dz * dz) - (br - 0.5 * er * gz * gz) + tA[kc];
  };
  double tmx = -CUDART_INF;
  for (int kc = lane; kc < K; kc += 32) tmx = fmax(tmx, logit(kc));
  tmx = warp_max(tmx);
  double tse = 0.0;
  for (int kc = lane; kc < K; kc += 32) tse += exp(logit(kc) - tmx);
  const double tlse = tmx + log(warp_sum(tse));
  // weights and the moments (one pass shifted by the Q mean, as bwd_out_moments)
  const float* rec = a.ws.colrec + (size_t)i * FwdLayout<1>::group_floats(K);
  const double cq = mi;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  bool bad = false;
  for (int kc = lane; kc < K; kc += 32) {
    const double w = rec[FwdLayout<1>::off(kc, 0)];
    double sp = A[NC - 1];
#pragma unroll
    for (int q = NC - 2; q >= 0; --q) sp = fma(sp, w, A[q]);
    const float wf = ex2((float)((logit(kc) - tlse) * kLog2eD)) * (float)sp;  // P(k'|k*) as the pair path's Lc
    bad |= isnan(wf);
    a.w[(size_t)i * K + kc] = wf;
    const double wv = wf, e = (double)zg[kc] - cq, we = wv * e;
    s0 += wv;
    s1 += we;
    s2 = fma(we, e, s2);
  }
  if (bad) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    const double m1 = cq * s0 + s1, dm = m1 - cq;
    a.m1[i] = m1;
    a.v[i] = s2 - 2.0 * dm * s1 + dm * dm * s0;
  }
}

template <int D>  // D = 1 (a template so each per-d translation unit has its own instance)
__global__ void __launch_bounds__(256) k_backward_mom1(TLArgs a) {
  const int K = a.K, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t nmom = 0;
  // warp gw owns groups gw + j TW (TW warps in the grid) and scans 32 of them at a time (one load of
  // their bounds per lane, a ballot), then works its moment groups one by one.  E_k = D'_k - D'_{k*}
  // (both re-centred on m_i), so 2x the forward's bound on |D'| bounds |E|: the cheap decision
  // k_backward takes too; the degree below comes from the group's own bound.
  const int64_t gw = (int64_t)blockIdx.x * nw + wid, TW = (int64_t)gridDim.x * nw;
  for (int64_t j0 = 0; gw + j0 * TW < a.n_local; j0 += 32) {
    const int64_t il = gw + (j0 + lane) * TW;
    const bool mine = il < a.n_local && bwd_mom_mode(a, 2.f * a.ws.gtb[il]) < 5;
    for (uint32_t bits = __ballot_sync(0xffffffffu, mine); bits; bits &= bits - 1) {
      const int64_t i = gw + (j0 + __ffs(bits) - 1) * TW;
      const float mi = a.q_m[i], W2m = a.ws.gstat[i], wm = sqrtf(W2m);
      // bound on |E_k(w)| = |beta_k w + gamma_k w^2| over the rows and the group's columns
      float tbb = 0.f;
      for (int k = lane; k < K; k += 32) {
        const float g = a.ws.bwd_coef[(size_t)k * 2 + 1];
        tbb = fmaxf(tbb, fabsf(fmaf(2.f * g, mi, a.ws.bwd_coef[(size_t)k * 2])) * wm + fabsf(g) * W2m);
      }
      const int md = bwd_mom_mode(a, fminf(warp_maxf(tbb), 2.f * a.ws.gtb[i]));
      ++nmom;
      switch (md) {
        case 0: bwd_mom_group<3>(a, i, mi); break;
        case 1: bwd_mom_group<4>(a, i, mi); break;
        case 2: bwd_mom_group<5>(a, i, mi); break;
        case 3: bwd_mom_group<7>(a, i, mi); break;
        default: bwd_mom_group<9>(a, i, mi); break;
      }
    }
  }
  if (lane == 0 && nmom) atomicAdd(&a.cnt->mode_hist[6], (unsigned long long)nmom);  // diagnostics slot 6
}

// ---------------------------------------------------------------- launchers

inline TLArgs make_args(qem_ctx* c) {
  TLArgs a{};
  const qem_model_desc& d = c->desc;
  a.K = d.K;
  a.J = d.n_obs;
  a.scale_kind = d.scale_kind;
  a.n_local = c->n_local;
  a.fixed_var = d.fixed_var;
  a.obs_var = d.obs_var;
  a.prior_mean = d.prior_mean;
  a.prior_var = d.prior_var;
  const qem_level& r = c->bufs.level[0];
  const qem_level& g = c->bufs.level[1];
  a.z_root = r.z;
  a.qr_m = r.q_mean;
  a.qr_v = r.q_var;
  a.w_root = r.w;
  a.m1_root = r.m1;
  a.v_root = r.v;
  a.z = g.z;
  a.q_m = g.q_mean;
  a.q_v = g.q_var;
  a.w = g.w;
  a.m1 = g.m1;
  a.v = g.v;
  a.x = c->bufs.x;
  a.y = c->bufs.y;
  a.log_pe = c->bufs.log_pe;
  a.trace = c->in_iterate ? c->bufs.trace : nullptr;
  a.trace_len = c->bufs.trace_len;
  a.t_host = 0;
  a.tc = c->tc;
  a.evidence_only = c->evidence_only;
  a.fuse_sample = c->fuse_sample;
  {  // column prep: enough warps per group that the rank's groups cover the colprep grid's warps ~4x
    const int64_t warps = (int64_t)c->grid_prep * 8, nit = d.K / 64;
    int sp = 1;
    while (sp < 8 && 2 * sp <= nit && c->n_local * sp < 4 * warps) sp *= 2;
    a.prep_split = sp;
  }
  a.t_sample = c->fuse_iter;
  a.skey = make_uint2((uint32_t)c->fuse_seed, (uint32_t)(c->fuse_seed >> 32));
  a.g_begin = c->g_begin;
  if (c->evidence_only) {
    a.log_pe = c->bufs.log_pe_fresh;  // log Pe(z_new)
    a.trace = nullptr;
  }
  // |D'| bound below which the degree-n Taylor remainder |D'|^{n+1}/(n+1)!,
  // accumulated over all N groups of the plate, stays under 2e-6
  {  // R41: 1e30 keeps the aux merge of 4 slices' sums finite; QEM_FWD_REDO_THR (tests) forces redos
    static const float thr = getenv("QEM_FWD_REDO_THR") ? (float)atof(getenv("QEM_FWD_REDO_THR")) : 1.0e30f;
    a.redo_thr = thr;
  }
  const int degs[5] = {3, 4, 5, 7, 9};
  for (int q = 0; q < 5; ++q) {
    double f = 1.0;
    for (int m = 2; m <= degs[q] + 1; ++m) f *= m;
    double t = pow(f * 2e-6 / (double)(d.n > 0 ? d.n : 1), 1.0 / (degs[q] + 1));
    a.thr[q] = (float)(t < 0.5 ? t : 0.5);
  }
  a.ws = c->tw;
  if (c->bufs.plate_sum) a.ws.red = c->bufs.plate_sum;
  a.cnt = c->cnt;
  return a;
}

static int rows_threads(int K, int rp) {
  int nt = (K + 2 * rp - 1) / (2 * rp);
  nt = (nt + 31) & ~31;
  return nt < 32 ? 32 : nt;
}
static int pick_rp(int K, int D) {
  static const int forced = [] {
    const char* e = getenv("QEM_RP");  // tuning override: 1 or 2 row pairs per thread
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  // 4 rows per thread amortise each column load (config 4: 4.68 -> 4.57 ms); wide latents keep
  // 2 rows per thread below K = 512 (register budget)
  return (K >= 512 || (K >= 256 && D <= 4)) ? 2 : 1;
}

template <int D>
static size_t bwd_smem(int K) {
  constexpr int RS = pad4(D + 3);
  size_t sm = (size_t)K * RS * sizeof(float) + (size_t)((K + 1) & ~1) * sizeof(float) + (32 * D + 32) * sizeof(double);
  return (sm + 15) & ~(size_t)15;
}

using KernelFn = void (*)(TLArgs);

// The forward's rows per thread: d <= 4 keeps 2 (one row pair, the 64-register budget of k_forward)
// up to K = 512, wider latents and larger K as the backward
static int pick_rp_fwd(int K, int D) {
  static const int forced = [] {
    const char* e = getenv("QEM_RP");
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  return (D <= 4 && K <= 512) ? 1 : pick_rp(K, D);  // k_forward's blocks stay <= 256 threads
}

template <int D>
static KernelFn fwd_fn(int rp) {
  return rp == 1 ? k_forward<D, 1> : k_forward<D, 2>;
}
template <int D>
static KernelFn prep_fn(int obs, bool tc) {
  if constexpr (D == 1) {
    if (obs == QEM_OBS_GAUSS) return tc ? k_colprep_tc1<QEM_OBS_GAUSS> : k_colprep<D, QEM_OBS_GAUSS, false>;
  }
  if constexpr (D >= 8 && D <= kTcD) {
    if (tc) return k_colprep_tc<D, QEM_OBS_BERNOULLI_LOGIT>;
  }
  return k_colprep<D, QEM_OBS_BERNOULLI_LOGIT, false>;
}
template <int D>
static KernelFn bwd_fn(int cp) {
  return cp == 1 ? k_backward<D, 1> : k_backward<D, 2>;
}

// Resident CTAs per SM for a kernel at (threads, dynamic smem).
static int occupancy(KernelFn f, int nt, size_t sm) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, nt, sm) != cudaSuccess || nb < 1) nb = 1;
  return nb;
}

template <int D>
static int prep_threads(int) { return 32 * FwdLayout<D>::PREP_WARPS; }
template <int D>
static size_t prep_smem(int K, int J, bool tc) {
  return tc ? (TcGeo<D <= kTcD ? D : 16>::COMPACT ? 0 : PrepTc::bytes(K, J)) : FwdLayout<D>::prep_bytes(K, J);
}
template <int D>
static int prep_threads_tc(int K, bool tc) { return tc ? 32 * PrepTc::WARPS : prep_threads<D>(K); }

template <int D>
static void grids(const qem_model_desc* d, int64_t n_local, int sms, bool tc, int* gf, int* gb, int* gp) {
  const int K = d->K, rp = pick_rp(K, D);
  int of, ob;
  if (tc) {
    if constexpr (D <= kTcD) {
      of = occupancy(k_forward_tc<D>, kFwdThreads, FwdTcL<D>::bytes(K));
      ob = occupancy(k_backward_tc<D>, kBwdThreads, BwdTcL<D>::bytes(K));
      if constexpr (!TcGeo<D>::COMPACT) {  // set the dynamic-SMEM attributes of the TMA-staged group kernels
        occupancy(k_bwd_cols_tc<D>, GroupStage::THREADS, GroupStage::bytes(K, D));
        occupancy(k_moments_tc<D>, GroupStage::THREADS, GroupStage::bytes(K, D));
      }
    } else {
      of = ob = 1;
    }
  } else {
    const int rpf = pick_rp_fwd(K, D);
    of = occupancy(fwd_fn<D>(rpf), rows_threads(K, rpf), FwdLayout<D>::bytes(K, d->n_obs));
    ob = occupancy(bwd_fn<D>(rp), rows_threads(K, rp), bwd_smem<D>(K));
  }
  const int op = occupancy(prep_fn<D>(d->obs_kind, tc), prep_threads_tc<D>(K, tc), prep_smem<D>(K, d->n_obs, tc));
  // Persistent-style grids: one full wave of resident CTAs, capped by the groups.
  int64_t f = (int64_t)sms * of, b = (int64_t)sms * ob, p = (int64_t)sms * op;
  *gf = (int)(f < n_local ? f : n_local);
  *gb = (int)(b < n_local ? b : n_local);
  *gp = (int)(p < n_local ? p : n_local);
}

template <int D>
static cudaError_t fwd_dispatch_obs(qem_ctx* c, const TLArgs& a, cudaStream_t st) {
  const int K = a.K, rp = pick_rp_fwd(K, D);
  int nt = (K + 31) & ~31;
  const bool tc = D <= kTcD && c->tc;
  if (tc) {  // k_ref in one block, then the rows over K/128 blocks
    k_root_prep<D><<<1, nt, 0, st>>>(a, 1);
    k_root_prep<D><<<(K + 127) / 128, 128, 0, st>>>(a, 2);
  } else {
    k_root_prep<D><<<1, nt, 0, st>>>(a, 0);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (c->desc.obs_kind == QEM_OBS_GAUSS && D != 1) return cudaErrorInvalidValue;
  if (tc) {
    k_rowop_tc<D><<<(K + 255) / 256, 256, 0, st>>>(a);
    c->launches += 2;  // + the second root-prep phase
  }
  prep_fn<D>(c->desc.obs_kind, tc)<<<c->grid_prep, prep_threads_tc<D>(K, tc), prep_smem<D>(K, a.J, tc), st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (c->ev[0]) cudaEventRecord((cudaEvent_t)c->ev[0], st);
  if (tc)
    k_forward_tc<(D <= kTcD ? D : 1)><<<c->grid_fwd, kFwdThreads, FwdTcL<(D <= kTcD ? D : 1)>::bytes(K), st>>>(a);
  else
    fwd_fn<D>(rp)<<<c->grid_fwd, rows_threads(K, rp), FwdLayout<D>::bytes(K, a.J), st>>>(a);
  if (c->ev[1]) cudaEventRecord((cudaEvent_t)c->ev[1], st);
  c->launches += 3;
  return cudaGetLastError();
}

template <int D>
static cudaError_t bwd_dispatch(qem_ctx* c, const TLArgs& a, cudaStream_t st) {
  const int K = a.K;
  const int nt = (K + 31) & ~31;
  k_root<D><<<1, nt, (size_t)(K + 32) * sizeof(double), st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (c->evidence_only) {  // fresh-denominator pass: the root evidence is all it needs
    c->launches += 1;
    return cudaSuccess;
  }
  const int cp = pick_rp(K, D);
  const bool tc = D <= kTcD && c->tc;
  constexpr int DT = D <= kTcD ? D : 1;
  if (tc) {
    if constexpr (TcGeo<DT>::COMPACT)
      k_bwd_cols_warp<DT><<<c->grid_prep, 256, 0, st>>>(a);
    else
      k_bwd_cols_tc<DT><<<c->grid_stage, GroupStage::THREADS, GroupStage::bytes(K, DT), st>>>(a);
    c->launches += 1;
  }
  if (c->ev[2]) cudaEventRecord((cudaEvent_t)c->ev[2], st);
  if (tc)
    k_backward_tc<DT><<<c->grid_bwd, kBwdThreads, BwdTcL<DT>::bytes(K), st>>>(a);
  else {
    if constexpr (D == 1 && kMomentTiles) {
      k_backward_mom1<D><<<c->grid_prep, 256, 0, st>>>(a);  // one warp per group, like the column prep
      c->launches += 1;
    }
    bwd_fn<D>(cp)<<<c->grid_bwd, rows_threads(K, cp), bwd_smem<D>(K), st>>>(a);
  }
  if (c->ev[3]) cudaEventRecord((cudaEvent_t)c->ev[3], st);
  if (tc) {
    if constexpr (TcGeo<DT>::COMPACT)
      k_moments_warp<DT><<<c->grid_prep, 256, 0, st>>>(a);
    else
      k_moments_tc<DT><<<c->grid_stage, GroupStage::THREADS, GroupStage::bytes(K, DT), st>>>(a);
    c->launches += 1;
  }
  c->launches += 2;
  return cudaGetLastError();
}

// Largest dynamic shared memory any two-level kernel of this model's path asks for (bytes): checked
// against the device's opt-in limit at context creation, so an oversized K / J is a model error up
// front instead of a failed launch inside a captured graph.
template <int D>
static size_t max_smem(const qem_model_desc* d, bool tc) {
  const int K = d->K, J = d->n_obs;
  size_t m = 0;
  auto up = [&](size_t v) { m = v > m ? v : m; };
  if (tc) {
    if constexpr (D <= kTcD) {
      up(FwdTcL<D>::bytes(K));
      up(BwdTcL<D>::bytes(K));
      if constexpr (!TcGeo<D>::COMPACT) {
        up(PrepTc::bytes(K, J));
        up(GroupStage::bytes(K, D));
      }
    }
  } else {
    up(FwdLayout<D>::prep_bytes(K, J));
    up(FwdLayout<D>::bytes(K, J));
    up(bwd_smem<D>(K));
  }
  return m;
}

// Per-D entry points (explicitly instantiated in qem_tl_d<D>.cu).
template <int D>
cudaError_t tl_forward_d(qem_ctx* c, cudaStream_t st) {
  TLArgs a = make_args(c);
  return fwd_dispatch_obs<D>(c, a, st);
}
template <int D>
cudaError_t tl_backward_d(qem_ctx* c, cudaStream_t st) {
  TLArgs a = make_args(c);
  return bwd_dispatch<D>(c, a, st);
}
template <int D>
void tl_grids_d(const qem_model_desc* d, int64_t n_local, int sms, int* gf, int* gb, int* gp) {
  grids<D>(d, n_local, sms, tl_use_tc(d) != 0, gf, gb, gp);
}
template <int D>
size_t tl_max_smem_d(const qem_model_desc* d) {
  return max_smem<D>(d, tl_use_tc(d) != 0);
}

#define QEM_TL_INSTANTIATE(D)                                                                          \
  template cudaError_t tl_forward_d<D>(qem_ctx*, cudaStream_t);                                         \
  template cudaError_t tl_backward_d<D>(qem_ctx*, cudaStream_t);                                        \
  template void tl_grids_d<D>(const qem_model_desc*, int64_t, int, int*, int*, int*);                   \
  template size_t tl_max_smem_d<D>(const qem_model_desc*);

}  // namespace qem
