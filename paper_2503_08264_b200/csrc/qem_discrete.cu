// qem_discrete.cu -- discrete (categorical) latents under a continuous root: the E-step side of
// NEXT row f1 (R30), on the explicit-table engine of qem_tables.cu.
//
// Model (Occupancy-shaped: a Bernoulli "true presence" latent per site whose
// logit is a product of root latents and a site covariate, observed through R repeated Bernoulli
// detections): root r in R^d with prior N(0, I) and Q_root = N(m, diag v); per instance i a
// categorical z_i in {0..C-1} with prior logits eta_ic(r) = x_ic . r and
// Q_i = Categorical(p_i); the observations enter through their per-state log-likelihood
// L_i(c) = log p(y_i | z_i = c) (a data-only table).  K samples of every latent (Alg. 1 line 4),
// log-factor tables
//   f_root(k)   = log N(r^k; 0, I) - log q(r^k)
//   f_i(k, k')  = log softmax_c(eta_i(r^k))[z_i^k'] + L_i(z_i^k') - log p_i(z_i^k')
// then qem_estep_tables (Eq. 7) and the moments E[onehot z_i] = sum_k' w_i(k') onehot(z_i^k'),
// E r, E r^2 under w_root (Eq. 7a), for the EMA + M-step of qem_mstep_family.
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

constexpr int kCatThreads = 256;

// z_i^k = min{c : u < sum_{c' <= c} p_i(c')} (fp64, sequential prefix), u = ((w >> 8) + 1/2) 2^-24
// from word k % 4 of Philox4x32-10 at counter (k / 4, 0, i, 3 << 24 | iter).
__global__ void __launch_bounds__(kCatThreads) k_cat_sample(int64_t n, int C, int K, uint2 key, uint32_t iterword,
                                                            const double* __restrict__ p, int32_t* __restrict__ z) {
  const int quads = (K + 3) >> 2;
  const int64_t q = (int64_t)blockIdx.x * kCatThreads + threadIdx.x;
  const int64_t i = q / quads;
  if (i >= n) return;
  const int k0 = (int)(q - i * quads) * 4;
  const uint4 o = philox4x32_10(make_uint4((uint32_t)(k0 >> 2), 0u, (uint32_t)i, iterword), key);
  const uint32_t wv[4] = {o.x, o.y, o.z, o.w};
  const double* pi = p + i * C;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = k0 + j;
    if (k >= K) break;
    const double u = ((double)(wv[j] >> 8) + 0.5) * 5.9604644775390625e-08;
    int c = 0;
    double cum = pi[0];
    while (c < C - 1 && u >= cum) cum += pi[++c];
    z[i * K + k] = c;
  }
}

// One block per instance (block n: the root row).  The K x C table h_i(k, c) =
// log softmax_c(eta_i(r^k)) + L_i(c) - log p_i(c) is built once per chunk of root samples in
// shared memory (thread per k), then the chunk's rows f_i(k, .) are written coalesced by
// gathering h_i(k, z_i^k') (z_i staged in shared memory).
constexpr int kCatTabThreads = 256;
constexpr int kCatTabH = 2048;  // doubles of h per chunk (16 KB)

__global__ void __launch_bounds__(kCatTabThreads) k_cat_tables(int64_t n, int C, int K, int d,
                                                               const float* __restrict__ rz,
                                                               const float* __restrict__ rm,
                                                               const float* __restrict__ rv,
                                                               const double* __restrict__ x,
                                                               const double* __restrict__ L,
                                                               const double* __restrict__ p,
                                                               const int32_t* __restrict__ z,
                                                               double* __restrict__ f_root, double* __restrict__ f) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* hs = reinterpret_cast<double*>(smem);              // [KC][C]
  int32_t* zs = reinterpret_cast<int32_t*>(hs + kCatTabH);   // [K]
  __shared__ double hc[QEM_CAT_MAX_C];                       // L_i(c) - log p_i(c)
  const int tid = threadIdx.x;
  if (blockIdx.x == n) {  // f_root(k) = sum_e [log N(r_e; 0, 1) - log N(r_e; m_e, v_e)]
    for (int k = tid; k < K; k += blockDim.x) {
      double s = 0.0;
      for (int e = 0; e < d; ++e) {
        const double r = rz[(int64_t)e * K + k], v = rv[e], dr = r - (double)rm[e];
        s += -0.5 * r * r + 0.5 * log(v) + 0.5 * dr * dr / v;  // the 2 pi terms cancel
      }
      f_root[k] = s;
    }
    return;
  }
  const int64_t i = blockIdx.x;
  if (tid < C) hc[tid] = L[i * C + tid] - log(p[i * C + tid]);
  for (int k = tid; k < K; k += blockDim.x) zs[k] = z[i * K + k];
  const int KC = kCatTabH / C;
  for (int kb = 0; kb < K; kb += KC) {
    const int kn = K - kb < KC ? K - kb : KC;
    __syncthreads();  // hc / zs ready; the previous chunk's gathers done
    for (int kk = tid; kk < kn; kk += blockDim.x) {
      const int k = kb + kk;
      double eta[QEM_CAT_MAX_C];
      double mx = -CUDART_INF;
#pragma unroll
      for (int c = 0; c < QEM_CAT_MAX_C; ++c) {
        double t = 0.0;
        if (c < C)
          for (int e = 0; e < d; ++e) t += x[(i * C + c) * d + e] * (double)rz[(int64_t)e * K + k];
        eta[c] = t;
        if (c < C) mx = fmax(mx, t);
      }
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < QEM_CAT_MAX_C; ++c)
        if (c < C) sum += exp(eta[c] - mx);
      const double lse = mx + log(sum);
#pragma unroll
      for (int c = 0; c < QEM_CAT_MAX_C; ++c)
        if (c < C) hs[kk * C + c] = (eta[c] - lse) + hc[c];
    }
    __syncthreads();
    double* fi = f + (i * K + kb) * (int64_t)K;
    if (K <= (int)blockDim.x) {  // several rows per pass
      const int rpp = blockDim.x / K, r = tid / K, kp = tid - r * K;
      if (r < rpp) {
        const int zc = zs[kp];
        for (int kk = r; kk < kn; kk += rpp) fi[(int64_t)kk * K + kp] = hs[kk * C + zc];
      }
    } else {
      for (int kk = 0; kk < kn; ++kk)
        for (int kp = tid; kp < K; kp += blockDim.x) fi[(int64_t)kk * K + kp] = hs[kk * C + zs[kp]];
    }
  }
}

// ---- the factorised E-step (qem_estep_categorical): f_i(k, k') = h_i(k, z_i^k') depends on k'
// only through the state, so with n_i(c) = #{k' : z_i^k' = c}
//   g_i(k)  = log sum_c n_i(c) exp(h_i(k, c)) - ln K                      (states with n_i(c) > 0)
//   w_i(k') = W_i(z_i^k'),  W_i(c) = sum_k w_root(k) exp(h_i(k, c) - ln K - g_i(k))
// -- the explicit-table results (Eq. 7) in O(n K C) instead of O(n K^2).
__device__ __forceinline__ void cat_h_row(int64_t i, int k, int C, int K, int d, const double* __restrict__ x,
                                          const float* __restrict__ rz, const double* hc,
                                          double (&h)[QEM_CAT_MAX_C]) {
  double mx = -CUDART_INF;
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c) {
    double eta = 0.0;
    if (c < C)
      for (int e = 0; e < d; ++e) eta += x[(i * C + c) * d + e] * (double)rz[(int64_t)e * K + k];
    h[c] = eta;
    if (c < C) mx = fmax(mx, eta);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c)
    if (c < C) s += exp(h[c] - mx);
  const double lse = mx + log(s);
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c)
    if (c < C) h[c] = (h[c] - lse) + hc[c];
}

// Warp-per-instance state: the counts n_i(c) by ballots over the instance's K samples and the
// per-state constants L_i(c) - log p_i(c) (lane c computes, every lane receives) -- no block sync.
__device__ __forceinline__ void cat_warp_setup(int64_t i, int C, int K, const double* L, const double* p,
                                               const int32_t* z, int lane, double (&hc)[QEM_CAT_MAX_C],
                                               int (&cnt)[QEM_CAT_MAX_C]) {
  const double mine = lane < C ? L[i * C + lane] - log(p[i * C + lane]) : 0.0;
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c) {
    hc[c] = __shfl_sync(0xffffffffu, mine, c);
    cnt[c] = 0;
  }
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    const int zc = k < K ? z[i * K + k] : -1;
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c) cnt[c] += __popc(__ballot_sync(0xffffffffu, zc == c));
  }
}

constexpr int kCatWarps = 8;

__global__ void __launch_bounds__(kCatWarps * 32) k_cat_fwd(int64_t n, int C, int K, int d,
                                                            const float* __restrict__ rz,
                                                            const float* __restrict__ rm,
                                                            const float* __restrict__ rv,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ L,
                                                            const double* __restrict__ p,
                                                            const int32_t* __restrict__ z, double* __restrict__ f_root,
                                                            double* __restrict__ g) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kCatWarps + (threadIdx.x >> 5);
  if (i > n) return;
  if (i == n) {  // f_root as in k_cat_tables
    for (int k = lane; k < K; k += 32) {
      double s = 0.0;
      for (int e = 0; e < d; ++e) {
        const double r = rz[(int64_t)e * K + k], v = rv[e], dr = r - (double)rm[e];
        s += -0.5 * r * r + 0.5 * log(v) + 0.5 * dr * dr / v;
      }
      f_root[k] = s;
    }
    return;
  }
  double hc[QEM_CAT_MAX_C];
  int cnt[QEM_CAT_MAX_C];
  cat_warp_setup(i, C, K, L, p, z, lane, hc, cnt);
  double lcnt[QEM_CAT_MAX_C];
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c) lcnt[c] = c < C && cnt[c] > 0 ? log((double)cnt[c]) : -CUDART_INF;
  const double lk = log((double)K);
  for (int k = lane; k < K; k += 32) {
    double h[QEM_CAT_MAX_C];
    cat_h_row(i, k, C, K, d, x, rz, hc, h);
    double mx = -CUDART_INF;
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c)
      if (lcnt[c] > -CUDART_INF) mx = fmax(mx, h[c] + lcnt[c]);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c)
      if (lcnt[c] > -CUDART_INF) s += exp(h[c] + lcnt[c] - mx);
    g[i * K + k] = mx == -CUDART_INF ? -CUDART_INF : mx + log(s) - lk;
  }
}

__global__ void __launch_bounds__(kCatWarps * 32) k_cat_bwd(int64_t n, int C, int K, int d,
                                                            const float* __restrict__ rz,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ L,
                                                            const double* __restrict__ p,
                                                            const int32_t* __restrict__ z,
                                                            const double* __restrict__ g,
                                                            const double* __restrict__ w_root,
                                                            double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kCatWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  double hc[QEM_CAT_MAX_C];
  int cnt[QEM_CAT_MAX_C];
  cat_warp_setup(i, C, K, L, p, z, lane, hc, cnt);
  const double lk = log((double)K);
  double acc[QEM_CAT_MAX_C];
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c) acc[c] = 0.0;
  for (int k = lane; k < K; k += 32) {
    const double wr = w_root[k];
    if (wr == 0.0) continue;  // zero-weight root samples carry no tuples (g may be -inf)
    double h[QEM_CAT_MAX_C];
    cat_h_row(i, k, C, K, d, x, rz, hc, h);
    const double gk = g[i * K + k];
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c)
      if (c < C && cnt[c] > 0) acc[c] += wr * exp(h[c] - lk - gk);
  }
  double W[QEM_CAT_MAX_C];
#pragma unroll
  for (int c = 0; c < QEM_CAT_MAX_C; ++c) W[c] = warp_sum(acc[c]);  // fixed shuffle tree
  for (int k = lane; k < K; k += 32) {
    const int zc = z[i * K + k];
    double v = W[0];
#pragma unroll
    for (int c = 1; c < QEM_CAT_MAX_C; ++c) v = zc == c ? W[c] : v;
    w[i * K + k] = v;
  }
}

// Moments (Eq. 7a): one warp per instance, E[onehot z_i](c) = sum_k' w_i(k') [z_i^k' = c];
// block 0's first d warps also do the root's (E r_e, E r_e^2) under w_root.
__global__ void __launch_bounds__(kCatThreads) k_cat_moments(int64_t n, int C, int K, int d,
                                                             const double* __restrict__ w_root,
                                                             const float* __restrict__ rz,
                                                             const double* __restrict__ w,
                                                             const int32_t* __restrict__ z,
                                                             double* __restrict__ root_m, double* __restrict__ pm) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (kCatThreads / 32) + (threadIdx.x >> 5);
  if (wid < n) {
    double acc[QEM_CAT_MAX_C];
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c) acc[c] = 0.0;
    for (int kp = lane; kp < K; kp += 32) {
      const int c = z[wid * K + kp];
      const double wk = w[wid * K + kp];
#pragma unroll
      for (int cc = 0; cc < QEM_CAT_MAX_C; ++cc) acc[cc] += cc == c ? wk : 0.0;
    }
#pragma unroll
    for (int c = 0; c < QEM_CAT_MAX_C; ++c) {
      const double t = warp_sum(acc[c]);
      if (lane == 0 && c < C) pm[wid * C + c] = t;
    }
  } else if (wid - n < d) {
    const int e = (int)(wid - n);
    double m1 = 0.0, m2 = 0.0;
    for (int k = lane; k < K; k += 32) {
      const double r = rz[(int64_t)e * K + k], wk = w_root[k];
      m1 += wk * r;
      m2 += wk * r * r;
    }
    m1 = warp_sum(m1);
    m2 = warp_sum(m2);
    if (lane == 0) {
      root_m[2 * e] = m1;
      root_m[2 * e + 1] = m2;
    }
  }
}

// EMA + M-step (one thread per root dim, then per instance).
__global__ void __launch_bounds__(kCatThreads) k_cat_mstep(int64_t n, int C, int d, double lam, double floor,
                                                           const double* __restrict__ root_m, double* root_ema,
                                                           float* root_mean, float* root_var,
                                                           const double* __restrict__ pm, double* p_ema, double* p,
                                                           unsigned long long* clamps) {
  const int64_t t = (int64_t)blockIdx.x * kCatThreads + threadIdx.x;
  if (t < d) {
    double* e = root_ema + 2 * t;
    e[0] = lam * e[0] + (1.0 - lam) * root_m[2 * t];
    e[1] = lam * e[1] + (1.0 - lam) * root_m[2 * t + 1];
    double v = e[1] - e[0] * e[0];
    if (!(v >= floor)) {
      v = floor;
      if (clamps) atomicAdd(clamps, 1ull);  // integer count: order-independent
    }
    root_mean[t] = (float)e[0];
    root_var[t] = (float)v;
  } else if (t - d < n) {
    const int64_t i = t - d;
    double s = 0.0;
    for (int c = 0; c < C; ++c) {
      const double v = lam * p_ema[i * C + c] + (1.0 - lam) * pm[i * C + c];
      p_ema[i * C + c] = v;
      s += v;
    }
    for (int c = 0; c < C; ++c) p[i * C + c] = p_ema[i * C + c] / s;
  }
}

// L_i(c) = sum_r y_ir l_irc - softplus(l_irc) (fp64), one thread per (i, c).
__global__ void __launch_bounds__(kCatThreads) k_cat_loglik(int64_t n, int C, int R, const uint8_t* __restrict__ y,
                                                            const double* __restrict__ logit, double* __restrict__ L) {
  const int64_t t = (int64_t)blockIdx.x * kCatThreads + threadIdx.x;
  if (t >= n * C) return;
  const int64_t i = t / C;
  const int c = (int)(t - i * C);
  double s = 0.0;
  for (int r = 0; r < R; ++r) {
    const double l = logit[(i * R + r) * C + c];
    s += (y[i * R + r] ? l : 0.0) - (fmax(l, 0.0) + log1p(exp(-fabs(l))));
  }
  L[t] = s;
}

cudaError_t launch_cat_mstep(int64_t n, int C, int d, double lam, double floor, const double* root_m, double* root_ema,
                             float* root_mean, float* root_var, const double* pm, double* p_ema, double* p,
                             int64_t* clamps, cudaStream_t st) {
  const int64_t threads = n + d;
  k_cat_mstep<<<(unsigned)((threads + kCatThreads - 1) / kCatThreads), kCatThreads, 0, st>>>(
      n, C, d, lam, floor, root_m, root_ema, root_mean, root_var, pm, p_ema, p,
      reinterpret_cast<unsigned long long*>(clamps));
  return cudaGetLastError();
}

cudaError_t launch_cat_loglik(int64_t n, int C, int R, const uint8_t* y, const double* logit, double* L,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_cat_loglik<<<(unsigned)((n * C + kCatThreads - 1) / kCatThreads), kCatThreads, 0, st>>>(n, C, R, y, logit, L);
  return cudaGetLastError();
}

cudaError_t launch_cat_estep(int64_t n, int C, int K, int d, const float* rz, const float* rm, const float* rv,
                             const double* x, const double* L, const double* p, const int32_t* z, double* f_root,
                             double* g, double* log_pe, double* w_root, double* w, cudaStream_t st) {
  k_cat_fwd<<<(unsigned)((n + 1 + kCatWarps - 1) / kCatWarps), kCatWarps * 32, 0, st>>>(n, C, K, d, rz, rm, rv, x, L,
                                                                                      p, z, f_root, g);
  cudaError_t e = launch_plate_root(n, K, f_root, g, w, log_pe, w_root, st);
  if (e != cudaSuccess) return e;
  if (n > 0)
    k_cat_bwd<<<(unsigned)((n + kCatWarps - 1) / kCatWarps), kCatWarps * 32, 0, st>>>(n, C, K, d, rz, x, L, p, z, g,
                                                                                     w_root, w);
  return cudaGetLastError();
}

cudaError_t launch_cat_sample(int64_t n, int C, int K, uint64_t seed, int32_t iter, const double* p, int32_t* z,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t threads = n * ((K + 3) / 4);
  const uint32_t iterword = (3u << 24) | ((uint32_t)iter & 0xffffffu);
  k_cat_sample<<<(unsigned)((threads + kCatThreads - 1) / kCatThreads), kCatThreads, 0, st>>>(
      n, C, K, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)), iterword, p, z);
  return cudaGetLastError();
}

cudaError_t launch_cat_tables(int64_t n, int C, int K, int d, const float* rz, const float* rm, const float* rv,
                              const double* x, const double* L, const double* p, const int32_t* z, double* f_root,
                              double* f, cudaStream_t st) {
  const size_t smem = kCatTabH * sizeof(double) + (size_t)K * sizeof(int32_t);
  cudaError_t e = cudaFuncSetAttribute(k_cat_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_cat_tables<<<(unsigned)(n + 1), kCatTabThreads, smem, st>>>(n, C, K, d, rz, rm, rv, x, L, p, z, f_root, f);
  return cudaGetLastError();
}

cudaError_t launch_cat_moments(int64_t n, int C, int K, int d, const double* w_root, const float* rz, const double* w,
                               const int32_t* z, double* root_m, double* pm, cudaStream_t st) {
  const int64_t warps = n + d;
  k_cat_moments<<<(unsigned)((warps + kCatThreads / 32 - 1) / (kCatThreads / 32)), kCatThreads, 0, st>>>(
      n, C, K, d, w_root, rz, w, z, root_m, pm);
  return cudaGetLastError();
}

}  // namespace qem
