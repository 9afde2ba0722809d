// qem_gamma.cu -- Gamma and Beta approximate posteriors on the E-step side (NEXT row f1,
// DESIGN.md R32): a Gamma-Poisson and a Beta-Binomial hierarchy under a Gaussian root, on the
// explicit-table engine (qem_tables.cu) and the Gamma / Beta M-steps of qem_expfam.cu.
// Beta-Binomial: p_i | mu ~ Beta(kappa s, kappa (1 - s)), s = sigmoid(mu); y_i ~ Binomial(N_i, p_i);
// Q_i = Beta(a_i, b_i), drawn as X / (X + Y) from two Marsaglia-Tsang Gammas on the Philox
// streams 7 << 24 (X) and 8 << 24 (Y).
//
// Model: root mu ~ N(0, 1) (log mean rate), Q_root = N(m, v); per group i a rate
// lambda_i | mu ~ Gamma(shape alpha, rate alpha e^-mu) and counts y_ij | lambda_i ~ Poisson(lambda_i),
// j < J; Q_i = Gamma(shape k_i, rate th_i) ("Gamma" among the families the paper names for the
// M-step).  K samples of every latent (Alg. 1 line 4) and the tables
//   f_root(k)   = log N(mu^k; 0, 1) - log N(mu^k; m, v)
//   f_i(k, k')  = log Gamma(l; alpha, alpha e^-mu^k) + sum_j log Pois(y_ij; l) - log Gamma(l; k_i, th_i),
//                 l = lambda_i^k'
// then qem_estep_tables (Eq. 7) and the mean parameters E[lambda_i], E[ln lambda_i] (Eq. 7a).
//
// Gamma draws: Marsaglia-Tsang in fp64.  Attempt a of sample (i, k) uses Philox4x32-10 at counter
// (k, a, i, 6 << 24 | iter): x = sqrt(-2 ln u0) cos(2 pi u1) (fp64 Box-Muller), acceptance
// uniform u2, and for shape < 1 the boost u3^(1/shape) of the accepted attempt, with
// u_j = (word_j + 1/2) 2^-32.  At most 64 attempts (then NaN, flagged downstream).
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

constexpr uint32_t kGammaTag = 6u << 24;
constexpr int kGammaMaxAttempts = 64;

__device__ __forceinline__ double u32d(uint32_t w) { return ((double)w + 0.5) * 2.3283064365386963e-10; }

// Gamma(a, rate 1) by Marsaglia-Tsang; attempt `att` uses Philox at (k, att, i, tag | iter).
__device__ __forceinline__ double mt_gamma(double a, int k, int64_t i, uint32_t iterword, uint2 key) {
  const double d = (a < 1.0 ? a + 1.0 : a) - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
  for (int att = 0; att < kGammaMaxAttempts; ++att) {
    const uint4 o = philox4x32_10(make_uint4((uint32_t)k, (uint32_t)att, (uint32_t)i, iterword), key);
    const double x = sqrt(-2.0 * log(u32d(o.x))) * cospi(2.0 * u32d(o.y));
    const double v1 = 1.0 + c * x;
    if (v1 <= 0.0) continue;
    const double v = v1 * v1 * v1;
    if (log(u32d(o.z)) < 0.5 * x * x + d - d * v + d * log(v)) {
      double g = d * v;
      if (a < 1.0) g *= pow(u32d(o.w), 1.0 / a);
      return g;
    }
  }
  return CUDART_NAN;
}

__global__ void __launch_bounds__(256) k_gamma_sample(int64_t n, int K, uint2 key, uint32_t iterword,
                                                      const double* __restrict__ q, double* __restrict__ z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const int64_t i = t / K;
  const int k = (int)(t - i * K);
  z[t] = mt_gamma(q[2 * i], k, i, iterword, key) / q[2 * i + 1];  // Q_i = (shape, rate)
}

// Beta(a, b) = X / (X + Y), X ~ Gamma(a), Y ~ Gamma(b) on the streams 7 << 24 and 8 << 24.
__global__ void __launch_bounds__(256) k_beta_sample(int64_t n, int K, uint2 key, uint32_t iter,
                                                     const double* __restrict__ q, double* __restrict__ z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const int64_t i = t / K;
  const int k = (int)(t - i * K);
  const double x = mt_gamma(q[2 * i], k, i, (7u << 24) | (iter & 0xffffffu), key);
  const double y = mt_gamma(q[2 * i + 1], k, i, (8u << 24) | (iter & 0xffffffu), key);
  z[t] = x / (x + y);
}

// Beta-Binomial tables (one warp per (i, k) row; row n*K: the root row):
//   f_i(k, k') = log Beta(p; kappa s_k, kappa (1 - s_k)) + y_i ln p + (N_i - y_i) ln(1 - p)
//                + ln C(N_i, y_i) - log Beta(p; a_i, b_i),   s_k = sigmoid(mu^k), p = z_i^k'
__global__ void __launch_bounds__(256) k_beta_tables(int64_t n, int K, double kappa, const float* __restrict__ mu,
                                                     const float* __restrict__ rm, const float* __restrict__ rv,
                                                     const int32_t* __restrict__ y, const int32_t* __restrict__ N,
                                                     const double* __restrict__ q, const double* __restrict__ z,
                                                     double* __restrict__ f_root, double* __restrict__ f) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row > n * K) return;
  if (row == n * K) {
    const double m = rm[0], v = rv[0];
    for (int k = lane; k < K; k += 32) {
      const double r = mu[k], dr = r - m;
      f_root[k] = -0.5 * r * r + 0.5 * log(v) + 0.5 * dr * dr / v;
    }
    return;
  }
  const int64_t i = row / K;
  const int k = (int)(row - i * K);
  const double sk = 1.0 / (1.0 + exp(-(double)mu[k]));
  const double pa = kappa * sk, pb = kappa * (1.0 - sk);
  const double cp = lgamma(kappa) - lgamma(pa) - lgamma(pb);
  const double yy = y[i], nn = N[i];
  const double cb = lgamma(nn + 1.0) - lgamma(yy + 1.0) - lgamma(nn - yy + 1.0);
  const double qa = q[2 * i], qb = q[2 * i + 1];
  const double cq = lgamma(qa + qb) - lgamma(qa) - lgamma(qb);
  const double* zi = z + i * K;
  double* fr = f + row * K;
  for (int kp = lane; kp < K; kp += 32) {
    const double p = zi[kp], lp = log(p), l1 = log1p(-p);
    const double prior = cp + (pa - 1.0) * lp + (pb - 1.0) * l1;
    const double lik = cb + yy * lp + (nn - yy) * l1;
    const double lq = cq + (qa - 1.0) * lp + (qb - 1.0) * l1;
    fr[kp] = prior + lik - lq;
  }
}

// Beta mean parameters (E ln p, E ln(1-p)) per group [n][2], root (E mu, E mu^2) [2].
__global__ void __launch_bounds__(256) k_beta_moments(int64_t n, int K, const double* __restrict__ w_root,
                                                      const float* __restrict__ mu, const double* __restrict__ w,
                                                      const double* __restrict__ z, double* __restrict__ root_m,
                                                      double* __restrict__ gm) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wid > n) return;
  double s1 = 0.0, s2 = 0.0;
  if (wid == n) {
    for (int k = lane; k < K; k += 32) {
      const double r = mu[k], wk = w_root[k];
      s1 += wk * r;
      s2 += wk * r * r;
    }
  } else {
    for (int k = lane; k < K; k += 32) {
      const double p = z[wid * K + k], wk = w[wid * K + k];
      s1 += wk * log(p);
      s2 += wk * log1p(-p);
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    double* o = wid == n ? root_m : gm + 2 * wid;
    o[0] = s1;
    o[1] = s2;
  }
}

// One warp per (i, k) row (row n*K: the root row).  Per group the count sufficient statistics
// S_i = sum_j y_ij and C_i = sum_j lgamma(y_ij + 1) are summed by the row's lanes.
__global__ void __launch_bounds__(256) k_gamma_tables(int64_t n, int K, int J, double alpha,
                                                      const float* __restrict__ mu, const float* __restrict__ rm,
                                                      const float* __restrict__ rv, const int32_t* __restrict__ y,
                                                      const double* __restrict__ q,
                                                      const double* __restrict__ z, double* __restrict__ f_root,
                                                      double* __restrict__ f) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row > n * K) return;
  if (row == n * K) {
    const double m = rm[0], v = rv[0];
    for (int k = lane; k < K; k += 32) {
      const double r = mu[k], dr = r - m;
      f_root[k] = -0.5 * r * r + 0.5 * log(v) + 0.5 * dr * dr / v;  // the 2 pi terms cancel
    }
    return;
  }
  const int64_t i = row / K;
  const int k = (int)(row - i * K);
  double S = 0.0, Cy = 0.0;
  for (int j = lane; j < J; j += 32) {
    const double yy = y[i * J + j];
    S += yy;
    Cy += lgamma(yy + 1.0);
  }
  S = warp_sum(S);
  Cy = warp_sum(Cy);
  const double muk = mu[k], bk = alpha * exp(-muk);
  const double ak = alpha * (log(alpha) - muk) - lgamma(alpha);       // alpha log(rate_k) - lgamma(alpha)
  const double sq = q[2 * i], tq = q[2 * i + 1];
  const double cq = sq * log(tq) - lgamma(sq);
  const double* zi = z + i * K;
  double* fr = f + row * K;
  for (int kp = lane; kp < K; kp += 32) {
    const double l = zi[kp], ll = log(l);
    const double prior = ak + (alpha - 1.0) * ll - bk * l;
    const double lik = S * ll - J * l - Cy;
    const double lq = cq + (sq - 1.0) * ll - tq * l;
    fr[kp] = prior + lik - lq;
  }
}

// Mean parameters under the weights: groups (E l, E ln l) [n][2], root (E mu, E mu^2) [2].
__global__ void __launch_bounds__(256) k_gamma_moments(int64_t n, int K, const double* __restrict__ w_root,
                                                       const float* __restrict__ mu,
                                                       const double* __restrict__ w,
                                                       const double* __restrict__ z, double* __restrict__ root_m,
                                                       double* __restrict__ gm) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wid > n) return;
  double s1 = 0.0, s2 = 0.0;
  if (wid == n) {
    for (int k = lane; k < K; k += 32) {
      const double r = mu[k], wk = w_root[k];
      s1 += wk * r;
      s2 += wk * r * r;
    }
  } else {
    for (int k = lane; k < K; k += 32) {
      const double l = z[wid * K + k], wk = w[wid * K + k];
      s1 += wk * l;
      s2 += wk * log(l);
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    double* o = wid == n ? root_m : gm + 2 * wid;
    o[0] = s1;
    o[1] = s2;
  }
}

cudaError_t launch_gamma_sample(int64_t n, int K, uint64_t seed, int32_t iter, const double* q, double* z,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint32_t iterword = kGammaTag | ((uint32_t)iter & 0xffffffu);
  k_gamma_sample<<<(unsigned)((n * K + 255) / 256), 256, 0, st>>>(
      n, K, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)), iterword, q, z);
  return cudaGetLastError();
}

cudaError_t launch_beta_sample(int64_t n, int K, uint64_t seed, int32_t iter, const double* q, double* z,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_beta_sample<<<(unsigned)((n * K + 255) / 256), 256, 0, st>>>(n, K, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)),
                                                                 (uint32_t)iter, q, z);
  return cudaGetLastError();
}

cudaError_t launch_beta_tables(int64_t n, int K, double kappa, const float* mu, const float* rm, const float* rv,
                               const int32_t* y, const int32_t* N, const double* q, const double* z, double* f_root,
                               double* f, cudaStream_t st) {
  const int64_t rows = n * K + 1;
  k_beta_tables<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(n, K, kappa, mu, rm, rv, y, N, q, z, f_root, f);
  return cudaGetLastError();
}

cudaError_t launch_beta_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                                const double* z, double* root_m, double* gm, cudaStream_t st) {
  k_beta_moments<<<(unsigned)((n + 1 + 7) / 8), 256, 0, st>>>(n, K, w_root, mu, w, z, root_m, gm);
  return cudaGetLastError();
}

cudaError_t launch_gamma_tables(int64_t n, int K, int J, double alpha, const float* mu, const float* rm, const float* rv,
                                const int32_t* y, const double* q, const double* z, double* f_root, double* f,
                                cudaStream_t st) {
  const int64_t rows = n * K + 1;
  k_gamma_tables<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(n, K, J, alpha, mu, rm, rv, y, q, z, f_root, f);
  return cudaGetLastError();
}

cudaError_t launch_gamma_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                                 const double* z, double* root_m, double* gm, cudaStream_t st) {
  k_gamma_moments<<<(unsigned)((n + 1 + 7) / 8), 256, 0, st>>>(n, K, w_root, mu, w, z, root_m, gm);
  return cudaGetLastError();
}

}  // namespace qem
