// qem_separable.cu -- the MPIW E-step for SEPARABLE log-factors, on chip: no n x K x K table.
//
// Eq. 7c with plate elimination for a root with K samples and n plate
// instances, when every log-factor splits into a row part and a column part:
//   f_i(k, k') = a_k + sum_{r<R} b_k[r] phi_i(k')[r] + psi_i(k'),   R <= 3
// (rows: the root sample k; columns: instance i's sample k').  The Gamma-Poisson and Beta-Binomial
// hierarchies of NEXT row f1 are of this form (R32, R37): their table builders wrote n K^2
// fp64 entries to HBM and read them twice (262 MB per iteration at n = 2000, K = 128); here each
// group's K (R + 1) column values are staged in shared memory and every pair is evaluated where it
// is used, in fp64 (the same arithmetic the table engine applied to the stored entries):
//   g_i(k)   = lse_k' f_i(k, k') - ln K                          (k_sep_fwd: block per group, thread per row)
//   a(k)     = f_root(k) + sum_i g_i(k), log Pe, w_root          (launch_plate_root, shared with qem_tables.cu)
//   w_i(k')  = sum_k w_root(k) exp(f_i(k, k') - ln K - g_i(k))   (k_sep_bwd: block per group, thread per column)
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

template <int R>
__device__ __forceinline__ double sep_pair(const double* row, const double* col) {
  double v = row[0] + col[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v = fma(row[1 + r], col[r], v);
  return v;
}

// Forward: block = one group, threads over rows k; the group's columns [K][R+1] in shared memory
// (broadcast reads).  Two passes over the columns: max, then the sum of exponentials (fp64).
template <int R>
__global__ void __launch_bounds__(256) k_sep_fwd(int64_t n, int K, const double* __restrict__ rows,
                                                 const double* __restrict__ cols, double* __restrict__ g) {
  extern __shared__ double sc[];  // [K][R+1]
  const int64_t i = blockIdx.x;
  const double* ci = cols + (size_t)i * K * (R + 1);
  for (int e = threadIdx.x; e < K * (R + 1); e += blockDim.x) sc[e] = ci[e];
  __syncthreads();
  const double lk = log((double)K);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double row[1 + R];
#pragma unroll
    for (int r = 0; r <= R; ++r) row[r] = rows[(size_t)k * (1 + R) + r];
    double m = -CUDART_INF;
    for (int kp = 0; kp < K; ++kp) m = fmax(m, sep_pair<R>(row, sc + kp * (R + 1)));
    double s = 0.0;
    if (m > -CUDART_INF)
      for (int kp = 0; kp < K; ++kp) s += exp(sep_pair<R>(row, sc + kp * (R + 1)) - m);
    // an all -inf row has g = -inf (its root sample then carries zero weight); NaN / +inf propagate
    g[i * K + k] = m == -CUDART_INF ? -CUDART_INF : m + log(s) - lk;
  }
}

// Backward: block = one group, threads over columns k'; rows, g_i and ln w_root in shared memory.
template <int R>
__global__ void __launch_bounds__(256) k_sep_bwd(int64_t n, int K, const double* __restrict__ rows,
                                                 const double* __restrict__ cols, const double* __restrict__ g,
                                                 const double* __restrict__ w_root, double* __restrict__ w) {
  extern __shared__ double sr[];  // [K][R+2]: a_k, b_k[R], ln w_root(k) - ln K - g_i(k)
  const int64_t i = blockIdx.x;
  const double lk = log((double)K);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
#pragma unroll
    for (int r = 0; r <= R; ++r) sr[k * (R + 2) + r] = rows[(size_t)k * (1 + R) + r];
    const double wr = w_root[k];
    // zero-weight rows drop out (their g may be -inf): -inf here makes exp() 0 exactly
    sr[k * (R + 2) + R + 1] = wr > 0.0 ? log(wr) - lk - g[i * K + k] : -CUDART_INF;
  }
  __syncthreads();
  const double* ci = cols + (size_t)i * K * (R + 1);
  for (int kp = threadIdx.x; kp < K; kp += blockDim.x) {
    double col[R + 1];
#pragma unroll
    for (int r = 0; r <= R; ++r) col[r] = ci[(size_t)kp * (R + 1) + r];
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
      const double* rw = sr + k * (R + 2);
      const double c = rw[R + 1];
      if (c > -CUDART_INF) acc += exp(sep_pair<R>(rw, col) + c);
    }
    w[i * K + kp] = acc;
  }
}

template <int R>
static cudaError_t sep_launch(int64_t n, int K, const double* f_root, const double* rows, const double* cols,
                              double* g, double* log_pe, double* w_root, double* w, cudaStream_t st) {
  const int threads = K >= 256 ? 256 : (K + 31) / 32 * 32;
  if (n > 0) {
    const size_t sm = (size_t)K * (R + 1) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_sep_fwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_sep_fwd<R><<<(unsigned)n, threads, sm, st>>>(n, K, rows, cols, g);
  }
  // stage-1 plate parts live in w (n x K >= parts x K), which the backward overwrites afterwards
  cudaError_t e = launch_plate_root(n, K, f_root, g, w, log_pe, w_root, st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const size_t sm = (size_t)K * (R + 2) * sizeof(double);
    e = cudaFuncSetAttribute(k_sep_bwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_sep_bwd<R><<<(unsigned)n, threads, sm, st>>>(n, K, rows, cols, g, w_root, w);
  }
  return cudaGetLastError();
}

cudaError_t launch_estep_separable(int64_t n, int K, int R, const double* f_root, const double* rows,
                                   const double* cols, double* g, double* log_pe, double* w_root, double* w,
                                   cudaStream_t st) {
  switch (R) {
    case 0: return sep_launch<0>(n, K, f_root, rows, cols, g, log_pe, w_root, w, st);
    case 1: return sep_launch<1>(n, K, f_root, rows, cols, g, log_pe, w_root, w, st);
    case 2: return sep_launch<2>(n, K, f_root, rows, cols, g, log_pe, w_root, w, st);
    case 3: return sep_launch<3>(n, K, f_root, rows, cols, g, log_pe, w_root, w, st);
  }
  return cudaErrorInvalidValue;
}

// ---- separable factors of the Gamma-Poisson and Beta-Binomial hierarchies (qem_gamma.cu's models)
// Root factor (both): f_root(k) = log N(mu^k; 0, 1) - log N(mu^k; m, v) (the 2 pi terms cancel).
__device__ __forceinline__ double root_factor(double r, double m, double v) {
  const double dr = r - m;
  return -0.5 * r * r + 0.5 * log(v) + 0.5 * dr * dr / v;
}

// Gamma-Poisson: log Gamma(l; alpha, beta_k) = alpha ln beta_k - lgamma(alpha) + (alpha - 1) ln l - beta_k l,
// beta_k = alpha e^-mu^k  ->  row (a_k, b_k) = (alpha (ln alpha - mu^k) - lgamma(alpha), -beta_k);
// column (phi, psi) = (l, (alpha - 1) ln l + sum_j log Pois(y_ij; l) - log Gamma(l; k_i, th_i)).
// Thread per (i, k') column (row n K + k: row k and the root factor).
__global__ void __launch_bounds__(256) k_gamma_cols(int64_t n, int K, int J, double alpha, const float* __restrict__ mu,
                                                    const float* __restrict__ rm, const float* __restrict__ rv,
                                                    const int32_t* __restrict__ y, const double* __restrict__ q,
                                                    const double* __restrict__ z, double* __restrict__ f_root,
                                                    double* __restrict__ rows, double* __restrict__ cols) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (n + 1) * K) return;
  if (t >= n * K) {
    const int k = (int)(t - n * K);
    const double muk = mu[k];
    f_root[k] = root_factor(muk, rm[0], rv[0]);
    rows[2 * k] = alpha * (log(alpha) - muk) - lgamma(alpha);
    rows[2 * k + 1] = -alpha * exp(-muk);
    return;
  }
  const int64_t i = t / K;
  double S = 0.0, Cy = 0.0;
  for (int j = 0; j < J; ++j) {
    const double yy = y[i * J + j];
    S += yy;
    Cy += lgamma(yy + 1.0);
  }
  const double sq = q[2 * i], tq = q[2 * i + 1];
  const double l = z[t], ll = log(l);
  const double lik = S * ll - J * l - Cy;
  const double lq = sq * log(tq) - lgamma(sq) + (sq - 1.0) * ll - tq * l;
  cols[2 * t] = l;
  cols[2 * t + 1] = (alpha - 1.0) * ll + lik - lq;
}

// Beta-Binomial: log Beta(p; kappa s_k, kappa (1 - s_k)) = lgamma(kappa) - lgamma(kappa s_k) - lgamma(kappa (1 - s_k))
// + (kappa s_k - 1) ln p + (kappa (1 - s_k) - 1) ln(1 - p)  ->  row (a_k, kappa s_k, kappa (1 - s_k));
// column (ln p, ln(1 - p), -ln p - ln(1 - p) + log Bin(y_i; N_i, p) - log Beta(p; a_i, b_i)).
__global__ void __launch_bounds__(256) k_beta_cols(int64_t n, int K, double kappa, const float* __restrict__ mu,
                                                   const float* __restrict__ rm, const float* __restrict__ rv,
                                                   const int32_t* __restrict__ y, const int32_t* __restrict__ N,
                                                   const double* __restrict__ q, const double* __restrict__ z,
                                                   double* __restrict__ f_root, double* __restrict__ rows,
                                                   double* __restrict__ cols) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (n + 1) * K) return;
  if (t >= n * K) {
    const int k = (int)(t - n * K);
    const double muk = mu[k], sk = 1.0 / (1.0 + exp(-muk)), pa = kappa * sk, pb = kappa * (1.0 - sk);
    f_root[k] = root_factor(muk, rm[0], rv[0]);
    rows[3 * k] = lgamma(kappa) - lgamma(pa) - lgamma(pb);
    rows[3 * k + 1] = pa;
    rows[3 * k + 2] = pb;
    return;
  }
  const int64_t i = t / K;
  const double yy = y[i], nn = N[i];
  const double cb = lgamma(nn + 1.0) - lgamma(yy + 1.0) - lgamma(nn - yy + 1.0);
  const double qa = q[2 * i], qb = q[2 * i + 1];
  const double cq = lgamma(qa + qb) - lgamma(qa) - lgamma(qb);
  const double p = z[t], lp = log(p), l1 = log1p(-p);
  const double lik = cb + yy * lp + (nn - yy) * l1;
  const double lq = cq + (qa - 1.0) * lp + (qb - 1.0) * l1;
  cols[3 * t] = lp;
  cols[3 * t + 1] = l1;
  cols[3 * t + 2] = -lp - l1 + lik - lq;
}

cudaError_t launch_gamma_cols(int64_t n, int K, int J, double alpha, const float* mu, const float* rm, const float* rv,
                              const int32_t* y, const double* q, const double* z, double* f_root, double* rows,
                              double* cols, cudaStream_t st) {
  const int64_t t = (n + 1) * K;
  k_gamma_cols<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(n, K, J, alpha, mu, rm, rv, y, q, z, f_root, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_beta_cols(int64_t n, int K, double kappa, const float* mu, const float* rm, const float* rv,
                             const int32_t* y, const int32_t* N, const double* q, const double* z, double* f_root,
                             double* rows, double* cols, cudaStream_t st) {
  const int64_t t = (n + 1) * K;
  k_beta_cols<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(n, K, kappa, mu, rm, rv, y, N, q, z, f_root, rows, cols);
  return cudaGetLastError();
}

}  // namespace qem
