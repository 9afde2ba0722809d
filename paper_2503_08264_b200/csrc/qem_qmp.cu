// qem_qmp.cu -- non-factorised massively parallel proposal Q_MP with its parent-copy schemes
// (App. A; R43), on the conjugate two-level Gaussian
// hierarchy  mu ~ N(0, pv), z_i | mu ~ N(mu, gv), x_ij | z_i ~ N(z_i, ov)  with the single-sample
// proposal  Q(mu) = N(m, v), Q(z_i | mu) = N(alpha_i + beta_i mu, s_i).
//
// Every child copy k' is drawn from its conditional at ONE copy of the parent,
//   z_i^k' = alpha_i + beta_i mu^copy[i][k'] + sqrt(s_i) eps_i^k',
// and its proposal density is, by scheme,
//   permutation  q_MP,i(k') = N(z_i^k'; alpha_i + beta_i mu^copy[i][k'], s_i)     (copy[i] a permutation)
//   mixture      q_MP,i(k') = (1/K) sum_k N(z_i^k'; alpha_i + beta_i mu^k, s_i)   (copy[i][k'] iid uniform)
// The MPIW log-factor (Eq. 7c) is separable in (k, k'):
//   f_i(k, k') = log N(z_i^k'; mu^k, gv) + sum_j log N(x_ij; z_i^k', ov) - log q_MP,i(k')
//              = a_k + b_k z_i^k' + psi_i(k'),   a_k = -ln(2 pi gv)/2 - mu_k^2 / (2 gv),  b_k = mu_k / gv,
//                psi_i(k') = -z^2 / (2 gv) + sum_j log N(x_ij; z, ov) - log q_MP,i(k'),
// so the E-step runs on chip through qem_estep_separable (R = 1): no n x K x K table.  All fp64.
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

namespace {
constexpr double kLn2Pi = 1.8378770664093454835606594728112;

// block = one group, threads over the child copies k'; the K parent samples in shared memory
__global__ void __launch_bounds__(256) k_qmp_cols(int K, int J, int scheme, double gv, double ov,
                                                  const float* __restrict__ mu, const double* __restrict__ q,
                                                  const int32_t* __restrict__ copy, const float* __restrict__ eps,
                                                  const float* __restrict__ x, double* __restrict__ z,
                                                  double* __restrict__ cols) {
  extern __shared__ double smu[];  // [K]
  const int64_t i = blockIdx.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x) smu[k] = (double)mu[k];
  __syncthreads();
  const double alpha = q[3 * i], beta = q[3 * i + 1], s = q[3 * i + 2];
  const double sd = sqrt(s), lns = -0.5 * (kLn2Pi + log(s)), lno = -0.5 * (kLn2Pi + log(ov));
  const double h_s = 0.5 / s, h_o = 0.5 / ov, h_g = 0.5 / gv;
  const float* xi = x + (size_t)i * J;
  for (int kp = threadIdx.x; kp < K; kp += blockDim.x) {
    const int c = copy[(size_t)i * K + kp];
    const double zz = alpha + beta * smu[c] + sd * (double)eps[(size_t)i * K + kp];
    double ll = 0.0;
    for (int j = 0; j < J; ++j) {
      const double d = (double)xi[j] - zz;
      ll += lno - d * d * h_o;
    }
    double lq;
    if (scheme == 0) {  // permutation: the conditional at the copy that was used
      const double d = zz - (alpha + beta * smu[c]);
      lq = lns - d * d * h_s;
    } else {  // mixture over the K parent copies: max-shifted log-mean-exp
      double mx = -CUDART_INF;
      for (int k = 0; k < K; ++k) {
        const double d = zz - (alpha + beta * smu[k]);
        mx = fmax(mx, -d * d * h_s);
      }
      double sum = 0.0;
      for (int k = 0; k < K; ++k) {
        const double d = zz - (alpha + beta * smu[k]);
        sum += exp(-d * d * h_s - mx);
      }
      lq = lns + mx + log(sum) - log((double)K);
    }
    z[(size_t)i * K + kp] = zz;
    cols[((size_t)i * K + kp) * 2] = zz;
    cols[((size_t)i * K + kp) * 2 + 1] = -zz * zz * h_g + ll - lq;
  }
}

__global__ void k_qmp_rows(int K, double pv, double gv, const float* __restrict__ mu, const float* __restrict__ rm,
                           const float* __restrict__ rv, double* __restrict__ f_root, double* __restrict__ rows) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double m = (double)mu[k], qm = (double)rm[0], qv = (double)rv[0];
  const double dq = m - qm;
  f_root[k] = (-0.5 * (kLn2Pi + log(pv)) - m * m * (0.5 / pv)) - (-0.5 * (kLn2Pi + log(qv)) - dq * dq * (0.5 / qv));
  rows[2 * k] = -0.5 * (kLn2Pi + log(gv)) - m * m * (0.5 / gv);
  rows[2 * k + 1] = m / gv;
}

// one warp per row: rows 0..n-1 the groups (E z_i, E z_i^2 under w_i), row n the root (E mu, E mu^2)
__global__ void __launch_bounds__(128) k_qmp_moments(int64_t n, int K, const double* __restrict__ w_root,
                                                     const float* __restrict__ mu, const double* __restrict__ w,
                                                     const double* __restrict__ z, double* __restrict__ root_m,
                                                     double* __restrict__ gm) {
  const int64_t r = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r > n) return;
  double s1 = 0.0, s2 = 0.0;
  for (int k = lane; k < K; k += 32) {
    const double wk = r < n ? w[(size_t)r * K + k] : w_root[k];
    const double v = r < n ? z[(size_t)r * K + k] : (double)mu[k];
    s1 += wk * v;
    s2 += wk * v * v;
  }
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    double* dst = r < n ? gm + 2 * r : root_m;
    dst[0] = s1;
    dst[1] = s2;
  }
}
}  // namespace

cudaError_t launch_qmp_cols(int64_t n, int K, int J, int scheme, double pv, double gv, double ov, const float* mu,
                            const float* rm, const float* rv, const double* q, const int32_t* copy, const float* eps,
                            const float* x, double* z, double* f_root, double* rows, double* cols, cudaStream_t st) {
  k_qmp_rows<<<(K + 255) / 256, 256, 0, st>>>(K, pv, gv, mu, rm, rv, f_root, rows);
  if (n > 0) k_qmp_cols<<<(unsigned)n, 256, (size_t)K * sizeof(double), st>>>(K, J, scheme, gv, ov, mu, q, copy, eps, x, z, cols);
  return cudaGetLastError();
}

cudaError_t launch_qmp_moments(int64_t n, int K, const double* w_root, const float* mu, const double* w,
                               const double* z, double* root_m, double* gm, cudaStream_t st) {
  k_qmp_moments<<<(unsigned)((n + 1 + 3) / 4), 128, 0, st>>>(n, K, w_root, mu, w, z, root_m, gm);
  return cudaGetLastError();
}

}  // namespace qem
