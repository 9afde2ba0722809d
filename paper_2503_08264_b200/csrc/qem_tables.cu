// qem_tables.cu -- the MPIW E-step on EXPLICIT log-factor tables (qem_estep_tables, include/qem.h).
//
// Eq. 7c for a root with K samples and n plate instances below it, each with K
// samples, when the caller has already tabulated the log-factors:
//   f_root(k)        = log p(root^k) - log q(root^k)
//   f_i(k, k')       = log p(z_i^k', x_i | root^k) - log q(z_i^k')
// Plate elimination:
//   g_i(k)   = lse_k' f_i(k, k') - ln K                         (k_tab_fwd, one warp per row)
//   a(k)     = f_root(k) + sum_i g_i(k)                          (k_tab_root, fixed order)
//   log Pe   = lse_k a(k) - ln K,   w_root(k) = softmax_k a(k)   (Eq. 7a/7c)
//   w_i(k')  = sum_k w_root(k) exp(f_i(k, k') - ln K - g_i(k))   (k_tab_bwd; Eq. 7a marginals)
// fp64 throughout (exp/log from libdevice).  This path carries any factor kind the caller can
// tabulate (discrete latents, crossed effects) and pins the reduction structure of the fused
// kernels independently of their factor arithmetic (SURVEY.md §8(b) "qem_estep_from_factors").
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

constexpr int kTabThreads = 256;

__global__ void __launch_bounds__(kTabThreads) k_tab_fwd(int64_t rows, int K, const double* __restrict__ f,
                                                         double* __restrict__ g) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (kTabThreads / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const double* fr = f + row * K;
  double m = -CUDART_INF;
  for (int k = lane; k < K; k += 32) m = fmax(m, fr[k]);
  m = warp_max(m);
  double s = 0.0;
  if (m > -CUDART_INF)
    for (int k = lane; k < K; k += 32) s += exp(fr[k] - m);
  s = warp_sum(s);
  // an all -inf row has g = -inf (its root samples then carry zero weight); NaN / +inf propagate
  if (lane == 0) g[row] = m == -CUDART_INF ? -CUDART_INF : m + log(s) - log((double)K);
}

__global__ void __launch_bounds__(1024) k_tab_root(int64_t n, int K, const double* __restrict__ f_root,
                                                   const double* __restrict__ g, double* log_pe, double* w_root) {
  extern __shared__ double a[];  // [K]
  __shared__ double scratch[32];
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = f_root[k];
    for (int64_t i = 0; i < n; ++i) s += g[i * K + k];  // index order: deterministic
    a[k] = s;
  }
  __syncthreads();
  double m = -CUDART_INF;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, a[k]);
  m = block_max(m, scratch);
  double s = 0.0;
  if (m > -CUDART_INF)
    for (int k = threadIdx.x; k < K; k += blockDim.x) s += exp(a[k] - m);
  s = block_sum(s, scratch);
  const double lse = m + log(s);
  if (threadIdx.x == 0) *log_pe = m == -CUDART_INF ? -CUDART_INF : lse - log((double)K);
  // degenerate evidence (every a(k) = -inf): weights are NaN, log Pe = -inf (SPEC.md:317's error, as data)
  for (int k = threadIdx.x; k < K; k += blockDim.x) w_root[k] = m == -CUDART_INF ? CUDART_NAN : exp(a[k] - lse);
}

__global__ void __launch_bounds__(kTabThreads) k_tab_bwd(int K, int kblocks, const double* __restrict__ f,
                                                         const double* __restrict__ g,
                                                         const double* __restrict__ w_root, double* __restrict__ w) {
  const int64_t i = blockIdx.x / kblocks;  // one block per (instance, 256 columns)
  const int kp = (int)(blockIdx.x % kblocks) * kTabThreads + threadIdx.x;
  if (kp >= K) return;
  const double* fi = f + i * K * K;
  const double* gi = g + i * K;
  const double lk = log((double)K);
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const double wr = w_root[k];
    if (wr != 0.0) acc += wr * exp(fi[(int64_t)k * K + kp] - lk - gi[k]);  // skip zero-weight rows (g may be -inf)
  }
  w[i * K + kp] = acc;
}

cudaError_t launch_estep_tables(int64_t n, int K, const double* f_root, const double* f, double* g, double* log_pe,
                                double* w_root, double* w, cudaStream_t st) {
  if (n > 0) {
    const int64_t rows = n * K;
    const int64_t blocks = (rows + kTabThreads / 32 - 1) / (kTabThreads / 32);
    k_tab_fwd<<<(unsigned)blocks, kTabThreads, 0, st>>>(rows, K, f, g);
  }
  const size_t smem = (size_t)K * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_tab_root, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_tab_root<<<1, 1024, smem, st>>>(n, K, f_root, g, log_pe, w_root);
  if (n > 0) {
    const int kblocks = (K + kTabThreads - 1) / kTabThreads;
    k_tab_bwd<<<(unsigned)(n * kblocks), kTabThreads, 0, st>>>(K, kblocks, f, g, w_root, w);
  }
  return cudaGetLastError();
}

}  // namespace qem
