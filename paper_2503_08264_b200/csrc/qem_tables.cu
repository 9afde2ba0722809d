// qem_tables.cu -- the MPIW E-step on EXPLICIT log-factor tables (qem_estep_tables, include/qem.h).
//
// Eq. 7c for a root with K samples and n plate instances below it, each with K
// samples, when the caller has already tabulated the log-factors:
//   f_root(k)        = log p(root^k) - log q(root^k)
//   f_i(k, k')       = log p(z_i^k', x_i | root^k) - log q(z_i^k')
// Plate elimination:
//   g_i(k)   = lse_k' f_i(k, k') - ln K                         (k_tab_fwd, one warp per row)
//   a(k)     = f_root(k) + sum_i g_i(k)                          (k_tab_plate + k_tab_root, fixed order)
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

// One W-lane group per (i, k) row (W = 32 for K > 128, else 8: short rows would leave most of a
// warp's lanes idle and pay 5 shuffle rounds per reduction).
template <int W>
__global__ void __launch_bounds__(kTabThreads) k_tab_fwd(int64_t rows, int K, const double* __restrict__ f,
                                                         double* __restrict__ g) {
  const int lane = threadIdx.x & (W - 1);
  const int64_t row = (int64_t)blockIdx.x * (kTabThreads / W) + (threadIdx.x / W);
  const bool live = row < rows;  // whole warps stay converged for the shuffles
  const double* fr = f + (live ? row : 0) * K;
  double m = -CUDART_INF;
  if (live)
    for (int k = lane; k < K; k += W) m = fmax(m, fr[k]);
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  double s = 0.0;
  if (live && m > -CUDART_INF)
    for (int k = lane; k < K; k += W) s += exp(fr[k] - m);
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  // an all -inf row has g = -inf (its root samples then carry zero weight); NaN / +inf propagate
  if (live && lane == 0) g[row] = m == -CUDART_INF ? -CUDART_INF : m + log(s) - log((double)K);
}

// Plate sum, stage 1: block b sums g_i(k) over its contiguous chunk of instances (index order)
// into part[b][k]; stage 2 (k_tab_root) adds the parts in block order -- deterministic.
__global__ void __launch_bounds__(128) k_tab_plate(int64_t n, int K, int64_t chunk, const double* __restrict__ g,
                                                   double* __restrict__ part) {
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = i0 + chunk < n ? i0 + chunk : n;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) s += g[i * K + k];
    part[(int64_t)blockIdx.x * K + k] = s;
  }
}

__global__ void __launch_bounds__(1024) k_tab_root(int nparts, int K, const double* __restrict__ f_root,
                                                   const double* __restrict__ part, double* log_pe, double* w_root) {
  extern __shared__ double a[];  // [K] + [nsub][K] sub-sums
  __shared__ double scratch[32];
  // nsub = blockDim / K sub-sums per k over parts b = sub, sub + nsub, ... (increasing), then added
  // in sub order: a fixed association, deterministic
  const int nsub = K < (int)blockDim.x ? (int)blockDim.x / K : 1;
  double* sub = a + K;
  for (int t = threadIdx.x; t < nsub * K; t += blockDim.x) {
    const int k = t % K, j = t / K;
    double s = 0.0;
    for (int b = j; b < nparts; b += nsub) s += part[(int64_t)b * K + k];
    sub[j * K + k] = s;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = f_root[k];
    for (int j = 0; j < nsub; ++j) s += sub[j * K + k];
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
  const int64_t i = blockIdx.x / kblocks;  // one block per (instance, blockDim columns)
  const int kp = (int)(blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
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

// a(k) = f_root(k) + sum_i g_i(k) (fixed order, `scratch` >= min(n, 296) x K doubles), then
// log Pe = lse a - ln K and w_root = softmax a.
cudaError_t launch_plate_root(int64_t n, int K, const double* f_root, const double* g, double* scratch,
                              double* log_pe, double* w_root, cudaStream_t st) {
  const int64_t parts = n < 148 * 2 ? n : 148 * 2, chunk = parts ? (n + parts - 1) / parts : 0;
  const int nparts = parts ? (int)((n + chunk - 1) / chunk) : 0;
  if (nparts) k_tab_plate<<<nparts, 128, 0, st>>>(n, K, chunk, g, scratch);
  const int nsub = K < 1024 ? 1024 / K : 1;
  const size_t smem = (size_t)K * (1 + nsub) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_tab_root, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_tab_root<<<1, 1024, smem, st>>>(nparts, K, f_root, scratch, log_pe, w_root);
  return cudaGetLastError();
}

cudaError_t launch_estep_tables(int64_t n, int K, const double* f_root, const double* f, double* g, double* log_pe,
                                double* w_root, double* w, cudaStream_t st) {
  if (n > 0) {
    const int64_t rows = n * K;
    if (K > 128) {
      k_tab_fwd<32><<<(unsigned)((rows + kTabThreads / 32 - 1) / (kTabThreads / 32)), kTabThreads, 0, st>>>(rows, K, f, g);
    } else {
      k_tab_fwd<8><<<(unsigned)((rows + kTabThreads / 8 - 1) / (kTabThreads / 8)), kTabThreads, 0, st>>>(rows, K, f, g);
    }
  }
  // stage-1 parts live in w (n x K >= parts x K), which the backward overwrites afterwards
  cudaError_t e = launch_plate_root(n, K, f_root, g, w, log_pe, w_root, st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const int threads = K >= kTabThreads ? kTabThreads : (K + 31) / 32 * 32;
    const int kblocks = (K + threads - 1) / threads;
    k_tab_bwd<<<(unsigned)(n * kblocks), threads, 0, st>>>(K, kblocks, f, g, w_root, w);
  }
  return cudaGetLastError();
}

}  // namespace qem
