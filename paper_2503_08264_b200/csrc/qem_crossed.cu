// qem_crossed.cu -- crossed effects (NEXT row f4, R33): observations whose factor has
// several parents on different plates, Bus-Breakdown-shaped (a delay's logit is
// YearBoroughWeight_yb + CompanyWeight_c(ybi) + JourneyTypeWeight_j(ybi), the company and journey
// weights picked out by per-observation index tables).
//
// Reading (R33): the crossed weights are global latents, so they join the root group and share
// its sample index k (R2); the plate below is the year-borough groups.  The group factor then
// couples both indices through every observation:
//   f_i(k, k') = log N(w_i^k'; mu^k, 1) + sum_j [y_ij eta - softplus(eta)] - log q_i(w_i^k'),
//   eta = w_i^k' + cw^k_{c_ij} + jw^k_{t_ij}
// -- a K x K x J contraction per group (the "rank-3 factor" of SURVEY.md §8(f)#4), written into
// explicit fp64 tables for qem_estep_tables.  Root samples: [R][K] fp32 with R = 1 + C + T
// (mu, the C company weights, the T journey-type weights), all N(0, 1) a priori.
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

constexpr int kCrossWarps = 8;

// One warp per (i, k) row; the row's per-observation offsets o_j = cw^k_{c_ij} + jw^k_{t_ij} and
// labels are staged in the warp's shared-memory slice, lanes run over k'.  Row n*K: f_root.
__global__ void __launch_bounds__(kCrossWarps * 32) k_crossed_tables(int64_t n, int K, int J, int C, int T,
                                                                     const float* __restrict__ rz,
                                                                     const float* __restrict__ rm,
                                                                     const float* __restrict__ rv,
                                                                     const float* __restrict__ z,
                                                                     const float* __restrict__ qm,
                                                                     const float* __restrict__ qv,
                                                                     const int32_t* __restrict__ comp,
                                                                     const int32_t* __restrict__ jtype,
                                                                     const uint8_t* __restrict__ y,
                                                                     double* __restrict__ f_root,
                                                                     double* __restrict__ f) {
  extern __shared__ double so[];  // [kCrossWarps][J] offsets
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kCrossWarps + wid;
  if (row > n * K) return;
  const int R = 1 + C + T;
  if (row == n * K) {  // f_root(k) = sum_r log N(r; 0, 1) - log N(r; m_r, v_r)
    for (int k = lane; k < K; k += 32) {
      double s = 0.0;
      for (int r = 0; r < R; ++r) {
        const double x = rz[(int64_t)r * K + k], v = rv[r], dx = x - (double)rm[r];
        s += -0.5 * x * x + 0.5 * log(v) + 0.5 * dx * dx / v;
      }
      f_root[k] = s;
    }
    return;
  }
  const int64_t i = row / K;
  const int k = (int)(row - i * K);
  double* o = so + (size_t)wid * J;
  for (int j = lane; j < J; j += 32)
    o[j] = (double)rz[(int64_t)(1 + comp[i * J + j]) * K + k] + (double)rz[(int64_t)(1 + C + jtype[i * J + j]) * K + k];
  __syncwarp();
  const double mu = rz[k], m = qm[i], v = qv[i];
  const uint8_t* yi = y + i * J;
  const float* zi = z + i * K;
  double* fr = f + row * K;
  for (int kp = lane; kp < K; kp += 32) {
    const double w = zi[kp];
    double lik = 0.0;
    for (int j = 0; j < J; ++j) {
      const double eta = w + o[j];
      lik += (yi[j] ? eta : 0.0) - (fmax(eta, 0.0) + log1p(exp(-fabs(eta))));
    }
    const double dw = w - mu, dq = w - m;
    // log N(w; mu, 1) - log N(w; m, v): the 2 pi terms cancel
    fr[kp] = -0.5 * dw * dw + 0.5 * log(v) + 0.5 * dq * dq / v + lik;
  }
}

// (E x, E x^2) under the weights: root dims [R][2] from w_root, groups [n][2] from w.
__global__ void __launch_bounds__(256) k_crossed_moments(int64_t n, int K, int R, const double* __restrict__ w_root,
                                                         const float* __restrict__ rz, const double* __restrict__ w,
                                                         const float* __restrict__ z, double* __restrict__ root_m,
                                                         double* __restrict__ gm) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wid >= n + R) return;
  const bool root = wid >= n;
  const int64_t r = wid - n;
  double s1 = 0.0, s2 = 0.0;
  for (int k = lane; k < K; k += 32) {
    const double x = root ? rz[r * K + k] : z[wid * K + k];
    const double wk = root ? w_root[k] : w[wid * K + k];
    s1 += wk * x;
    s2 += wk * x * x;
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    double* out = root ? root_m + 2 * r : gm + 2 * wid;
    out[0] = s1;
    out[1] = s2;
  }
}

// ---- the same E-step on chip (no n x K x K table): the pair factor is evaluated where it is used.
// Per group (one block): the group's samples, labels and the crossed root weights' index tables in
// shared memory; the forward's thread per row k keeps its J offsets o_j = cw^k_{c_j} + jw^k_{t_j}
// in shared memory and takes an online (max, sum) over k'; the backward's thread per column k'
// recomputes the pair against every row.  fp64, the arithmetic of k_crossed_tables.
struct CrossedArgs {
  int64_t n;
  int K, J, C, T;
  const float *rz, *z, *qm, *qv;
  const int32_t *comp, *jtype;
  const uint8_t* y;
};

__device__ __forceinline__ double crossed_pair(double w, double mu, const double* o, const uint8_t* yi, int J,
                                               double colterm) {
  double lik = 0.0;
  for (int j = 0; j < J; ++j) {
    const double eta = w + o[j];
    lik += (yi[j] ? eta : 0.0) - (fmax(eta, 0.0) + log1p(exp(-fabs(eta))));
  }
  const double dw = w - mu;
  return -0.5 * dw * dw + colterm + lik;
}

// Four threads per row (forward) / per column (backward), each over every 4th partner index, their
// partial (max, sum) / sums combined by shuffles: the fp64 softplus chains are long, so the block
// needs the threads for latency (one group per block).
constexpr int kCrossSplit = 4;

// shared memory: [K] w, [K] column terms, [blockDim / 4][J] row offsets, [J] labels (bytes)
__global__ void __launch_bounds__(256) k_crossed_fwd(CrossedArgs a, double* __restrict__ g) {
  extern __shared__ double sm[];
  const int K = a.K, J = a.J, tid = threadIdx.x, part = tid % kCrossSplit;
  const int rows_per_pass = blockDim.x / kCrossSplit, rr = tid / kCrossSplit;
  const int64_t i = blockIdx.x;
  double* sw = sm;
  double* sc = sw + K;
  double* so = sc + K;  // [rows_per_pass][J]
  uint8_t* sy = reinterpret_cast<uint8_t*>(so + (size_t)rows_per_pass * J);
  const double m = a.qm[i], v = a.qv[i];
  for (int k = tid; k < K; k += blockDim.x) {
    const double w = a.z[i * K + k], dq = w - m;
    sw[k] = w;
    sc[k] = 0.5 * log(v) + 0.5 * dq * dq / v;  // - log N(w; m, v) + the cancelled 2 pi
  }
  for (int j = tid; j < J; j += blockDim.x) sy[j] = a.y[i * J + j];
  const double lk = log((double)K);
  for (int k0 = 0; k0 < K; k0 += rows_per_pass) {
    __syncthreads();  // (first pass: the column data; later: the previous rows' offsets are consumed)
    const int k = k0 + rr;
    double* o = so + (size_t)rr * J;
    if (k < K)
      for (int j = part; j < J; j += kCrossSplit)
        o[j] = (double)a.rz[(int64_t)(1 + a.comp[i * J + j]) * K + k] +
               (double)a.rz[(int64_t)(1 + a.C + a.jtype[i * J + j]) * K + k];
    __syncthreads();
    double mx = -CUDART_INF, s = 0.0;
    if (k < K) {
      const double mu = a.rz[k];
      for (int kp = part; kp < K; kp += kCrossSplit) {
        const double t = crossed_pair(sw[kp], mu, o, sy, J, sc[kp]);
        if (t > mx) {
          s = (mx == -CUDART_INF ? 0.0 : s * exp(mx - t)) + 1.0;
          mx = t;
        } else {
          s += exp(t - mx);
        }
      }
    }
#pragma unroll
    for (int off = 1; off < kCrossSplit; off <<= 1) {  // combine the row's partial (max, sum)
      const double om = __shfl_xor_sync(0xffffffffu, mx, off), os = __shfl_xor_sync(0xffffffffu, s, off);
      const double nm = fmax(mx, om);
      s = (mx == -CUDART_INF ? 0.0 : s * exp(mx - nm)) + (om == -CUDART_INF ? 0.0 : os * exp(om - nm));
      mx = nm;
    }
    if (k < K && part == 0) g[i * K + k] = mx == -CUDART_INF ? -CUDART_INF : mx + log(s) - lk;
  }
}

// shared memory: [K] c_k = ln w_root(k) - ln K - g_i(k), [K] mu^k, [K][J] row offsets, [J] labels
__global__ void __launch_bounds__(256) k_crossed_bwd(CrossedArgs a, const double* __restrict__ g,
                                                     const double* __restrict__ w_root, double* __restrict__ w) {
  extern __shared__ double sm[];
  const int K = a.K, J = a.J, tid = threadIdx.x, part = tid % kCrossSplit;
  const int cols_per_pass = blockDim.x / kCrossSplit;
  const int64_t i = blockIdx.x;
  double* sc = sm;
  double* smu = sc + K;
  double* so = smu + K;  // [K][J]
  uint8_t* sy = reinterpret_cast<uint8_t*>(so + (size_t)K * J);
  const double lk = log((double)K);
  for (int k = tid; k < K; k += blockDim.x) {
    const double wr = w_root[k];
    sc[k] = wr > 0.0 ? log(wr) - lk - g[i * K + k] : -CUDART_INF;  // zero-weight rows drop out
    smu[k] = a.rz[k];
  }
  for (int e = tid; e < K * J; e += blockDim.x) {
    const int k = e / J, j = e - k * J;
    so[e] = (double)a.rz[(int64_t)(1 + a.comp[i * J + j]) * K + k] + (double)a.rz[(int64_t)(1 + a.C + a.jtype[i * J + j]) * K + k];
  }
  for (int j = tid; j < J; j += blockDim.x) sy[j] = a.y[i * J + j];
  __syncthreads();
  const double m = a.qm[i], v = a.qv[i];
  for (int kp0 = 0; kp0 < K; kp0 += cols_per_pass) {
    const int kp = kp0 + tid / kCrossSplit;
    double acc = 0.0;
    if (kp < K) {
      const double wv = a.z[i * K + kp], dq = wv - m;
      const double col = 0.5 * log(v) + 0.5 * dq * dq / v;
      for (int k = part; k < K; k += kCrossSplit) {
        const double c = sc[k];
        if (c > -CUDART_INF) acc += exp(crossed_pair(wv, smu[k], so + (size_t)k * J, sy, J, col) + c);
      }
    }
#pragma unroll
    for (int off = 1; off < kCrossSplit; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (kp < K && part == 0) w[i * K + kp] = acc;
  }
}

__global__ void k_crossed_root(int K, int R, const float* __restrict__ rz, const float* __restrict__ rm,
                               const float* __restrict__ rv, double* __restrict__ f_root) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < R; ++r) {
      const double x = rz[(int64_t)r * K + k], v = rv[r], dx = x - (double)rm[r];
      s += -0.5 * x * x + 0.5 * log(v) + 0.5 * dx * dx / v;
    }
    f_root[k] = s;
  }
}

cudaError_t launch_crossed_estep(int64_t n, int K, int J, int C, int T, const float* rz, const float* rm,
                                 const float* rv, const float* z, const float* qm, const float* qv,
                                 const int32_t* comp, const int32_t* jtype, const uint8_t* y, double* f_root,
                                 double* g, double* log_pe, double* w_root, double* w, cudaStream_t st) {
  CrossedArgs a{n, K, J, C, T, rz, z, qm, qv, comp, jtype, y};
  k_crossed_root<<<(K + 127) / 128, 128, 0, st>>>(K, 1 + C + T, rz, rm, rv, f_root);
  const int threads = 256;  // kCrossSplit threads per row / column, 64 rows / columns per pass
  if (n > 0) {
    const size_t sf = (size_t)(2 * K + (size_t)(threads / kCrossSplit) * J) * sizeof(double) + J + 8;
    cudaError_t e = cudaFuncSetAttribute(k_crossed_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
    if (e != cudaSuccess) return e;
    k_crossed_fwd<<<(unsigned)n, threads, sf, st>>>(a, g);
  }
  cudaError_t e = launch_plate_root(n, K, f_root, g, w, log_pe, w_root, st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const size_t sb = (size_t)(2 * K + (size_t)K * J) * sizeof(double) + J + 8;
    e = cudaFuncSetAttribute(k_crossed_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    if (e != cudaSuccess) return e;
    k_crossed_bwd<<<(unsigned)n, threads, sb, st>>>(a, g, w_root, w);
  }
  return cudaGetLastError();
}

cudaError_t launch_crossed_tables(int64_t n, int K, int J, int C, int T, const float* rz, const float* rm,
                                  const float* rv, const float* z, const float* qm, const float* qv, const int32_t* comp,
                                  const int32_t* jtype, const uint8_t* y, double* f_root, double* f, cudaStream_t st) {
  const int64_t rows = n * K + 1;
  const size_t smem = (size_t)kCrossWarps * (J > 0 ? J : 1) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_crossed_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_crossed_tables<<<(unsigned)((rows + kCrossWarps - 1) / kCrossWarps), kCrossWarps * 32, smem, st>>>(
      n, K, J, C, T, rz, rm, rv, z, qm, qv, comp, jtype, y, f_root, f);
  return cudaGetLastError();
}

cudaError_t launch_crossed_moments(int64_t n, int K, int R, const double* w_root, const float* rz, const double* w,
                                   const float* z, double* root_m, double* gm, cudaStream_t st) {
  k_crossed_moments<<<(unsigned)((n + R + 7) / 8), 256, 0, st>>>(n, K, R, w_root, rz, w, z, root_m, gm);
  return cudaGetLastError();
}

}  // namespace qem
