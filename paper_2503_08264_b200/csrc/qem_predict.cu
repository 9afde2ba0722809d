// qem_predict.cu -- backward ancestral index resampling and the predictive log-likelihood
// (NEXT row f3, R31): "we draw latent samples conditioned on 'training' data ...
// and use these to predict a separate 'test' set", "averaged over 100
// predictive samples".
//
// After a two-level forward + root pass the plate elimination defines the posterior over index
// tuples r_k / sum r (Eq. 7a-c).  Ancestral sampling in reverse elimination order draws from it
// exactly:
//   k_root ~ w_root                                   (the root softmax, Eq. 7a)
//   k_i | k_root ~ P_i(k' | k_root) proportional to exp(B_i(k_root, k') + A_i(k'))
// with A_i(k') = t_ref(k') - B(k_ref, k') from the column prep, so a row is
//   t(k') = t_ref(k') + [B(k_root, z_i^k') - B(k_ref, z_i^k')]         (fp64)
// and the draw is the inverse CDF of its max-shifted exponentials (fp64 prefix in k' order).
// Uniforms: ((w >> 8) + 1/2) 2^-24 from word 0 of Philox4x32-10 at counter (s, 0, 0, 5 << 24)
// (root) and (s, 1 + global i, 0, 5 << 24) (instances), key = seed.
// The predictive log-likelihood of test observations is
//   ll_s = sum_i sum_j log p(x_test_ij | z_i^{k_i,s}),   PLL = log (1/S) sum_s exp(ll_s).
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

constexpr uint32_t kResampleTag = 5u << 24;

__device__ __forceinline__ double uniform24(uint32_t w) { return ((double)(w >> 8) + 0.5) * 5.9604644775390625e-08; }

struct ResampleArgs {
  int K, D, S, scale_kind;
  int64_t n_local, g_begin;
  double fixed_var;
  const float* z_root;  // [R][K]
  const float* w_root;  // [K]
  const float* z;       // [n_local][D][K]
  const double* tA;     // [n_local][K]
  const RefInfo* ref;
  uint2 key;
  int32_t* idx_root;  // [S]
  int32_t* idx;       // [S][n_local]
};

// root indices: one thread per s, sequential fp64 prefix over the fp32 root weights
__global__ void k_resample_root(ResampleArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  const uint4 o = philox4x32_10(make_uint4((uint32_t)s, 0u, 0u, kResampleTag), a.key);
  double tot = 0.0;
  for (int k = 0; k < a.K; ++k) tot += (double)a.w_root[k];
  const double target = uniform24(o.x) * tot;
  int k = 0;
  double cum = (double)a.w_root[0];
  while (k < a.K - 1 && target >= cum) cum += (double)a.w_root[++k];
  a.idx_root[s] = k;
}

__device__ __forceinline__ double lnv_of(const ResampleArgs& a, int k) {
  if (a.scale_kind == QEM_SCALE_FIXED) return log(a.fixed_var);
  const double s = (double)a.z_root[a.D * a.K + k];
  return a.scale_kind == QEM_SCALE_LOGSIGMA ? 2.0 * s : s;
}

// The warp's row t[0..K) (fp64, lane-strided max mx already taken per lane): exponentials in
// place, then the inverse-CDF draw for (s, i) -> a.idx.
__device__ __forceinline__ void draw_row(const ResampleArgs& a, double* t, double mx, int s, int64_t i, int lane) {
  const int K = a.K;
  mx = warp_max(mx);
  double tot = 0.0;
  for (int k = lane; k < K; k += 32) {
    // fp32 exponential of the fp64 shifted value (<= 2^-22 relative): a draw can differ from an
    // fp64 evaluation only when u lies within ~1e-6 of a CDF boundary (R31)
    const double e = (double)ex2((float)((t[k] - mx) * 1.4426950408889634));
    t[k] = e;
    tot += e;
  }
  tot = warp_sum(tot);
  __syncwarp();
  const uint4 o = philox4x32_10(make_uint4((uint32_t)s, (uint32_t)(1 + a.g_begin + i), 0u, kResampleTag), a.key);
  const double target = uniform24(o.x) * tot;
  double base = 0.0;
  int pick = K - 1;
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    double cs = k < K ? t[k] : 0.0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // inclusive scan
      const double v = __shfl_up_sync(0xffffffffu, cs, off);
      if (lane >= off) cs += v;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, k < K && base + cs > target);
    if (hit) {
      pick = k0 + __ffs(hit) - 1;
      break;
    }
    base += __shfl_sync(0xffffffffu, cs, 31);
  }
  if (lane == 0) a.idx[(int64_t)s * a.n_local + i] = pick;
  __syncwarp();  // the row buffer is rewritten by the warp's next draw
}

// Root-difference coefficients of draw s: D_kr(z) = a0 + c . z + gam |z|^2 (fp64).
template <int D>
__device__ __forceinline__ void row_coef(const ResampleArgs& a, int kr, int kf, double (&c)[D], double& a0,
                                         double& gam) {
  const int K = a.K;
  const double lv_r = lnv_of(a, kr), lv_f = lnv_of(a, kf);
  const double e_r = exp(-lv_r), e_f = exp(-lv_f);
  a0 = -0.5 * D * (lv_r - lv_f);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const double mr = a.z_root[r * K + kr], mf = a.z_root[r * K + kf];
    c[r] = e_r * mr - e_f * mf;
    a0 -= 0.5 * (e_r * mr * mr - e_f * mf * mf);
  }
  gam = -0.5 * (e_r - e_f);
}

// Tile variant: one CTA per group with the group's z (fp64), |z|^2 and t_ref staged in shared
// memory once; its 8 warps take the S draws in turn (z re-reads hit SMEM, no per-draw
// conversions).  Used when (D + 2 + 8) K doubles fit in shared memory.
constexpr int kTileWarps = 8;
template <int D>
__global__ void __launch_bounds__(kTileWarps * 32) k_resample_tile(ResampleArgs a) {
  extern __shared__ double sm[];
  const int K = a.K, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* zt = sm;                 // [D][K]
  double* zz = zt + (size_t)D * K;  // [K]
  double* ta = zz + K;              // [K]
  double* t = ta + K + (size_t)wid * K;
  const int64_t i = blockIdx.x;
  const float* zi = a.z + (size_t)i * D * K;
  for (int e = threadIdx.x; e < D * K; e += blockDim.x) zt[e] = zi[e];
  for (int k = threadIdx.x; k < K; k += blockDim.x) ta[k] = a.tA[(size_t)i * K + k];
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double q = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) q = fma(zt[(size_t)r * K + k], zt[(size_t)r * K + k], q);
    zz[k] = q;
  }
  __syncthreads();
  const int kf = a.ref->k_ref;
  for (int s = wid; s < a.S; s += kTileWarps) {
    double c[D], a0, gam;
    row_coef<D>(a, a.idx_root[s], kf, c, a0, gam);
    double mx = -CUDART_INF;
    for (int k = lane; k < K; k += 32) {
      double dot = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) dot = fma(c[r], zt[(size_t)r * K + k], dot);
      const double v = ta[k] + a0 + fma(gam, zz[k], dot);
      t[k] = v;
      mx = fmax(mx, v);
    }
    draw_row(a, t, mx, s, i, lane);
  }
}

// instance indices (fallback for large tiles): one warp per (s, i).  The row t(k') = t_ref(k') + D_kr(z_i^k') is evaluated
// once into the warp's shared-memory row (fp64, D_k(z) = B(k,z) - B(k_ref,z) expanded as
// a0 + c . z + gam |z|^2), then max, exponentials (in place), and the inverse CDF: chunks of 32
// columns, an inclusive warp scan per chunk (fixed association), the first column whose prefix
// passes u * sum.
constexpr int kResWarps = 4;

template <int D>
__global__ void __launch_bounds__(kResWarps * 32) k_resample_groups(ResampleArgs a) {
  extern __shared__ double rowbuf[];  // [kResWarps][K]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kResWarps + wid;
  if (row >= (int64_t)a.S * a.n_local) return;
  // group-major: the S draws of one group run on neighbouring warps, so its z tile (D x K) and
  // t_ref row are read from HBM once and then hit in L1/L2
  const int64_t i = row / a.S;
  const int s = (int)(row - i * a.S);
  const int K = a.K, kr = a.idx_root[s], kf = a.ref->k_ref;
  double* t = rowbuf + (size_t)wid * K;
  double c[D], a0, gam;
  row_coef<D>(a, kr, kf, c, a0, gam);
  const float* zi = a.z + (size_t)i * D * K;
  const double* ti = a.tA + (size_t)i * K;
  double mx = -CUDART_INF;
  for (int k = lane; k < K; k += 32) {
    double dot = 0.0, zz = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double zr = zi[(size_t)r * K + k];
      dot = fma(c[r], zr, dot);
      zz = fma(zr, zr, zz);
    }
    const double v = ti[k] + a0 + fma(gam, zz, dot);
    t[k] = v;
    mx = fmax(mx, v);
  }
  draw_row(a, t, mx, s, i, lane);
}

// ---- global importance weighting (App. A, Eq. glob_iw): K joint draws with
// every latent at the same index k (no index mixing):
//   log r_k = f_root(k) + sum_i [B_i(k, z_i^k) + A_i(z_i^k)],  log Pe_glob = lse_k log r_k - ln K,
// weights softmax(log r).  The per-group diagonal is t_ref_i(k) + D_k(z_i^k) (fp64), then the
// plate-root reduction of the table engine does the rest.
template <int D>
__global__ void __launch_bounds__(256) k_global_diag(ResampleArgs a, double* __restrict__ diag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n_local * a.K) return;
  const int64_t i = t / a.K;
  const int k = (int)(t - i * a.K);
  double c[D], a0, gam;
  row_coef<D>(a, k, a.ref->k_ref, c, a0, gam);
  const float* zi = a.z + (size_t)i * D * a.K + k;
  double dot = 0.0, zz = 0.0;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const double zr = zi[(size_t)r * a.K];
    dot = fma(c[r], zr, dot);
    zz = fma(zr, zr, zz);
  }
  diag[t] = a.tA[t] + a0 + fma(gam, zz, dot);
}

// group means under the global weights: m1[i][r] = sum_k w_k z_i^{r,k} (one warp per (i, r))
__global__ void __launch_bounds__(256) k_global_m1(int64_t rows, int K, const double* __restrict__ w,
                                                   const float* __restrict__ z, double* __restrict__ m1) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  double s = 0.0;
  for (int k = lane; k < K; k += 32) s += w[k] * (double)z[row * K + k];
  s = warp_sum(s);
  if (lane == 0) m1[row] = s;
}

cudaError_t launch_global_iw(qem_ctx* c, double* diag, double* scratch, double* log_pe, double* w, double* m1,
                             cudaStream_t st) {
  ResampleArgs a{};
  a.K = c->desc.K;
  a.D = c->desc.d;
  a.scale_kind = c->desc.scale_kind;
  a.n_local = c->n_local;
  a.fixed_var = c->desc.fixed_var;
  a.z_root = c->bufs.level[0].z;
  a.z = c->bufs.level[1].z;
  a.tA = c->tw.tA;
  a.ref = c->tw.ref;
  const int64_t t = a.n_local * a.K;
  switch (a.D) {
#define X(v)                                                                      \
  case v:                                                                         \
    k_global_diag<v><<<(unsigned)((t + 255) / 256), 256, 0, st>>>(a, diag);       \
    break;
    X(1) X(2) X(3) X(4) X(8) X(16) X(18)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
  cudaError_t e = launch_plate_root(a.n_local, a.K, c->tw.f_root, diag, scratch, log_pe, w, st);
  if (e != cudaSuccess) return e;
  if (m1) {
    const int64_t rows = a.n_local * a.D;
    k_global_m1<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, a.K, w, a.z, m1);
  }
  return cudaGetLastError();
}

struct PredictArgs {
  int K, D, S, J, obs_kind;
  int64_t n_local;
  double obs_var;
  const float* z;        // [n_local][D][K]
  const int32_t* idx;    // [S][n_local]
  const void* x;         // Bernoulli: uint8 [n_local][J][D]; Gaussian: float [n_local][J]
  const uint8_t* y;      // Bernoulli: [n_local][J]
  double* ll_part;       // [S][n_local]
};

// one thread per (s, i): the test log-likelihood at z_i^{k_i,s} (fp64)
__global__ void __launch_bounds__(256) k_predict(PredictArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.S * a.n_local) return;
  const int64_t i = t % a.n_local;
  const int k = a.idx[t];
  const float* zi = a.z + (size_t)i * a.D * a.K + k;
  double ll = 0.0;
  if (a.obs_kind == QEM_OBS_GAUSS) {
    const double zz = zi[0], c = -0.5 * (kLn2Pi + log(a.obs_var));
    const float* x = reinterpret_cast<const float*>(a.x) + (size_t)i * a.J;
    for (int j = 0; j < a.J; ++j) {
      const double dx = (double)x[j] - zz;
      ll += c - 0.5 * dx * dx / a.obs_var;
    }
  } else {
    const uint8_t* x = reinterpret_cast<const uint8_t*>(a.x) + (size_t)i * a.J * a.D;
    for (int j = 0; j < a.J; ++j) {
      double eta = 0.0;
      for (int r = 0; r < a.D; ++r)
        if (x[j * a.D + r]) eta += (double)zi[(size_t)r * a.K];
      ll += (a.y[i * a.J + j] ? eta : 0.0) - (fmax(eta, 0.0) + log1p(exp(-fabs(eta))));
    }
  }
  a.ll_part[t] = ll;
}

// ll_s = sum_i ll_part[s][i] (one warp per s, lane-strided then a fixed shuffle tree)
__global__ void k_predict_sum(int S, int64_t n, const double* ll_part, double* ll_s) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S) return;
  double acc = 0.0;
  for (int64_t i = lane; i < n; i += 32) acc += ll_part[(int64_t)s * n + i];
  acc = warp_sum(acc);
  if (lane == 0) ll_s[s] = acc;
}

// out = log (1/n) sum exp(x) (one block, fixed order)
__global__ void __launch_bounds__(1024) k_logmeanexp(int64_t n, const double* x, double* out) {
  __shared__ double scratch[32];
  double m = -CUDART_INF;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, x[i]);
  m = block_max(m, scratch);
  double s = 0.0;
  if (m > -CUDART_INF)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += exp(x[i] - m);
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = m == -CUDART_INF ? -CUDART_INF : m + log(s) - log((double)n);
}

cudaError_t launch_resample(qem_ctx* c, int S, uint64_t seed, int32_t* idx_root, int32_t* idx, cudaStream_t st) {
  ResampleArgs a{};
  a.K = c->desc.K;
  a.D = c->desc.d;
  a.S = S;
  a.scale_kind = c->desc.scale_kind;
  a.n_local = c->n_local;
  a.g_begin = c->g_begin;
  a.fixed_var = c->desc.fixed_var;
  a.z_root = c->bufs.level[0].z;
  a.w_root = c->bufs.level[0].w;
  a.z = c->bufs.level[1].z;
  a.tA = c->tw.tA;
  a.ref = c->tw.ref;
  a.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  a.idx_root = idx_root;
  a.idx = idx;
  k_resample_root<<<(S + 127) / 128, 128, 0, st>>>(a);
  const int64_t rows = (int64_t)S * a.n_local;
  const unsigned blocks = (unsigned)((rows + kResWarps - 1) / kResWarps);
  const size_t smem = (size_t)kResWarps * a.K * sizeof(double);
  const size_t smem_tile = (size_t)(a.D + 2 + kTileWarps) * a.K * sizeof(double);
  // QEM_RESAMPLE_NO_TILE: force the per-draw kernel (tests cover both)
  const bool tile = smem_tile <= 220 * 1024 && getenv("QEM_RESAMPLE_NO_TILE") == nullptr;
  switch (a.D) {
#define X(v)                                                                                          \
  case v:                                                                                             \
    if (tile) {                                                                                       \
      if (cudaFuncSetAttribute(k_resample_tile<v>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                               (int)smem_tile) != cudaSuccess)                                        \
        return cudaErrorInvalidValue;                                                                 \
      k_resample_tile<v><<<(unsigned)a.n_local, kTileWarps * 32, smem_tile, st>>>(a);                 \
    } else {                                                                                          \
      if (cudaFuncSetAttribute(k_resample_groups<v>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                               (int)smem) != cudaSuccess)                                             \
        return cudaErrorInvalidValue;                                                                 \
      k_resample_groups<v><<<blocks, kResWarps * 32, smem, st>>>(a);                                  \
    }                                                                                                 \
    break;
    X(1) X(2) X(3) X(4) X(8) X(16) X(18)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_predict(qem_ctx* c, int S, const int32_t* idx, int J, const void* x, const uint8_t* y,
                           double* ll_part, double* ll_s, double* pll, cudaStream_t st) {
  PredictArgs a{};
  a.K = c->desc.K;
  a.D = c->desc.d;
  a.S = S;
  a.J = J;
  a.obs_kind = c->desc.obs_kind;
  a.n_local = c->n_local;
  a.obs_var = c->desc.obs_var;
  a.z = c->bufs.level[1].z;
  a.idx = idx;
  a.x = x;
  a.y = y;
  a.ll_part = ll_part;
  const int64_t t = (int64_t)S * a.n_local;
  k_predict<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(a);
  k_predict_sum<<<(S + 7) / 8, 256, 0, st>>>(S, a.n_local, ll_part, ll_s);
  if (pll) k_logmeanexp<<<1, 1024, 0, st>>>(S, ll_s, pll);
  return cudaGetLastError();
}

cudaError_t launch_logmeanexp(int64_t n, const double* x, double* out, cudaStream_t st) {
  k_logmeanexp<<<1, 1024, 0, st>>>(n, x, out);
  return cudaGetLastError();
}

}  // namespace qem
