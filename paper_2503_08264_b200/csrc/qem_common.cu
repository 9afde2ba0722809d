// qem_common.cu -- K1 (Q sampler) and K5 (EMA + Gaussian M-step) for every
// model family.  sm_100a.
#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

// n / d for 32-bit n by a runtime-constant d via multiply-high (Granlund-Montgomery):
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
struct FastDiv {
  uint32_t d, m, l;
  __host__ void init(uint32_t div) {
    d = div;
    l = 0;
    while ((1ull << l) < div) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> l);
  }
};

struct SampleLevel {
  float* z;            // [inst][dims][K]
  const float* qm;     // [inst*dims]
  const float* qv;
  const float* eps;    // [inst*dims][K] or nullptr (Philox)
  int64_t rows;        // inst*dims
  int64_t quads_begin; // prefix over levels, in units of 4 samples
  int dims;
  int level;
  int64_t inst_offset; // global instance index of local instance 0
  FastDiv fdims;
};

struct SampleArgs {
  SampleLevel lv[3];
  int nlev;
  int K;
  int quads_per_row;
  int units_per_row;  // quads_per_row / QPT
  FastDiv fqpr;
  FastDiv fupr;
  int64_t total_quads;  // < 2^31 (checked at launch)
  uint2 key;
  int t_host;
  uint32_t iter_or;  // OR-ed into the iteration word (bit 23: the fresh-denominator stream)
  const int32_t* d_iter;
  const int32_t* d_base;  // eps bank mode (qem_iterate parity mode): slice (t - *d_base) of every level's eps
};

// K1: z = fmaf(sqrtf(v), eps, m)  (Alg. 1 line 4; location-scale
// sampling, App. E; fp32 definition DESIGN.md R22).
// One thread = 4 consecutive samples k of one latent dim (one Philox call,
// two Box-Muller pairs).
// One Philox4x32-10 call per quad of 4 samples; a thread takes QPT consecutive quads of one row
// (QPT = 2 when K % 8 == 0: the row's mean / sd loads, the index divisions and the counter
// setup are shared), grid-stride over the units of each level in turn (the level's parameters
// are hoisted out of the loop).
template <int QPT>
__device__ __forceinline__ void sample_unit(const SampleArgs& a, const SampleLevel& s, uint32_t local, int t) {
  const uint32_t row32 = a.fupr.div(local);
  const int64_t row = row32;
  const int k0 = (int)(local - row32 * (uint32_t)a.units_per_row) * 4 * QPT;
  const float m = s.qm[row];
  const float sd = __fsqrt_rn(s.qv[row]);
  float e[QPT][4];
  if (s.eps != nullptr) {
#pragma unroll
    for (int u = 0; u < QPT; ++u)
#pragma unroll
      for (int j = 0; j < 4; ++j) e[u][j] = (k0 + 4 * u + j < a.K) ? s.eps[row * a.K + k0 + 4 * u + j] : 0.f;
  } else {
    const uint32_t inst = s.fdims.div(row32);
    const int dim = (int)(row32 - inst * (uint32_t)s.dims);
    const uint32_t ginst = (uint32_t)(inst + s.inst_offset);
    const uint32_t word = ((uint32_t)s.level << 24) | (((uint32_t)t | a.iter_or) & 0xffffffu);
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
      const float4 n4 = philox_normal4(make_uint4((uint32_t)(k0 >> 2) + u, (uint32_t)dim, ginst, word), a.key);
      e[u][0] = n4.x;
      e[u][1] = n4.y;
      e[u][2] = n4.z;
      e[u][3] = n4.w;
    }
  }
  float* zr = s.z + row * a.K + k0;
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    if (k0 + 4 * u + 4 <= a.K && (a.K & 3) == 0) {
      *reinterpret_cast<float4*>(zr + 4 * u) = make_float4(__fmaf_rn(sd, e[u][0], m), __fmaf_rn(sd, e[u][1], m),
                                                           __fmaf_rn(sd, e[u][2], m), __fmaf_rn(sd, e[u][3], m));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (k0 + 4 * u + j < a.K) zr[4 * u + j] = __fmaf_rn(sd, e[u][j], m);
    }
  }
}

template <int QPT>
__global__ void __launch_bounds__(256) k_sample(SampleArgs a) {
  const int t = resolve_iter(a.t_host, a.d_iter);
  const uint32_t stride = gridDim.x * blockDim.x;
  const int64_t bj = a.d_base ? (int64_t)(t - *a.d_base) : 0;  // eps bank slice of iteration t
  for (int L = 0; L < a.nlev; ++L) {
    SampleLevel s = a.lv[L];
    if (s.eps) s.eps += bj * s.rows * a.K;
    const uint32_t units = (uint32_t)s.rows * (uint32_t)a.units_per_row;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += stride) sample_unit<QPT>(a, s, u, t);
  }
}

static cudaError_t launch_k_sample(SampleArgs& a, int64_t cap_blocks, cudaStream_t st) {
  const int qpt = (a.K % 16 == 0) ? 4 : ((a.K % 8 == 0) ? 2 : 1);
  a.units_per_row = a.quads_per_row / qpt;
  a.fupr.init((uint32_t)a.units_per_row);
  int64_t units = 0;
  for (int l = 0; l < a.nlev; ++l) units += a.lv[l].rows * a.units_per_row;
  int64_t blocks = (units + 255) / 256;
  if (blocks == 0) return cudaSuccess;
  if (blocks > cap_blocks) blocks = cap_blocks;
  if (qpt == 4)
    k_sample<4><<<(unsigned)blocks, 256, 0, st>>>(a);
  else if (qpt == 2)
    k_sample<2><<<(unsigned)blocks, 256, 0, st>>>(a);
  else
    k_sample<1><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Context-free Gaussian sampler (qem_sample_normal): `rows` latent rows of K samples, one level
// tag (the Philox counter's top byte) and global row index = instance with dims = 1.
cudaError_t launch_sample_rows(int64_t rows, int K, int level, uint64_t seed, int32_t iter, const float* qm,
                               const float* qv, const float* eps, float* z, cudaStream_t st) {
  SampleArgs a{};
  a.K = K;
  a.quads_per_row = (K + 3) / 4;
  a.fqpr.init((uint32_t)a.quads_per_row);
  a.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  a.t_host = iter;
  a.d_iter = nullptr;
  a.nlev = 1;
  SampleLevel& s = a.lv[0];
  s.z = z;
  s.qm = qm;
  s.qv = qv;
  s.eps = eps;
  s.rows = rows;
  s.dims = 1;
  s.fdims.init(1u);
  s.level = level;
  s.inst_offset = 0;
  s.quads_begin = 0;
  a.total_quads = rows * a.quads_per_row;
  if (a.total_quads == 0) return cudaSuccess;
  if (a.total_quads >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
  return launch_k_sample(a, 148 * 32, st);
}

cudaError_t launch_sample(qem_ctx* c, uint64_t seed, int32_t iter, const float* const* d_eps, cudaStream_t st,
                          uint32_t iter_or, int root_only) {
  SampleArgs a{};
  a.iter_or = iter_or;
  if (!d_eps && iter == 0 && iter_or == 0 && c->bufs.eps_bank[0]) {  // qem_iterate in eps bank mode
    d_eps = c->bufs.eps_bank;
    a.d_base = &c->cnt->trace_base;
  }
  const int K = c->desc.K;
  a.K = K;
  a.quads_per_row = (K + 3) / 4;
  a.fqpr.init((uint32_t)a.quads_per_row);
  a.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  a.t_host = iter;
  a.d_iter = &c->cnt->iter;
  int nlev = root_only ? 1 : (c->desc.family == QEM_FAMILY_TWO_LEVEL ? 2 : 3);
  int64_t quads = 0;
  for (int l = 0; l < nlev; ++l) {
    SampleLevel& s = a.lv[l];
    const qem_level& b = c->bufs.level[l];
    int64_t inst, dims, off = 0;
    if (l == 0) {
      inst = 1;
      dims = c->R;
    } else if (c->desc.family == QEM_FAMILY_TWO_LEVEL) {
      inst = c->n_local;
      dims = c->desc.d;
      off = c->g_begin;
    } else if (l == 1) {
      inst = c->desc.n;
      dims = 1;
    } else {
      inst = c->desc.n * c->desc.n_sub;
      dims = 1;
    }
    s.z = b.z;
    s.qm = b.q_mean;
    s.qv = b.q_var;
    s.eps = d_eps ? d_eps[l] : nullptr;
    s.rows = inst * dims;
    s.dims = (int)dims;
    s.fdims.init((uint32_t)dims);
    s.level = l;
    s.inst_offset = off;
    s.quads_begin = quads;
    quads += s.rows * a.quads_per_row;
  }
  a.nlev = nlev;
  a.total_quads = quads;
  if (quads == 0) return cudaSuccess;
  if (quads >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;  // 32-bit sample indexing
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int64_t cap = (int64_t)sms * 8 * 4;  // four waves of 8 resident 256-thread blocks per SM
  const cudaError_t e = launch_k_sample(a, cap, st);
  if (e != cudaSuccess) return e;
  c->launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ M-step

struct MstepLevel {
  double* m1;
  double* v;
  const double* m1n;
  const double* vn;
  float* qm;
  float* qv;
  int64_t begin;  // prefix offset
};

struct MstepArgs {
  MstepLevel lv[3];
  int nlev;
  int64_t total;
  double new_weight, p, floor_v;
  int t_host;
  const double* log_pe;        // fresh denominator: ratio = exp(log_pe - log_pe_fresh)
  const double* log_pe_fresh;  // nullptr: self-normalised moments (Eq. 7a)
  Counters* cnt;
};

// K5: EMA over mean parameters (Eq. 9; Alg. 1 line 6) in
// centred form (R19), then the Gaussian M-step (Alg. 1
// line 3) with the variance floor (R8).  lambda = history weight (R5).
__global__ void __launch_bounds__(256) k_mstep(MstepArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = resolve_iter(a.t_host, &a.cnt->iter);
  const double lam = a.p > 0.0 ? 1.0 - pow((double)t, -a.p) : 1.0 - a.new_weight;
  if (e < a.total) {
    int L = 0;
#pragma unroll
    for (int l = 1; l < 3; ++l)
      if (l < a.nlev && e >= a.lv[l].begin) L = l;
    const MstepLevel& s = a.lv[L];
    const int64_t j = e - s.begin;
    const double m1 = s.m1[j], v = s.v[j];
    double a1 = s.m1n[j], av = s.vn[j];
    if (a.log_pe_fresh) {
      // fresh-sample denominator: mean parameters (a1, av + a1^2) times
      // r = Pe(z)/Pe(z_new); centred: a1' = r a1, av' = r av + r (1 - r) a1^2
      const double r = exp(*a.log_pe - *a.log_pe_fresh);
      av = r * av + r * (1.0 - r) * a1 * a1;
      a1 = r * a1;
    }
    const double d = m1 - a1;
    const double nm1 = lam * m1 + (1.0 - lam) * a1;
    const double nv = lam * v + (1.0 - lam) * av + lam * (1.0 - lam) * d * d;
    s.m1[j] = nm1;
    s.v[j] = nv;
    double qv = nv;
    if (!(nv >= a.floor_v)) {
      qv = a.floor_v;
      atomicAdd(&a.cnt->clamps, 1ull);
      atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_CLAMP);
    }
    if (isnan(nm1) || isnan(nv)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
    s.qm[j] = (float)nm1;
    s.qv[j] = (float)qv;
  }
  if (a.t_host <= 0) {
    // graph mode: the last block advances the device iteration counter.
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const uint32_t tk = atomicAdd(&a.cnt->ticket_mstep, 1u);
      if (tk == gridDim.x - 1) {
        a.cnt->iter = t + 1;
        a.cnt->ticket_mstep = 0;
        __threadfence();
      }
    }
  }
}

cudaError_t launch_mstep(qem_ctx* c, int32_t t, cudaStream_t st) {
  MstepArgs a{};
  int nlev = c->desc.family == QEM_FAMILY_TWO_LEVEL ? 2 : 3;
  int64_t tot = 0;
  for (int l = 0; l < nlev; ++l) {
    const qem_level& b = c->bufs.level[l];
    int64_t cnt;
    if (l == 0)
      cnt = c->R;
    else if (c->desc.family == QEM_FAMILY_TWO_LEVEL)
      cnt = c->n_local * c->desc.d;
    else if (l == 1)
      cnt = c->desc.n;
    else
      cnt = c->desc.n * c->desc.n_sub;
    a.lv[l] = MstepLevel{b.ema_m1, b.ema_v, b.m1, b.v, b.q_mean, b.q_var, tot};
    tot += cnt;
  }
  a.nlev = nlev;
  a.total = tot;
  a.new_weight = c->opts.new_weight;
  a.p = c->opts.schedule_p;
  a.floor_v = c->opts.var_floor;
  a.t_host = t;
  a.cnt = c->cnt;
  if (c->opts.fresh_denominator) {
    a.log_pe = c->bufs.log_pe;
    a.log_pe_fresh = c->bufs.log_pe_fresh;
  }
  const int threads = 256;
  const int64_t blocks = (tot + threads - 1) / threads;
  k_mstep<<<(unsigned)(blocks > 0 ? blocks : 1), threads, 0, st>>>(a);
  c->launches += 1;
  return cudaGetLastError();
}

}  // namespace qem
