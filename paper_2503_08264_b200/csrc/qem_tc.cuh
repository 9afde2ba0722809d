// qem_tc.cuh -- tcgen05 tensor-core pair-tile kernels for d = 16 (config 5).
// Included inside namespace qem by qem_two_level.cu (needs TLArgs, expm1_poly).
//
// The d-dim part of every log-factor is a dense contraction over the latent
// dimension: D_k(k') = alpha_k + gamma_k |u_k'|^2 + c_k . u_k'  (DESIGN.md
// "Forward"), so the K x K x 16 product c . u runs on the 5th-gen tensor
// cores: tcgen05.mma kind::f16 with both operands split into three bf16 terms
// and the six leading partial products accumulated small-first in TMEM
// (fp32-exact to ~1e-7 of sum|c_r u_r|, unbiased; tools/tc_probe.cu).  The
// exp / log-sum-exp epilogue reads the 128 x 256 fp32 tile from TMEM
// (tcgen05.ld) and runs on the SFU / FMA pipes while the next tile's MMAs run
// into the other half of TMEM (2 x 256 columns).  One CTA per SM; 4*CQ warps:
// warp w reads TMEM lane quarter (w % 4) and column slice (w / 4) of width 256/CQ.
//
//  k_rowop           c_k -> bf16x3 operand (K rows x 96 B), once per E-step
//  k_forward_tc<CQ>  M = 128 parent rows (static operand, resident in SMEM) x
//                    N = 256 child columns (per-group operand, TMA double buffer);
//                    thread = row x column slice; same tile modes as k_forward
//  k_backward_tc<CQ> M = 128 child columns (per-group operand) x N = 256 parent
//                    rows (static); thread = column x row slice
#pragma once

constexpr int kTcD = 16;
constexpr uint32_t kTcColBlockBytes = 256 * kTcRowBytes;  // forward B tile (256 columns)
constexpr uint32_t kTcBwdBlockBytes = 128 * kTcRowBytes;  // backward A tile (128 columns)
constexpr int kTcCQ = 4;                                  // column slices per TMEM lane quarter

__global__ void __launch_bounds__(256) k_rowop(TLArgs a) {
  const int K = a.K;
  unsigned char* rop = reinterpret_cast<unsigned char*>(a.ws.rowop);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * kTcD; e += gridDim.x * blockDim.x) {
    const int k = e / kTcD, r = e % kTcD;
    __nv_bfloat16 s3[3];
    split3_bf16(a.ws.fwd_coef[(size_t)k * (kTcD + 2) + 2 + r], s3);
#pragma unroll
    for (int q = 0; q < 3; ++q) *reinterpret_cast<__nv_bfloat16*>(rop + tc_offset(k, q * 16 + r)) = s3[q];
  }
}


// 16 consecutive floats from shared memory as four 128-bit loads
__device__ __forceinline__ void lds16(const float* p, float (&o)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 v = reinterpret_cast<const float4*>(p)[q];
    o[4 * q] = v.x;
    o[4 * q + 1] = v.y;
    o[4 * q + 2] = v.z;
    o[4 * q + 3] = v.w;
  }
}

// Walk NC16 chunks of 16 TMEM columns with the next chunk's tcgen05.ld in
// flight while the current one is processed (two register buffers).
template <int NC16, class F>
__device__ __forceinline__ void tmem_pipeline16(uint32_t taddr, F&& f) {
  uint32_t r0[16], r1[16];
  tmem_ld16_async(taddr, r0);
  tmem_wait16(r0);
#pragma unroll
  for (int c = 0; c < NC16; ++c) {
    if (c & 1) {
      if (c + 1 < NC16) tmem_ld16_async(taddr + (c + 1) * 16, r0);
      f(c, r1);
      if (c + 1 < NC16) tmem_wait16(r0);
    } else {
      if (c + 1 < NC16) tmem_ld16_async(taddr + (c + 1) * 16, r1);
      f(c, r0);
      if (c + 1 < NC16) tmem_wait16(r1);
    }
  }
}

// Forward epilogue, online log-sum-exp over t' = tm + gamma |u|^2 + ln P (the
// row constant kappa is added at the end): state (st0 = running max, st1 = sum).
template <int NC16>
__device__ __forceinline__ void fwd_epi_online(uint32_t taddr, const float* u2, const float* lp, float g, float& st0,
                                               float& st1) {
  tmem_pipeline16<NC16>(taddr, [&](int c16, uint32_t(&r)[16]) {
    float a[16], b[16], v[16];
    lds16(u2 + c16 * 16, a);
    lds16(lp + c16 * 16, b);
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const float2 t = add2(fma2(f2(g), make_float2(a[c], a[c + 1]), make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1]))),
                            make_float2(b[c], b[c + 1]));
      v[c] = t.x;
      v[c + 1] = t.y;
    }
    float mx[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) mx[q] = fmaxf(fmaxf(v[q], v[q + 4]), fmaxf(v[q + 8], v[q + 12]));
    const float mn = fmaxf(st0, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])));
    const float nm = -mn * kLog2e;
    float2 ps[2] = {f2(0.f), f2(0.f)};
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const float2 e = fma2(make_float2(v[c], v[c + 1]), f2(kLog2e), f2(nm));
      ps[(c >> 1) & 1] = add2(ps[(c >> 1) & 1], make_float2(ex2(e.x), ex2(e.y)));
    }
    const float2 tot = add2(ps[0], ps[1]);
    st1 = fmaf(st1, ex2((st0 - mn) * kLog2e), tot.x + tot.y);
    st0 = mn;
  });
}

// Forward epilogue, polynomial mode: st0 += sum P expm1_N(tm + gamma |u|^2 + kappa).
template <int N, int NC16>
__device__ __forceinline__ void fwd_epi_poly(uint32_t taddr, const float* u2, const float* pp, float g, float kap,
                                             float& st0) {
  float2 acc[2] = {f2(0.f), f2(0.f)};
  tmem_pipeline16<NC16>(taddr, [&](int c16, uint32_t(&r)[16]) {
    float a[16], b[16];
    lds16(u2 + c16 * 16, a);
    lds16(pp + c16 * 16, b);
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const float2 dp =
          add2(fma2(f2(g), make_float2(a[c], a[c + 1]), make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1]))),
               f2(kap));
      acc[(c >> 1) & 1] = fma2(make_float2(b[c], b[c + 1]), expm1_poly<N>(dp), acc[(c >> 1) & 1]);
    }
  });
  const float2 t2 = add2(acc[0], acc[1]);
  st0 += t2.x + t2.y;
}

template <int CQ>
struct FwdTcLayout {
  static __host__ __device__ size_t colop(int K) { return (size_t)K * kTcRowBytes; }  // rowop at 0
  static __host__ __device__ size_t aux(int K) { return colop(K) + 2 * (size_t)kTcColBlockBytes; }
  static __host__ __device__ size_t kappa(int K) { return aux(K) + 2 * (size_t)K * 12; }
  static __host__ __device__ size_t st0(int K) { return kappa(K) + (size_t)K * 4; }
  static __host__ __device__ size_t st1(int K) { return st0(K) + (size_t)CQ * K * 4; }
  static __host__ __device__ size_t gsum(int K) { return st1(K) + (size_t)CQ * K * 4; }
  static __host__ __device__ size_t u0(int K) { return gsum(K) + (size_t)K * 8; }
  static __host__ __device__ size_t bars(int K) { return u0(K) + 32 * 4; }
  static __host__ __device__ size_t bytes(int K) { return bars(K) + 64; }
};

// Forward: warp w, lane l -> row k = rb*128 + 32*(w%4) + l, columns cq*(256/CQ).. of each tile.
template <int CQ>
__global__ void __launch_bounds__(128 * CQ, 1) k_forward_tc(TLArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  using L = FwdTcLayout<CQ>;
  constexpr int NT = 128 * CQ, CW = 256 / CQ, NC16 = CW / 16;
  const int K = a.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, cq = warp >> 2;
  const int NB = K / 256, RB = K / 128, TPG = NB * RB;
  unsigned char* s_rowop = smem;
  unsigned char* s_colop = smem + L::colop(K);
  float* s_aux = reinterpret_cast<float*>(smem + L::aux(K));  // 2 x [3][K] SoA
  float* s_kappa = reinterpret_cast<float*>(smem + L::kappa(K));
  float* s_st0 = reinterpret_cast<float*>(smem + L::st0(K));
  float* s_st1 = reinterpret_cast<float*>(smem + L::st1(K));
  double* s_g = reinterpret_cast<double*>(smem + L::gsum(K));
  float* s_u0 = reinterpret_cast<float*>(smem + L::u0(K));  // [16] u0, [16] |u0|^2
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::bars(K));  // [0,1] tma, [2,3] mma, [4] rowop
  __shared__ uint32_t s_tmem;
  __shared__ int s_mode[4 * CQ];

  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nblocks = ngroups * NB, ntiles = ngroups * TPG;
  const uint32_t idesc = umma_idesc_bf16(128, 256);

  if (tid == 0) {
    for (int b = 0; b < 5; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int k = tid; k < K; k += NT) s_g[k] = 0.0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  auto issue_block = [&](int64_t J) {  // colop block J (and the group's aux with its first block)
    if (J >= nblocks) return;
    const int64_t j = J / NB;
    const int cb = (int)(J % NB);
    const int64_t i = blockIdx.x + j * gridDim.x;
    const int st = (int)(J & 1);
    const uint32_t bytes = kTcColBlockBytes + (cb == 0 ? (uint32_t)K * 12 : 0u);
    mbar_expect_tx(&bar[st], bytes);
    tma_bulk_g2s(s_colop + st * kTcColBlockBytes,
                 reinterpret_cast<const unsigned char*>(a.ws.colop) + ((size_t)i * K + (size_t)cb * 256) * kTcRowBytes,
                 kTcColBlockBytes, &bar[st]);
    if (cb == 0)
      tma_bulk_g2s(s_aux + (size_t)(j & 1) * 3 * K, a.ws.colaux + (size_t)i * 3 * K, (uint32_t)K * 12, &bar[st]);
  };
  auto issue_mma = [&](int64_t T) {
    const int64_t J = T / TPG * NB + (T % TPG) / RB;
    const int rb = (int)(T % TPG % RB);
    mbar_wait(&bar[J & 1], (uint32_t)((J >> 1) & 1));
    tc_fence_after();
    umma_bf16x3(tmem + (uint32_t)(T & 1) * 256, smem_u32(s_rowop) + (uint32_t)rb * 128 * kTcRowBytes,
                smem_u32(s_colop) + (uint32_t)(J & 1) * kTcColBlockBytes, idesc);
    umma_commit(&bar[2 + (T & 1)]);
  };

  if (tid == 0) {
    mbar_expect_tx(&bar[4], (uint32_t)K * kTcRowBytes);
    tma_bulk_g2s(s_rowop, a.ws.rowop, (uint32_t)K * kTcRowBytes, &bar[4]);
    issue_block(0);
    issue_block(1);
  }
  mbar_wait(&bar[4], 0);
  if (tid == 0 && ntiles > 0) issue_mma(0);

  double csum = 0.0;
  int md = 0;
  for (int64_t T = 0; T < ntiles; ++T) {
    const int64_t j = T / TPG;
    const int t = (int)(T % TPG), cb = t / RB, rb = t % RB;
    const int64_t J = j * NB + cb;
    const int64_t i = blockIdx.x + j * gridDim.x;
    if (t == 0) {
      // ---- group setup: re-centring constants of all rows and the tile mode
      float u0[kTcD];
      float U0sq = 0.f;
#pragma unroll
      for (int r = 0; r < kTcD; ++r) {
        u0[r] = a.q_m[i * kTcD + r] - a.ws.ref->mu_ref[r];
        U0sq = fmaf(u0[r], u0[r], U0sq);
      }
      if (tid < kTcD) s_u0[tid] = u0[tid];
      if (tid == 0) s_u0[kTcD] = U0sq;
      const float W2max = a.ws.gstat[i];
      const float wmax = sqrtf(W2max);
      if (tid == 0) csum += a.ws.cvec[i];
      float tb = 0.f;
      for (int k = tid; k < K; k += NT) {
        const float* fc = a.ws.fwd_coef + (size_t)k * (kTcD + 2);
        const float g = fc[1];
        float kap = g * U0sq;
        float cn = 0.f;
#pragma unroll
        for (int r = 0; r < kTcD; ++r) {
          const float c = fc[2 + r];
          kap = fmaf(c, u0[r], kap);
          const float cp = fmaf(2.f * g, u0[r], c);
          cn = fmaf(cp, cp, cn);
        }
        s_kappa[k] = -kap;
        tb = fmaxf(tb, sqrtf(cn) * wmax + fabsf(g) * W2max);
      }
      int m = tb <= a.thr[0] ? 0 : (tb <= a.thr[1] ? 1 : (tb <= a.thr[2] ? 2 : (tb <= a.thr[3] ? 3 : (tb <= a.thr[4] ? 4 : 5))));
      m = __reduce_max_sync(0xffffffffu, m);
      if (lane == 0) s_mode[warp] = m;
      __syncthreads();
      md = 0;
#pragma unroll
      for (int w = 0; w < 4 * CQ; ++w) md = max(md, s_mode[w]);
      for (int e = tid; e < CQ * K; e += NT) {
        s_st0[e] = md == 5 ? -CUDART_INF_F : 0.f;
        s_st1[e] = 0.f;
      }
      if (tid == 0) atomicAdd(&a.cnt->mode_hist[md], 1ull);
      __syncthreads();
    }
    if (rb == 0) mbar_wait(&bar[J & 1], (uint32_t)((J >> 1) & 1));  // visibility of the block's aux data
    // ---- MMA of tile T done?  then queue tile T+1 (other TMEM buffer) before the epilogue
    mbar_wait(&bar[2 + (T & 1)], (uint32_t)((T >> 1) & 1));
    tc_fence_after();
    if (tid == 0 && T + 1 < ntiles) issue_mma(T + 1);

    // ---- epilogue: row k, columns cb*256 + cq*CW .. +CW
    const int k = rb * 128 + quarter * 32 + lane;
    const float g = a.ws.fwd_coef[(size_t)k * (kTcD + 2) + 1], kap = s_kappa[k];
    const float* axb = s_aux + (size_t)(j & 1) * 3 * K + cb * 256 + cq * CW;
    const uint32_t taddr = tmem + (uint32_t)(T & 1) * 256 + (uint32_t)(cq * CW) + ((uint32_t)(quarter * 32) << 16);
    float st0 = s_st0[cq * K + k], st1 = s_st1[cq * K + k];
    switch (md) {
      case 0: fwd_epi_poly<3, NC16>(taddr, axb, axb + K, g, kap, st0); break;
      case 1: fwd_epi_poly<4, NC16>(taddr, axb, axb + K, g, kap, st0); break;
      case 2: fwd_epi_poly<5, NC16>(taddr, axb, axb + K, g, kap, st0); break;
      case 3: fwd_epi_poly<7, NC16>(taddr, axb, axb + K, g, kap, st0); break;
      case 4: fwd_epi_poly<9, NC16>(taddr, axb, axb + K, g, kap, st0); break;
      default: fwd_epi_online<NC16>(taddr, axb, axb + 2 * K, g, st0, st1); break;
    }
    s_st0[cq * K + k] = st0;
    s_st1[cq * K + k] = st1;
    if (cb == NB - 1) {
      // ---- the row block is complete: merge the CQ column slices, finalise h and dg
      __syncthreads();
      if (cq == 0) {
        float h;
        if (md == 5) {
          float mx = -CUDART_INF_F;
#pragma unroll
          for (int q = 0; q < CQ; ++q) mx = fmaxf(mx, s_st0[q * K + k]);
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < CQ; ++q) s += s_st1[q * K + k] * ex2((s_st0[q * K + k] - mx) * kLog2e);
          h = s_kappa[k] + mx + logf(s);  // the online state excludes the row constant kappa
        } else {
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < CQ; ++q) s += s_st0[q * K + k];
          h = log1pf(s);
        }
        // alpha'_ik = alpha_k + gamma_k |u0|^2 + c_k . u0 in fp64
        const float* fc = a.ws.fwd_coef + (size_t)k * (kTcD + 2);
        double ap = a.ws.alpha_d[k] + (double)fc[1] * (double)s_u0[kTcD];
#pragma unroll
        for (int r = 0; r < kTcD; ++r) ap += (double)fc[2 + r] * (double)s_u0[r];
        const double dgd = ap + (double)h;
        a.ws.hmsg[(size_t)i * K + k] = h - s_kappa[k];  // TC path: the backward's row constant is -(h - kappa)
        a.ws.dg[(size_t)i * K + k] = (float)dgd;
        s_g[k] += dgd;
      }
    }
    tc_fence_before();
    __syncthreads();
    // the block's colop stage is free once all its tiles are consumed: refill it
    if (tid == 0 && rb == RB - 1) issue_block(J + 2);
  }

  // ---- teardown, per-CTA partial plate sums, last-CTA fixed-order reduce
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  double* part = a.ws.partial + (size_t)blockIdx.x * (K + 1);
  for (int k = tid; k < K; k += NT) part[k] = s_g[k];
  if (tid == 0) part[K] = csum;
  __threadfence();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) s_last = (atomicAdd(&a.cnt->ticket_fwd, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int k = tid; k <= K; k += NT) {
      double sum = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(a.ws.partial + (size_t)b * (K + 1) + k);
      a.ws.red[k] = sum;
    }
    if (tid == 0) a.cnt->ticket_fwd = 0;
  }
}

template <int CQ>
struct BwdTcLayout {
  static __host__ __device__ size_t colop(int K) { return (size_t)K * kTcRowBytes; }  // rowop at 0
  static __host__ __device__ size_t rowtab(int K) { return colop(K) + 2 * (size_t)kTcBwdBlockBytes; }
  static __host__ __device__ size_t wsm(int K) { return rowtab(K) + (size_t)K * 12; }
  static __host__ __device__ size_t wpart(int K) { return wsm(K) + (size_t)K * 4; }
  static __host__ __device__ size_t red(int K) { return wpart(K) + (size_t)CQ * 128 * 4; }
  static __host__ __device__ size_t bars(int K) { return red(K) + (4 * CQ * kTcD + kTcD) * 8; }
  static __host__ __device__ size_t bytes(int K) { return bars(K) + 64; }
};

// Backward: warp w, lane l -> column k' = cb*128 + 32*(w%4) + l, rows cq*(256/CQ).. of each tile.
template <int CQ>
__global__ void __launch_bounds__(128 * CQ, 1) k_backward_tc(TLArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  using L = BwdTcLayout<CQ>;
  constexpr int NT = 128 * CQ, NW = NT / 32, CW = 256 / CQ, NC16 = CW / 16;
  const int K = a.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, cq = warp >> 2;
  const int CB = K / 128, RB = K / 256, TPG = CB * RB;
  unsigned char* s_rowop = smem;
  unsigned char* s_colop = smem + L::colop(K);
  float* s_rt = reinterpret_cast<float*>(smem + L::rowtab(K));  // SoA [2][K]: gamma log2e, (kappa-h) log2e + log2 w_root
  float* s_w = reinterpret_cast<float*>(smem + L::wsm(K));
  float* s_wp = reinterpret_cast<float*>(smem + L::wpart(K));
  double* s_red = reinterpret_cast<double*>(smem + L::red(K));  // [NW][16]
  double* s_mom = s_red + NW * kTcD;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::bars(K));  // [0,1] tma, [2,3] mma, [4] rowop
  __shared__ uint32_t s_tmem;

  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nblocks = ngroups * CB, ntiles = ngroups * TPG;
  const uint32_t idesc = umma_idesc_bf16(128, 256);

  if (tid == 0) {
    for (int b = 0; b < 5; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  auto issue_block = [&](int64_t J) {
    if (J >= nblocks) return;
    const int64_t j = J / CB;
    const int cb = (int)(J % CB);
    const int64_t i = blockIdx.x + j * gridDim.x;
    const int st = (int)(J & 1);
    mbar_expect_tx(&bar[st], kTcBwdBlockBytes);
    tma_bulk_g2s(s_colop + st * kTcBwdBlockBytes,
                 reinterpret_cast<const unsigned char*>(a.ws.colop) + ((size_t)i * K + (size_t)cb * 128) * kTcRowBytes,
                 kTcBwdBlockBytes, &bar[st]);
  };
  auto issue_mma = [&](int64_t T) {
    const int64_t J = T / TPG * CB + (T % TPG) / RB;
    const int rb = (int)(T % TPG % RB);
    mbar_wait(&bar[J & 1], (uint32_t)((J >> 1) & 1));
    tc_fence_after();
    umma_bf16x3(tmem + (uint32_t)(T & 1) * 256, smem_u32(s_colop) + (uint32_t)(J & 1) * kTcBwdBlockBytes,
                smem_u32(s_rowop) + (uint32_t)rb * 256 * kTcRowBytes, idesc);
    umma_commit(&bar[2 + (T & 1)]);
  };

  if (tid == 0) {
    mbar_expect_tx(&bar[4], (uint32_t)K * kTcRowBytes);
    tma_bulk_g2s(s_rowop, a.ws.rowop, (uint32_t)K * kTcRowBytes, &bar[4]);
    issue_block(0);
    issue_block(1);
  }
  mbar_wait(&bar[4], 0);
  if (tid == 0 && ntiles > 0) issue_mma(0);

  float wacc = 0.f, U2 = 0.f, Lc = 0.f;
  for (int64_t T = 0; T < ntiles; ++T) {
    const int64_t j = T / TPG;
    const int t = (int)(T % TPG), cb = t / RB, rb = t % RB;
    const int64_t J = j * CB + cb;
    const int64_t i = blockIdx.x + j * gridDim.x;
    if (t == 0) {
      // ---- group row table (SoA): gamma log2e | (kappa - h) log2e + log2 w_root
      for (int k = tid; k < K; k += NT) {
        // the TC forward stored h - kappa (kappa = -(gamma |u0|^2 + c . u0), the re-centring constant)
        const float hk = a.ws.hmsg[(size_t)i * K + k];
        s_rt[k] = a.ws.fwd_coef[(size_t)k * (kTcD + 2) + 1] * kLog2e;
        s_rt[K + k] = -hk * kLog2e + log2f(a.w_root[k]);  // w_root folded in (log2 0 = -inf)
      }
      __syncthreads();
    }
    const int r_in = quarter * 32 + lane;  // column within the block
    if (rb == 0) {
      const float* xa = a.ws.colaux + (size_t)i * 3 * K + cb * 128 + r_in;
      U2 = xa[0];
      Lc = xa[2 * K] * kLog2e;
      wacc = 0.f;
    }
    mbar_wait(&bar[2 + (T & 1)], (uint32_t)((T >> 1) & 1));
    tc_fence_after();
    if (tid == 0 && T + 1 < ntiles) issue_mma(T + 1);
    // ---- epilogue: column k', rows rb*256 + cq*CW .. +CW
    const uint32_t taddr = tmem + (uint32_t)(T & 1) * 256 + (uint32_t)(cq * CW) + ((uint32_t)(quarter * 32) << 16);
    const float* rt = s_rt + rb * 256 + cq * CW;
    // pairs of rows as float2 (FFMA2/FADD2); w_root is folded into the row
    // constant as log2(w), so each pair costs 3 FMA-pipe lane-ops + 1 ex2 + 1 add
    float2 wp[2] = {f2(0.f), f2(0.f)};
    tmem_pipeline16<NC16>(taddr, [&](int c16, uint32_t(&r)[16]) {
      float gg[16], rc[16];
      lds16(rt + c16 * 16, gg);
      lds16(rt + K + c16 * 16, rc);
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        float2 x = fma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), f2(kLog2e),
                        make_float2(rc[c], rc[c + 1]));
        x = add2(fma2(make_float2(gg[c], gg[c + 1]), f2(U2), x), f2(Lc));
        wp[(c >> 1) & 1] = add2(wp[(c >> 1) & 1], make_float2(ex2(x.x), ex2(x.y)));
      }
    });
    {
      const float2 t2 = add2(wp[0], wp[1]);
      wacc += t2.x + t2.y;
    }
    if (rb == RB - 1) {
      s_wp[cq * 128 + r_in] = wacc;
      __syncthreads();
      if (cq == 0) {
        float wv = 0.f;
#pragma unroll
        for (int q = 0; q < CQ; ++q) wv += s_wp[q * 128 + r_in];
        const int kc = cb * 128 + r_in;
        a.w[(size_t)i * K + kc] = wv;
        s_w[kc] = wv;
        if (isnan(wv)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
      }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0 && rb == RB - 1) issue_block(J + 2);
    if (t == TPG - 1) {
      // ---- moments of group i (fp64): E z, then Var z
      double s1[kTcD];
#pragma unroll
      for (int r = 0; r < kTcD; ++r) s1[r] = 0.0;
      for (int kc = tid; kc < K; kc += NT) {
        const double wv = s_w[kc];
#pragma unroll
        for (int r = 0; r < kTcD; ++r) s1[r] += wv * (double)a.z[((size_t)i * kTcD + r) * K + kc];
      }
#pragma unroll
      for (int r = 0; r < kTcD; ++r) {
        const double v = warp_sum(s1[r]);
        if (lane == 0) s_red[warp * kTcD + r] = v;
      }
      __syncthreads();
      if (tid < kTcD) {
        double m = 0.0;
        for (int w = 0; w < NW; ++w) m += s_red[w * kTcD + tid];
        s_mom[tid] = m;
      }
      __syncthreads();
      double s2[kTcD];
#pragma unroll
      for (int r = 0; r < kTcD; ++r) s2[r] = 0.0;
      for (int kc = tid; kc < K; kc += NT) {
        const double wv = s_w[kc];
#pragma unroll
        for (int r = 0; r < kTcD; ++r) {
          const double dz = (double)a.z[((size_t)i * kTcD + r) * K + kc] - s_mom[r];
          s2[r] += wv * dz * dz;
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kTcD; ++r) {
        const double v = warp_sum(s2[r]);
        if (lane == 0) s_red[warp * kTcD + r] = v;
      }
      __syncthreads();
      if (tid < kTcD) {
        double vv = 0.0;
        for (int w = 0; w < NW; ++w) vv += s_red[w * kTcD + tid];
        a.m1[i * kTcD + tid] = s_mom[tid];
        a.v[i * kTcD + tid] = vv;
      }
      __syncthreads();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
