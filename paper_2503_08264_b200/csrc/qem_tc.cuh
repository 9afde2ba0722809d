// qem_tc.cuh -- tcgen05 tensor-core pair-tile kernels for d = 16 (config 5).
// Included inside namespace qem by qem_two_level.cu (needs TLArgs, inv_fact).
//
// Every log-factor of a pair is an affine function of a 16-dim contraction
// ("Tensor cores"):
//   log2e * (D_k(k') + ln P(k')) = c2_k . u_k' + g2_k |u_k'|^2 + lP(k') + const_k,
// with c2 = log2e c, g2 = log2e gamma, lP = log2e ln P, u = z - mu_ref.  The
// whole expression up to the row constant runs on the 5th-gen tensor cores as
// ONE accumulation into TMEM (kind::f16, fp32 accumulate):
//   6 MMAs  c2 . u       both operands split into three bf16 terms, the six
//                        leading partial products small-first (tools/tc_probe.cu)
//   1 MMA   the "extra" K-slab: row entries [g0 g0 g1 g0 g2 g1 rho0 rho1 | rho2 1 1 1 0 0 0 0]
//                        x column entries  [U0 U1 U0 U2 U0 U1 1 1       | 1 lP0 lP1 lP2 0 0 0 0]
//           (U = |u|^2 and lP split in three bf16; rho = backward row constant)
// so the epilogue per pair is one tcgen05.ld'd value -> ex2 -> add: the SFU
// (MUFU.EX2, 16/clk/SM) and the TMEM read port (64 B/clk/SM) are the ceilings.
//
// Warp roles (one CTA per SM, persistent over groups): warps 0-15 epilogue
// (warp w reads TMEM lane quarter w%4 and column slice w/4), warp 16 TMA
// producer (cp.async.bulk), warp 17 MMA issuer (one thread).  All hand-offs are
// mbarriers: operand stages full/empty, TMEM accumulator buffers (2 x 256
// columns) full/empty; epilogue-only sync uses named barriers.
//
//  k_rowop_tc     c2 -> rowop_c (K x 96 B), forward row extra -> rowop_x (K x 32 B)
//  k_colprep_tc   K2a for d = 16 Bernoulli: unary terms, reference softmax, the
//                 group's tile mode, column operand (128 B per column) + {P, ln P}
//  k_forward_tc   M = 128 parent rows (streamed, static) x N = 256 child columns
//                 (per group); thread = row, online log-sum-exp / expm1 polynomial
//  k_backward_tc  M = 128 child columns (per group) x N = 256 parent rows
//                 (static + per-group extra slab built in SMEM); thread = column
#pragma once

constexpr int kTcD = 16;
constexpr int kTcEpiWarps = 16;
constexpr int kTcThreads = (kTcEpiWarps + 2) * 32;  // + TMA warp + MMA warp
constexpr int kTcEpiThreads = kTcEpiWarps * 32;
constexpr int kTcRowCBytes = kTcRowBytes;  // 96: c2 split (6 chunks)
// Of every 16 exponentials an epilogue thread evaluates, kPolyExp{Fwd,Bwd} go to the FMA
// pipe (exp2_poly2) and the rest to the SFU, so the two pipes share the binding exp load
// (measured on config 5, profiles/r01_poly_exp_sweep.txt: forward best at 2, backward at 4).
#ifndef QEM_POLY_EXP_FWD
#define QEM_POLY_EXP_FWD 2
#endif
#ifndef QEM_POLY_EXP_BWD
#define QEM_POLY_EXP_BWD 4
#endif
constexpr int kPolyExpFwd = QEM_POLY_EXP_FWD, kPolyExpBwd = QEM_POLY_EXP_BWD;
// Where the forward's online mode adds log2e ln P(k'): 1 = the epilogue (fp32, round to nearest), 0 =
// inside the MMA through the extra slab (the tensor core's truncating accumulation biases it by
// ~3e-8 |lP| toward zero, tools/tc_bias.cu; measured cost and accuracy in DESIGN.md "Forward numerics")
#ifndef QEM_LP_EPI
#define QEM_LP_EPI 0
#endif
constexpr bool kLpEpi = QEM_LP_EPI != 0;

// Operand geometry per latent dimension:
//  D = 8..16 ("split"): the c-region of a row / column is the bf16x3 split of the 16-dim
//    (zero-padded) contraction, 96 B, contracted by 6 MMAs (the six leading partial products);
//    the 16-entry extra slab carries gamma |w|^2 (its S pattern), the row constant and ln P.
//  D = 1 ("compact", config 4): the c-region is ONE 16-entry slab holding the six leading partial
//    products of c w AND of gamma S explicitly -- row [c2 c1 c0 c1 c0 c0 g0 g0 | g1 g0 g2 g1 0 0 0 0],
//    column [w0 w1 w2 w0 w1 w0 S0 S1 | S0 S2 S0 S1 0 0 0 0] -- 32 B and one MMA; the extra slab
//    carries only the row constant and ln P (its gamma / S entries are zero).  A column is 64 B.
template <int D>
struct TcGeo {
  static constexpr bool COMPACT = D == 1;
  static constexpr int CB = COMPACT ? 32 : 96;   // c-region bytes per row / column
  static constexpr int COL = CB + kTcRowXBytes;  // column operand bytes (c-region + extra slab)
  static constexpr int XKK = CB / 2;             // bf16 index where a column's extra slab starts
  __host__ __device__ static int col_off(int row, int kk) { return tc_off(row, kk, COL); }
  __host__ __device__ static int row_off(int row, int kk) { return tc_off(row, kk, CB); }
};

// compact c-region (D = 1) of a row (c = log2e c_k, g = log2e gamma_k) and of a column (w, S)
__device__ __forceinline__ void compact_row(float c, float g, uint4& c0, uint4& c1) {
  __nv_bfloat16 cs[3], gs[3];
  split3_bf16(c, cs);
  split3_bf16(g, gs);
  const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
  const __nv_bfloat16 a[8] = {cs[2], cs[1], cs[0], cs[1], cs[0], cs[0], gs[0], gs[0]};
  const __nv_bfloat16 b[8] = {gs[1], gs[0], gs[2], gs[1], z, z, z, z};
  c0 = pack8_bf16(a);
  c1 = pack8_bf16(b);
}
__device__ __forceinline__ void compact_col(float w, float S, uint4& c0, uint4& c1) {
  __nv_bfloat16 ws[3], ss[3];
  split3_bf16(w, ws);
  split3_bf16(S, ss);
  const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
  const __nv_bfloat16 a[8] = {ws[0], ws[1], ws[2], ws[0], ws[1], ws[0], ss[0], ss[1]};
  const __nv_bfloat16 b[8] = {ss[0], ss[2], ss[0], ss[1], z, z, z, z};
  c0 = pack8_bf16(a);
  c1 = pack8_bf16(b);
}

// named barriers: 1 = all epilogue warps, 2..5 = the 4 warps of one TMEM lane quarter
__device__ __forceinline__ void epi_bar() { named_bar(1, kTcEpiThreads); }
__device__ __forceinline__ void quarter_bar(int q) { named_bar(2 + q, 128); }

// bf16x3 split of the 16-entry extra slab of a row / column (two 16-byte chunks)
__device__ __forceinline__ void extra_row(float g2, float lp_on, float rho, uint4& c0, uint4& c1) {
  __nv_bfloat16 g[3], r[3];
  split3_bf16(g2, g);
  split3_bf16(rho, r);
  const __nv_bfloat16 z = __float2bfloat16_rn(0.f), on = __float2bfloat16_rn(lp_on);
  // chunk 6: the six gamma split terms + rho0 rho1; chunk 7: rho2 + the lP switch (x3) -- the
  // column side keeps every lP entry in chunk 7, so patching lP rewrites one whole 16-byte chunk
  const __nv_bfloat16 a[8] = {g[0], g[0], g[1], g[0], g[2], g[1], r[0], r[1]};
  const __nv_bfloat16 b[8] = {r[2], on, on, on, z, z, z, z};
  c0 = pack8_bf16(a);
  c1 = pack8_bf16(b);
}
__device__ __forceinline__ void extra_col(float U, float lp, uint4& c0, uint4& c1) {
  __nv_bfloat16 u[3], l[3];
  split3_bf16(U, u);
  split3_bf16(lp, l);
  const __nv_bfloat16 z = __float2bfloat16_rn(0.f), one = __float2bfloat16_rn(1.f);
  const __nv_bfloat16 a[8] = {u[0], u[1], u[0], u[2], u[0], u[1], one, one};
  const __nv_bfloat16 b[8] = {one, l[0], l[1], l[2], z, z, z, z};
  c0 = pack8_bf16(a);
  c1 = pack8_bf16(b);
}

// 7 MMAs of one 128 x 256 tile: 6 split products (small first) + the extra slab.
__device__ __forceinline__ void umma_tile7(uint32_t tmem_d, uint32_t a_c, uint32_t a_sbo, uint32_t b_c, uint32_t b_sbo,
                                           uint32_t a_x, uint32_t a_xsbo, uint32_t b_x, uint32_t b_xsbo,
                                           uint32_t idesc) {
  const int pa[6] = {2, 1, 0, 1, 0, 0}, pb[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
  for (int q = 0; q < 6; ++q)
    umma_bf16(tmem_d, umma_desc(a_c + pa[q] * 256, 128, a_sbo), umma_desc(b_c + pb[q] * 256, 128, b_sbo), idesc,
              q > 0);
  umma_bf16(tmem_d, umma_desc(a_x, 128, a_xsbo), umma_desc(b_x, 128, b_xsbo), idesc, 1u);
}

// One tile: the c-region MMAs (6 split products, or the compact slab) + the extra slab.
template <int D>
__device__ __forceinline__ void umma_tile(uint32_t tmem_d, uint32_t a_c, uint32_t a_sbo, uint32_t b_c, uint32_t b_sbo,
                                          uint32_t a_x, uint32_t a_xsbo, uint32_t b_x, uint32_t b_xsbo, uint32_t idesc) {
  if constexpr (TcGeo<D>::COMPACT) {
    umma_bf16(tmem_d, umma_desc(a_c, 128, a_sbo), umma_desc(b_c, 128, b_sbo), idesc, 0u);
    umma_bf16(tmem_d, umma_desc(a_x, 128, a_xsbo), umma_desc(b_x, 128, b_xsbo), idesc, 1u);
  } else {
    umma_tile7(tmem_d, a_c, a_sbo, b_c, b_sbo, a_x, a_xsbo, b_x, b_xsbo, idesc);
  }
}

// 16-dim row vector -> bf16x3 split in the 96-byte canonical row layout (tc_offset)
__device__ __forceinline__ void store_row_split16(unsigned char* base, int k, const float (&v)[kTcD]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // 8 dims per 16-byte chunk
    __nv_bfloat16 s[3][8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      __nv_bfloat16 t[3];
      split3_bf16(v[8 * h + r], t);
      s[0][r] = t[0];
      s[1][r] = t[1];
      s[2][r] = t[2];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) *reinterpret_cast<uint4*>(base + tc_offset(k, q * 16 + 8 * h)) = pack8_bf16(s[q]);
  }
}

template <int D>
__device__ __forceinline__ double root_lnv(const TLArgs& a, int k) {
  if (a.scale_kind == QEM_SCALE_FIXED) return log(a.fixed_var);
  const double s = (double)a.z_root[D * a.K + k];
  return a.scale_kind == QEM_SCALE_LOGSIGMA ? 2.0 * s : s;
}

// Inside k_root (one block, after the root softmax; w = root weights in fp64):
// the backward reference row k* = argmax_k w_root(k) (ties -> lowest k) and the
// k*-differenced rows  E_k(z) = B(k,z) - B(k*,z) = Ea_k + Eb_k . z + Eg_k |z|^2,
// Eb_k = e_k mu_k - e_* mu_*, Eg_k = -(e_k - e_*)/2, differenced in fp64 (DESIGN.md
// "Backward reference"): bf16x3 row operand + log2e Eg for the tensor-core path,
// fp32 [K][D+1] rows for the FFMA path.
template <int D>
__device__ void k_root_star(const TLArgs& a, const double* w) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  const int K = a.K, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int k = tid; k < K; k += blockDim.x)
    if (w[k] > best) {
      best = w[k];
      bi = k;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_v[wid] = best;
    s_i[wid] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 1; q < (int)((blockDim.x + 31) >> 5); ++q)
      if (s_v[q] > s_v[0] || (s_v[q] == s_v[0] && s_i[q] < s_i[0])) {
        s_v[0] = s_v[q];
        s_i[0] = s_i[q];
      }
    if (s_i[0] >= K) s_i[0] = 0;  // all weights NaN (degenerate evidence, flagged by k_root): stay in range
    const int ks = s_i[0];
    RefInfo* ref = a.ws.ref;
    ref->k_star = ks;
    float mu[D];  // loads before stores (they could alias)
#pragma unroll
    for (int r = 0; r < D; ++r) mu[r] = a.z_root[r * K + ks];
#pragma unroll
    for (int r = 0; r < D; ++r) ref->mu_star[r] = mu[r];
    const double lnv = root_lnv<D>(a, ks);
    ref->e_star = exp(-lnv);
    ref->bstar_const = -0.5 * D * (kLn2Pi + lnv);
  }
  __syncthreads();
  const int ks = s_i[0];
  const double es = exp(-root_lnv<D>(a, ks));
  // the reference rows' coordinates in registers before the row loop (its stores could alias them)
  float zs_[D], zref_[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    zs_[r] = a.z_root[r * K + ks];
    zref_[r] = a.ws.ref->mu_ref[r];
  }
  for (int k = tid; k < K; k += blockDim.x) {
    const double ek = exp(-root_lnv<D>(a, k));
    float zk_[D];
#pragma unroll
    for (int r = 0; r < D; ++r) zk_[r] = a.z_root[r * K + k];
    if constexpr (TcGeo<D>::COMPACT) {
      if (a.tc) {  // Eb and Eg both in the compact c-region; the per-group slab's gamma stays 0
        uint4 c0, c1;
        const double zr0 = zref_[0];
        compact_row((float)((ek * ((double)zk_[0] - zr0) - es * ((double)zs_[0] - zr0)) * kLog2eD),
                    (float)(-0.5 * (ek - es) * kLog2eD), c0, c1);
        unsigned char* rb = reinterpret_cast<unsigned char*>(a.ws.rowop_b);
        *reinterpret_cast<uint4*>(rb + TcGeo<D>::row_off(k, 0)) = c0;
        *reinterpret_cast<uint4*>(rb + TcGeo<D>::row_off(k, 8)) = c1;
        a.ws.bgam[k] = 0.f;
        continue;
      }
    } else if constexpr (D <= kTcD) {
      if (a.tc) {
        float v[kTcD];
#pragma unroll
        for (int r = 0; r < kTcD; ++r)
          v[r] = r < D ? (float)((ek * ((double)zk_[r] - (double)zref_[r]) - es * ((double)zs_[r] - (double)zref_[r])) *
                                 kLog2eD)
                       : 0.f;
        store_row_split16(reinterpret_cast<unsigned char*>(a.ws.rowop_b), k, v);
        a.ws.bgam[k] = (float)(-0.5 * (ek - es) * kLog2eD);
        continue;
      }
    }
    float* bc = a.ws.bwd_coef + (size_t)k * (D + 1);
    for (int r = 0; r < D; ++r) bc[r] = (float)(ek * (double)zk_[r] - es * (double)zs_[r]);
    bc[D] = (float)(-0.5 * (ek - es));
  }
}

// ------------------------------------------------------------------ rowop
template <int D>
__global__ void __launch_bounds__(256) k_rowop_tc(TLArgs a) {
  const int K = a.K;
  unsigned char* rc = reinterpret_cast<unsigned char*>(a.ws.rowop);
  unsigned char* rx = reinterpret_cast<unsigned char*>(a.ws.rowop_x);
  constexpr int RS = pad4(D + 3);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    // log2e c_k, log2e gamma_k rounded once from fp64 (k_root_prep's bwd_table row; coef_d holds the
    // same values in natural units for the aux merge)
    const float* bt = a.ws.bwd_table + (size_t)k * RS;
    if constexpr (TcGeo<D>::COMPACT) {
      uint4 c0, c1;
      compact_row(bt[2], bt[1], c0, c1);
      *reinterpret_cast<uint4*>(rc + TcGeo<D>::row_off(k, 0)) = c0;
      *reinterpret_cast<uint4*>(rc + TcGeo<D>::row_off(k, 8)) = c1;
      extra_row(0.f, kLpEpi ? 0.f : 1.f, 0.f, c0, c1);  // forward: no row constant, gamma in the c-region
      *reinterpret_cast<uint4*>(rx + tc_rowx_offset(k, 0)) = c0;
      *reinterpret_cast<uint4*>(rx + tc_rowx_offset(k, 8)) = c1;
      continue;
    }
    float v[kTcD];  // contraction zero-padded to 16 dims
#pragma unroll
    for (int r = 0; r < kTcD; ++r) v[r] = r < D ? bt[2 + r] : 0.f;
    store_row_split16(rc, k, v);
    uint4 c0, c1;
    extra_row(bt[1], kLpEpi ? 0.f : 1.f, 0.f, c0, c1);  // forward: no row constant; lP switch
    *reinterpret_cast<uint4*>(rx + tc_rowx_offset(k, 0)) = c0;
    *reinterpret_cast<uint4*>(rx + tc_rowx_offset(k, 8)) = c1;
  }
}

// -------------------------------------------------------------- colprep (K2a)
// One warp per group.  For column k': A_i(k') (fp64), t_i(k') = B(k_ref,k') + A_i(k'),
// c_i = lse t - log K, P = softmax t; the group's tile mode from the bound on
// |D'|; the column operand and {P, ln P}.
// softplus(eta) = max(eta, 0) + log1p(e^-|eta|): v = 2^(-|eta| log2e) on the SFU, log1p(v) by a
// polynomial on the FMA pipe; absolute error <= ~1.5e-7 per observation (R26).

// log1p(v), v in [0, 1], two at a time on the FMA pipe: v p(v) with p of degree 8 (near-minimax
// for the absolute error, 5e-9; <= 1.4e-7 evaluated in fp32)
__device__ __forceinline__ float2 log1p01_poly2(float2 v) {
  float2 p = f2(3.929332364e-03f);
  p = fma2(p, v, f2(-2.385043912e-02f));
  p = fma2(p, v, f2(6.807538122e-02f));
  p = fma2(p, v, f2(-1.268995851e-01f));
  p = fma2(p, v, f2(1.856928021e-01f));
  p = fma2(p, v, f2(-2.467250526e-01f));
  p = fma2(p, v, f2(3.328963518e-01f));
  p = fma2(p, v, f2(-4.999709129e-01f));
  p = fma2(p, v, f2(9.999993443e-01f));
  return mul2(p, v);
}

// softplus of an observation pair {eta_2p, eta_2p+1} summed (the second dropped when it is the
// zero padding of an odd J): max(eta, 0) + log1p(2^(-|eta| log2e)), one MUFU per observation
__device__ __forceinline__ float softplus_pair(float2 eta, bool two) {
  const float2 v = make_float2(ex2(-fabsf(eta.x) * kLog2e), two ? ex2(-fabsf(eta.y) * kLog2e) : 0.f);
  const float2 l = log1p01_poly2(v);
  return (fmaxf(eta.x, 0.f) + (two ? fmaxf(eta.y, 0.f) : 0.f)) + (l.x + l.y);
}

#ifndef QEM_COLPREP_MINB
#define QEM_COLPREP_MINB 2  // resident CTAs per SM the column prep is compiled for (register budget)
#endif
#ifndef QEM_PREP_ZST
#define QEM_PREP_ZST 2  // z stages per warp (1: the loads of a bound z are not prefetched, less SMEM)
#endif
struct PrepTc {
  static constexpr int WARPS = 8;
  static constexpr int ZST = QEM_PREP_ZST;
  static constexpr int ZS_FLOATS = ZST * 2 * kTcD * 32;  // z ring: [stage][half][r][32 columns]
  static constexpr size_t ZS_BYTES = ZS_FLOATS * 4;
  __host__ __device__ static size_t warp_bytes(int K, int J) {
    size_t b = 3 * kTcD * 8 + 3 * kTcD * 4 + (size_t)((J + 1) / 2) * kTcD * 8 + ZS_BYTES;
    return (b + 15) & ~(size_t)15;
  }
  __host__ __device__ static size_t bytes(int K, int J) { return WARPS * warp_bytes(K, J); }
};

// 8 <= D <= 16 latent dims (the contraction is zero-padded to 16); Bernoulli-logit observations
// (configs 2/5 shape; the OBS parameter keeps the Gaussian likelihood for d = 1 experiments).
template <int D, int OBS>
__global__ void __launch_bounds__(256, QEM_COLPREP_MINB) k_colprep_tc(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  static_assert(D <= kTcD, "tensor-core path: d <= 16");
  static_assert(D % 2 == 0, "pairs of dims per 8-byte load");
  const int K = a.K, J = a.J, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* wb = smem + (size_t)wid * PrepTc::warp_bytes(K, J);
  // per-group column quadratic (fp64): with w = z - m_i (exact in fp64),
  //   B(k_ref, k') - ln q(z) + sum_j y_j eta_j = C_i + sum_r w_r (alpha_r w_r + beta_r),
  //   alpha_r = 1/(2 v_r) - e_ref/2,  beta_r = (sum_j y_j x_jr) - e_ref (m_r - mu_ref,r),
  //   C_i = bref_const - (e_ref/2) |m - mu_ref|^2 + sum_r (ln 2pi v_r)/2 + (sum_j y_j x_j) . m
  // (the three terms of t_ref collected per dimension; oracle: separate fp64 sums)
  double* qm = reinterpret_cast<double*>(wb);                      // [D]  m_i
  double2* qab = reinterpret_cast<double2*>(qm + kTcD);            // [D]  {alpha_r, beta_r}
  float* qmf = reinterpret_cast<float*>(qab + kTcD);               // [D]  m_i (fp32, exact: R22)
  float* u0f = qmf + kTcD;                                         // [D]  u0_i = m_i - mu_ref (fp32)
  float* sdf = u0f + kTcD;                                         // [D]  sqrt(v_i) (fp32, the sampler's)
  float2* xp = reinterpret_cast<float2*>(sdf + kTcD);              // [(J+1)/2][D] {x_2p, x_2p+1} as 0/1
  const int Jh = (J + 1) / 2;
  float* zs = reinterpret_cast<float*>(xp + (size_t)Jh * kTcD);    // z ring (PrepTc::ZS_FLOATS)
  // z of 32 column pairs {kc, kc + K/2} of group g into ring stage st: LDGSTS, so the loads of
  // iteration it + 1 fly while iteration it computes (the column loop is latency-bound otherwise)
  auto stage_z = [&](int64_t g, int it, int st) {
    const float* zg = a.z + (size_t)g * D * K + it * 32;
    float* dst = zs + st * (2 * kTcD * 32);
#pragma unroll
    for (int c = lane; c < 2 * D * 8; c += 32) {
      const int h = c / (D * 8), r = (c / 8) % D, p = c % 8;
      cp_async16(dst + (h * kTcD + r) * 32 + p * 4, zg + (size_t)r * K + h * (K / 2) + p * 4);
    }
    cp_async_commit();
  };
  // Fused sampler (qem_sample_estep_forward / qem_iterate): instead of loading z, draw it -- the
  // same Philox counters and Box-Muller as k_sample (philox_normal4), z = fmaf(sqrt(v), eps, m) in
  // fp32 (R22), so the samples are bit-identical -- write it to the bound z (the backward's column
  // constants and the moments read it) and into the stage.  Lane: one quad of 4 columns x one dim.
  const bool fuse = a.fuse_sample != 0;
  const uint32_t zword = (1u << 24) | ((uint32_t)resolve_iter(a.t_sample, &a.cnt->iter) & 0xffffffu);
  float* zout = const_cast<float*>(a.z);
  auto gen_z = [&](int64_t g, int it, int st) {
    float* dst = zs + st * (2 * kTcD * 32);
    const uint32_t ginst = (uint32_t)(a.g_begin + g);
#pragma unroll
    for (int c = lane; c < 2 * D * 8; c += 32) {
      const int h = c / (D * 8), r = (c / 8) % D, p = c % 8;
      const int k0 = h * (K / 2) + it * 32 + p * 4;
      const float4 e = philox_normal4(make_uint4((uint32_t)(k0 >> 2), (uint32_t)r, ginst, zword), a.skey);
      const float m = qmf[r], sd = sdf[r];
      const float4 zz = make_float4(__fmaf_rn(sd, e.x, m), __fmaf_rn(sd, e.y, m), __fmaf_rn(sd, e.z, m),
                                    __fmaf_rn(sd, e.w, m));
      *reinterpret_cast<float4*>(dst + (h * kTcD + r) * 32 + p * 4) = zz;
      *reinterpret_cast<float4*>(zout + ((size_t)g * D + r) * K + k0) = zz;
    }
  };
  const int NIT = K / 64;  // K % 256 == 0 on this path
  const double bref_const = a.ws.ref->bref_const, e_ref = a.ws.ref->e_ref;
  const float mref_l = lane < D ? a.ws.ref->mu_ref[lane] : 0.f;
  const double logK = log((double)K);
  double gc0 = 0.0, gc1 = 0.0;
  if constexpr (OBS == QEM_OBS_GAUSS) {
    gc0 = -0.5 * J * (kLn2Pi + log(a.obs_var));
    gc1 = 0.5 / a.obs_var;
  }
  unsigned char* colop = reinterpret_cast<unsigned char*>(a.ws.colop);
  // S = a.prep_split warps share a group (1, 2, 4 or 8, <= K/64; more when the rank's groups are too
  // few to fill the SMs one warp each): warp slice sl takes the column iterations it = sl, sl + S, ...
  // Every group-wide quantity is formed in an order that does not depend on S (the softmax over the
  // t_ref the slices wrote, max reductions), so the results are bit-identical for every S.
  const int S = a.prep_split, gslot = wid / S, sl = wid % S;
  const int64_t gstride = (int64_t)gridDim.x * (PrepTc::WARPS / S);
  const int64_t gfirst = (int64_t)blockIdx.x * (PrepTc::WARPS / S) + gslot;
  __shared__ float s_w2[PrepTc::WARPS];
  // max_k |gamma_k| (the rows are the same for every group): the tile-mode bound below is >= max_k
  // |gamma_k| max |w|^2, so a group whose that alone passes the highest Taylor threshold is online
  // without the bound's K x D pass over the rows
  float gmax = 0.f;
  for (int k = lane; k < K; k += 32) gmax = fmaxf(gmax, fabsf(__ldg(a.ws.fwd_coef + (size_t)k * (D + 2) + 1)));
  gmax = warp_maxf(gmax);
  constexpr int ZST = PrepTc::ZST;
  if (ZST == 2 && !fuse && gfirst < a.n_local) stage_z(gfirst, sl, 0);
  for (int64_t i = gfirst; i < a.n_local; i += gstride) {
    __syncwarp();
    double sx = 0.0, sxx = 0.0;
    int yxi = 0;  // sum_j y_j x_j,lane (integer)
    if constexpr (OBS == QEM_OBS_GAUSS) {
      // sufficient statistics of the group's observations (d = 1)
      const float* x = reinterpret_cast<const float*>(a.x) + i * J;
      for (int jj = lane; jj < J; jj += 32) {
        const double xv = x[jj];
        sx += xv;
        sxx += xv * xv;
      }
      sx = warp_sum(sx);
      sxx = warp_sum(sxx);
    } else {
      const uint8_t* x = reinterpret_cast<const uint8_t*>(a.x) + (size_t)i * J * D;
      const uint8_t* y = reinterpret_cast<const uint8_t*>(a.y) + (size_t)i * J;
      for (int e = lane; e < Jh * D; e += 32) {
        const int jp = e / D, r = e % D, j0 = 2 * jp, j1 = 2 * jp + 1;
        xp[e] = make_float2(x[j0 * D + r] ? 1.f : 0.f, (j1 < J && x[j1 * D + r]) ? 1.f : 0.f);
      }
      if (lane < D)
        for (int j = 0; j < J; ++j) yxi += (y[j] && x[j * D + lane]) ? 1 : 0;
    }
    double ci = 0.0;
    if (lane < D) {
      const double m = a.q_m[i * D + lane], v = a.q_v[i * D + lane], dl = m - (double)mref_l;
      qm[lane] = m;
      qmf[lane] = (float)m;
      u0f[lane] = (float)m - mref_l;
      sdf[lane] = __fsqrt_rn(a.q_v[i * D + lane]);  // as k_sample
      qab[lane] = make_double2(0.5 / v - 0.5 * e_ref, (double)yxi - e_ref * dl);
      ci = 0.5 * (kLn2Pi + log(v)) - 0.5 * e_ref * dl * dl + (double)yxi * m;
    }
    const double Ci = bref_const + warp_sum(ci);
    __syncwarp();
    unsigned char* cop = colop + (size_t)i * K * kTcColBytes;
    float w2max = 0.f;
    // the rest of a column once its likelihood is known: log q, the column operand, t_ref
    auto finish = [&](int kc, const float (&zr)[D], double ll) {
      // group constants re-read from SMEM (volatile keeps ptxas from hoisting them into registers)
      const volatile double* qmv = qm;
      const volatile double2* qabv = qab;
      const volatile float* qmfv = qmf;
      const volatile float* u0fv = u0f;
      double quad = Ci;
      // column operand re-centred on the group's Q mean: w = z - m_i and
      // S = |w|^2 + 2 u0_i . w, u0_i = m_i - mu_ref (so D_k(z) = alpha'_ik + c_k . w + gamma_k S)
      float W2 = 0.f, mw = 0.f;
      float wv[kTcD];
#pragma unroll
      for (int r = 0; r < kTcD; ++r) {
        if (r < D) {
          const double md = qmv[r];
          const double2 ab = const_cast<const double2&>(qabv[r]);
          const double wd = (double)zr[r] - md;
          quad = fma(wd, fma(ab.x, wd, ab.y), quad);
          const float m = qmfv[r];
          wv[r] = zr[r] - m;
          W2 = fmaf(wv[r], wv[r], W2);
          mw = fmaf(u0fv[r], wv[r], mw);
        } else {
          wv[r] = 0.f;  // zero-padded contraction
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // bf16x3 split of w, 8 dims (one 16-byte chunk per term) at a time
        if (8 * h >= D) {
          const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int q = 0; q < 3; ++q) *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, q * 16 + 8 * h)) = zero;
          continue;
        }
        __nv_bfloat16 s0[8], s1[8], s2[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          __nv_bfloat16 t[3];
          split3_bf16(wv[8 * h + r], t);
          s0[r] = t[0];
          s1[r] = t[1];
          s2[r] = t[2];
        }
        *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, 0 * 16 + 8 * h)) = pack8_bf16(s0);
        *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, 1 * 16 + 8 * h)) = pack8_bf16(s1);
        *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, 2 * 16 + 8 * h)) = pack8_bf16(s2);
      }
      {  // extra slab, first chunk: [S pattern | 1 1]; the second (1, lP) is written below
        uint4 c0, c1;
        extra_col(fmaf(2.f, mw, W2), 0.f, c0, c1);
        *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, 48)) = c0;
      }
      // t_ref(k') = B(k_ref,k') + A_i(k') (fp64; the backward rebuilds A from it)
      const double t = quad + ll;
      a.ws.tA[(size_t)i * K + kc] = t;
      w2max = fmaxf(w2max, W2);
    };
    // Two columns per lane at a time (kc and kc + K/2): the per-observation feature loads are
    // shared and the two likelihood chains hide each other's latency.
    for (int it = sl, li = 0; it < NIT; it += S, ++li) {
      if (fuse) {
        gen_z(i, it, (li & 1) & (ZST - 1));
      } else if (ZST == 1) {
        stage_z(i, it, 0);
        cp_async_wait<0>();
      } else if (it + S < NIT) {
        stage_z(i, it + S, (li + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const float* zst = zs + ((li & 1) & (ZST - 1)) * (2 * kTcD * 32);
      const int kcA = it * 32 + lane, kcB = kcA + K / 2;
      float zA[D], zB[D];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        zA[r] = zst[r * 32 + lane];
        zB[r] = zst[(kTcD + r) * 32 + lane];
      }
      double llA, llB;
      if constexpr (OBS == QEM_OBS_GAUSS) {
        const double za = zA[0], zb = zB[0];
        llA = gc0 - (sxx - 2.0 * za * sx + (double)J * za * za) * gc1;
        llB = gc0 - (sxx - 2.0 * zb * sx + (double)J * zb * zb) * gc1;
      } else {
        // label part sum_j y_j eta_j is in the column quadratic (beta_r, C_i); softplus part per
        // observation, two observations at a time (FFMA2), for both columns
        double lspA = 0.0, lspB = 0.0;
        for (int jp = 0; jp < Jh; ++jp) {
          const float2* xr = xp + jp * D;
          float2 a0 = f2(0.f), a1 = f2(0.f), b0 = f2(0.f), b1 = f2(0.f);
          if constexpr (D % 2 == 0) {
#pragma unroll
            for (int q = 0; q < D / 2; ++q) {  // 128-bit loads: features 2q, 2q+1 of both observations
              const float4 xv = reinterpret_cast<const float4*>(xr)[q];
              a0 = fma2(make_float2(xv.x, xv.y), f2(zA[2 * q]), a0);
              a1 = fma2(make_float2(xv.z, xv.w), f2(zA[2 * q + 1]), a1);
              b0 = fma2(make_float2(xv.x, xv.y), f2(zB[2 * q]), b0);
              b1 = fma2(make_float2(xv.z, xv.w), f2(zB[2 * q + 1]), b1);
            }
          } else {
#pragma unroll
            for (int r = 0; r < D; ++r) {
              if (r & 1) {
                a1 = fma2(xr[r], f2(zA[r]), a1);
                b1 = fma2(xr[r], f2(zB[r]), b1);
              } else {
                a0 = fma2(xr[r], f2(zA[r]), a0);
                b0 = fma2(xr[r], f2(zB[r]), b0);
              }
            }
          }
          const float2 ea = add2(a0, a1), eb = add2(b0, b1);
          const bool two = 2 * jp + 1 < J;
          lspA += (double)softplus_pair(ea, two);
          lspB += (double)softplus_pair(eb, two);
        }
        llA = -lspA;
        llB = -lspB;
      }
      finish(kcA, zA, llA);
      finish(kcB, zB, llB);
      __syncwarp();  // the stage is refilled two iterations on
    }
    if (ZST == 2 && !fuse && i + gstride < a.n_local) stage_z(i + gstride, sl, 0);  // next group's first stage, under the passes below
    // the group's slices meet: t_ref (global) and the slices' max |w|^2 (shared) visible to all of them
    float W2max = warp_maxf(w2max);
    if (S > 1) {
      if (lane == 0) s_w2[wid] = W2max;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + gslot), "r"(32 * S) : "memory");
      W2max = 0.f;
      for (int q = 0; q < S; ++q) W2max = fmaxf(W2max, s_w2[gslot * S + q]);
    }
    // softmax over the group's columns from t_ref in a fixed order (lane l: columns l, l + 32, ...;
    // then the warp tree), whatever S wrote them: M, then sum of e^(t - M)
    const double* tref = a.ws.tA + (size_t)i * K;
    double tmax = -CUDART_INF;
    for (int kc = lane; kc < K; kc += 32) tmax = fmax(tmax, __ldcg(tref + kc));
    const double M = warp_max(tmax);
    double tsum = 0.0;
    for (int kc = lane; kc < K; kc += 32) tsum += (double)expf((float)(__ldcg(tref + kc) - M));
    const double logS = log(warp_sum(tsum));
    // tile mode: bound on |D'_k(k')| = |c'_k . w + gamma_k |w|^2|, c' = c0 + 2 gamma m_i
    float u0[D];
#pragma unroll
    for (int r = 0; r < D; ++r) u0[r] = u0f[r];
    const float wmax = sqrtf(W2max);
    float tb = gmax * W2max;
#pragma unroll 4  // fwd_coef rows stream from L2: keep several rows' loads in flight
    for (int k = tb > a.thr[4] ? K : lane; k < K; k += 32) {
      const float2* fc = reinterpret_cast<const float2*>(a.ws.fwd_coef + (size_t)k * (D + 2));  // D even
      const float2 h = __ldg(fc);
      const float g = h.y;
      float cn = 0.f;
#pragma unroll
      for (int q = 0; q < D / 2; ++q) {
        const float2 c = __ldg(fc + 1 + q);
        const float cp0 = fmaf(2.f * g, u0[2 * q], c.x), cp1 = fmaf(2.f * g, u0[2 * q + 1], c.y);
        cn = fmaf(cp0, cp0, cn);
        cn = fmaf(cp1, cp1, cn);
      }
      tb = fmaxf(tb, sqrtf(cn) * wmax + fabsf(g) * W2max);
    }
    tb = warp_maxf(tb);
    const int md = tb <= a.thr[0] ? 0 : (tb <= a.thr[1] ? 1 : (tb <= a.thr[2] ? 2 : (tb <= a.thr[3] ? 3 : (tb <= a.thr[4] ? 4 : 5))));
    float* aux = a.ws.colaux + (size_t)i * 2 * K;  // P (the forward's poly modes), first K slots
    for (int kb = lane + 32 * sl; kb < K; kb += 256 * S) {  // 8 columns per lane per batch: loads in flight together
      double tb4[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tb4[u] = kb + 32 * S * u < K ? __ldcg(tref + kb + 32 * S * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kc = kb + 32 * S * u;
        if (kc >= K) break;
        const double lpd = tb4[u] - M - logS;
        // the forward's per-column weight: P (polynomial modes) or log2e ln P (online mode), which the
        // epilogue ADDS to the MMA's D' in fp32 (round to nearest).  Inside the MMA the tensor core's
        // accumulation (aligned to the largest product, truncated) would bias every pair by ~3e-8 |lP|
        // toward zero -- upward, coherently over the groups' plate sum (tools/tc_bias.cu).  log2e ln P
        // is rounded once from fp64 (the fp32 log2e would scale it by 1 - 1.3e-8: the same kind of bias).
        const float lp2 = (float)(lpd * kLog2eD);
        aux[kc] = (md == 5 && kLpEpi) ? lp2 : expf((float)lpd);
        uint4 c0, c1;
        extra_col(0.f, (md == 5 && !kLpEpi) ? lp2 : 0.f, c0, c1);  // (the backward writes L* there)
        *reinterpret_cast<uint4*>(cop + tc_col_offset(kc, 56)) = c1;  // chunk 7: 1 lP0 lP1 lP2 0...
      }
    }
    if (lane == 0 && sl == 0) {
      a.ws.cvec[i] = M + logS - logK;
      a.ws.gstat[i] = W2max;
      a.ws.gmode[i] = md;
    }
    if (S > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + gslot), "r"(32 * S) : "memory");  // s_w2 reuse
  }
}

// -------------------------------------------- colprep, compact path (K2a, D = 1, config 4)
// One warp per group (persistent over groups), lanes over the group's columns.  Per column k':
//   t_ref(k') = B(k_ref,k') + A_i(k') = bref - (e_ref/2)(z - mu_ref)^2 + ll(z) - ln q(z)   (fp64;
//   ll = the Gaussian likelihood through the group's sufficient statistics, as k_colprep),
//   w = z - m_i, S = w^2 + 2 m_i w (fp32)  -> the compact c-region + extra chunk 0 [0 .. 0 1 1];
// then P = softmax t_ref from the lanes' online (max, sum), the group's tile mode from the bound on
// |D'_k(k')| = |c'_k w + gamma_k w^2| (c' = c0 + 2 gamma m_i), P -> colaux, and ln P into the extra
// slab's second chunk (online mode only).  No shared memory: t_ref is re-read from L1/L2.
template <int OBS>
__global__ void __launch_bounds__(256) k_colprep_tc1(TLArgs a) {
  using G = TcGeo<1>;
  static_assert(OBS == QEM_OBS_GAUSS, "compact tensor-core path: Gaussian observations");
  const int K = a.K, J = a.J, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const double bref = a.ws.ref->bref_const, e_ref = a.ws.ref->e_ref;
  const double mref = (double)a.ws.ref->mu_ref[0];
  const double logK = log((double)K);
  const double gc0 = -0.5 * J * (kLn2Pi + log(a.obs_var)), gc1 = 0.5 / a.obs_var;
  unsigned char* colop = reinterpret_cast<unsigned char*>(a.ws.colop);
  for (int64_t i = (int64_t)blockIdx.x * nw + wid; i < a.n_local; i += (int64_t)gridDim.x * nw) {
    const float* x = reinterpret_cast<const float*>(a.x) + i * J;
    double sx = 0.0, sxx = 0.0;
    for (int j = lane; j < J; j += 32) {
      const double xv = x[j];
      sx += xv;
      sxx += xv * xv;
    }
    sx = warp_sum(sx);
    sxx = warp_sum(sxx);
    const float mf = a.q_m[i];
    const float u0f = mf - (float)mref;  // u0_i = m_i - mu_ref (the columns' S = w^2 + 2 u0 w)
    const double m = mf, v = a.q_v[i];
    const double lqc = -0.5 * (kLn2Pi + log(v)), iv2 = 0.5 / v;
    unsigned char* cop = colop + (size_t)i * K * G::COL;
    const float* zi = a.z + (size_t)i * K;
    double* tref = a.ws.tA + (size_t)i * K;
    double tmax = -CUDART_INF, tsum = 0.0;
    float w2max = 0.f;
#pragma unroll 4
    for (int kc = lane; kc < K; kc += 32) {
      const float zf = zi[kc];
      const double z = zf, dz = z - m, u = z - mref;
      const double lq = lqc - dz * dz * iv2;
      const double ll = gc0 - (sxx - 2.0 * z * sx + (double)J * z * z) * gc1;
      const double t = bref - 0.5 * e_ref * u * u + (ll - lq);
      tref[kc] = t;
      if (t > tmax) {
        tsum = fma(tsum, (double)expf((float)(tmax - t)), 1.0);
        tmax = t;
      } else {
        tsum += (double)expf((float)(t - tmax));
      }
      const float w = zf - mf, W2 = w * w;
      uint4 c0, c1;
      compact_col(w, fmaf(2.f, u0f * w, W2), c0, c1);
      *reinterpret_cast<uint4*>(cop + G::col_off(kc, 0)) = c0;
      *reinterpret_cast<uint4*>(cop + G::col_off(kc, 8)) = c1;
      extra_col(0.f, 0.f, c0, c1);  // chunk 0: [0 0 0 0 0 0 1 1]; chunk 1 (1, lP) below
      *reinterpret_cast<uint4*>(cop + G::col_off(kc, G::XKK)) = c0;
      w2max = fmaxf(w2max, W2);
    }
    const double M = warp_max(tmax);
    const float W2max = warp_maxf(w2max);
    const double logS = log(warp_sum(tsum * (double)expf((float)(tmax - M))));
    const float wmax = sqrtf(W2max);
    float tb = 0.f;
    for (int k = lane; k < K; k += 32) {
      const float g = a.ws.fwd_coef[(size_t)k * 3 + 1], c = a.ws.fwd_coef[(size_t)k * 3 + 2];
      tb = fmaxf(tb, fabsf(fmaf(2.f * g, u0f, c)) * wmax + fabsf(g) * W2max);
    }
    tb = warp_maxf(tb);
    const int md = tb <= a.thr[0] ? 0 : (tb <= a.thr[1] ? 1 : (tb <= a.thr[2] ? 2 : (tb <= a.thr[3] ? 3 : (tb <= a.thr[4] ? 4 : 5))));
    float* aux = a.ws.colaux + (size_t)i * 2 * K;
    __syncwarp();
#pragma unroll 4
    for (int kc = lane; kc < K; kc += 32) {
      const double lpd = tref[kc] - M - logS;  // this lane's own store above
      const float lp2 = (float)(lpd * kLog2eD);
      aux[kc] = (md == 5 && kLpEpi) ? lp2 : expf((float)lpd);  // P or log2e ln P (see k_colprep_tc)
      uint4 c0, c1;
      extra_col(0.f, (md == 5 && !kLpEpi) ? lp2 : 0.f, c0, c1);
      *reinterpret_cast<uint4*>(cop + G::col_off(kc, G::XKK + 8)) = c1;
    }
    if (lane == 0) {
      a.ws.cvec[i] = M + logS - logK;
      a.ws.gstat[i] = W2max;
      a.ws.gmode[i] = md;
    }
  }
}

// ------------------------------- backward column constants, compact path (K4a, D = 1)
// As k_bwd_cols_tc, one warp per group: L*(k') = log2e log P(k'|k*), the softmax over the group's
// columns of t_ref(k') + B(k*,k') - B(k_ref,k') (fp64), into the extra slab's lP slots.  Three
// passes over the columns (max, sum, write); the re-reads of z / t_ref hit L1.
template <int D>
__global__ void __launch_bounds__(256) k_bwd_cols_warp(TLArgs a) {
  static_assert(TcGeo<D>::COMPACT, "warp-per-group column constants: compact path");
  using G = TcGeo<D>;
  const int K = a.K, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double mus = (double)a.ws.ref->mu_star[0], mur = (double)a.ws.ref->mu_ref[0];
  const double es = a.ws.ref->e_star, bs = a.ws.ref->bstar_const;
  const double er = a.ws.ref->e_ref, br = a.ws.ref->bref_const;
  for (int64_t i = (int64_t)blockIdx.x * nw + wid; i < a.n_local; i += (int64_t)gridDim.x * nw) {
    const float* zi = a.z + (size_t)i * K;
    const double* tr = a.ws.tA + (size_t)i * K;
    auto tcol = [&](int kc) {
      const double z = zi[kc], ds = z - mus, dr = z - mur;
      return (bs - 0.5 * es * ds * ds) - (br - 0.5 * er * dr * dr) + tr[kc];
    };
    double mx = -CUDART_INF;
    for (int kc = lane; kc < K; kc += 32) mx = fmax(mx, tcol(kc));
    mx = warp_max(mx);
    double se = 0.0;
    for (int kc = lane; kc < K; kc += 32) se += (double)expf((float)(tcol(kc) - mx));
    const double lse = mx + log(warp_sum(se));
    unsigned char* cop = reinterpret_cast<unsigned char*>(a.ws.colop) + (size_t)i * K * G::COL;
    for (int kc = lane; kc < K; kc += 32) {
      uint4 x0, x1;
      extra_col(0.f, (float)((tcol(kc) - lse) * kLog2eD), x0, x1);
      *reinterpret_cast<uint4*>(cop + G::col_off(kc, G::XKK + 8)) = x1;
    }
  }
}

// ------------------------------------------------- moments, warp per group (K4c, small D)
// E z = c + S1/S0, Var z = S2/S0 - (S1/S0)^2, S_p = sum_k' w (z - c)^p (fp64, shifted by the Q mean
// c = m_i, self-normalised: R24), one warp per (group, dim).
template <int D>
__global__ void __launch_bounds__(256) k_moments_warp(TLArgs a) {
  const int K = a.K, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t rows = a.n_local * D;
  for (int64_t rr = (int64_t)blockIdx.x * nw + wid; rr < rows; rr += (int64_t)gridDim.x * nw) {
    const int64_t i = rr / D;
    const float* zr = a.z + (size_t)rr * K;
    const float* wi = a.w + (size_t)i * K;
    const double c = a.q_m[rr];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int kc = lane; kc < K; kc += 32) {
      const double w = wi[kc], e = (double)zr[kc] - c, pe = w * e;
      s0 += w;
      s1 += pe;
      s2 = fma(pe, e, s2);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      const double mm = s1 / s0;
      a.m1[rr] = c + mm;
      a.v[rr] = s2 / s0 - mm * mm;
    }
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

// 2^x - 1 by its Taylor polynomial of degree N in x ln 2 (Horner, FMA pipe)
template <int N>
__device__ __forceinline__ float2 expm1_2_poly(float2 x) {
  constexpr double ln2 = 0.69314718055994530942;
  double cN = inv_fact(N);
  for (int i = 0; i < N; ++i) cN *= ln2;
  float2 p = f2((float)cN);
#pragma unroll
  for (int n = N - 1; n >= 1; --n) {
    double c = inv_fact(n);
    for (int i = 0; i < n; ++i) c *= ln2;
    p = fma2(p, x, f2((float)c));
  }
  return mul2(p, x);
}

// Forward epilogue, online mode: (m, s) = running max / sum of 2^(v - m) over
// v = c2.u + g2 U + lP (log2 domain; the row constant is added at the end).
// The max is lazy: s is rescaled only when a chunk raises it.
// QEM_FWD_LAZY: past a row's first column block (`nomax`) the max pass is skipped and the exponentials
// are taken against the running max the earlier blocks left (2^(v - m) may exceed 1; a sum is as
// accurate at any scale); should a chunk come near overflow (or NaN), the warp re-reads its TMEM
// columns and takes the exact pass (warp-uniform: tcgen05.ld is .sync.aligned).
#ifndef QEM_FWD_REDO_COUNT
#define QEM_FWD_REDO_COUNT 0  // 1: count the epilogue warps that redid a chunk in mode-hist slot 7 (costs 1 %)
#endif
#ifndef QEM_FWD_LAZY
#define QEM_FWD_LAZY 1  // config 5 forward 2.66 -> 2.60 ms (interleaved A/B); fallbacks: 0.6 % of chunks at t = 1, 0 from t = 3
#endif
__device__ __forceinline__ void fwd_epi_online(uint32_t taddr, const float* lpp, float& m, float& s, bool nomax,
                                               float redo_thr, bool& redo) {
  for (;;) {
    uint32_t r[4][16];
    tmem_ld64(taddr, r);  // the thread's 64 columns of this tile, one TMEM round trip
    // + log2e ln P of the columns (SMEM broadcast: every lane of the warp reads the same columns), in
    // fp32 round to nearest (QEM_LP_EPI; else the MMA added it)
#pragma unroll
    for (int q = 0; q < 4 && kLpEpi; ++q)
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 l = reinterpret_cast<const float4*>(lpp + q * 16)[c4];
        r[q][4 * c4] = __float_as_uint(__uint_as_float(r[q][4 * c4]) + l.x);
        r[q][4 * c4 + 1] = __float_as_uint(__uint_as_float(r[q][4 * c4 + 1]) + l.y);
        r[q][4 * c4 + 2] = __float_as_uint(__uint_as_float(r[q][4 * c4 + 2]) + l.z);
        r[q][4 * c4 + 3] = __float_as_uint(__uint_as_float(r[q][4 * c4 + 3]) + l.w);
      }
    if (!QEM_FWD_LAZY || !nomax) {
      // four independent FMNMX3 chains (one per 16-column load), then combined: a dependency chain
      // of 8 + 2 instead of 32
      float mq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        mq[q] = fmaxf(__uint_as_float(r[q][0]), __uint_as_float(r[q][1]));
#pragma unroll
        for (int c = 2; c < 16; c += 2) mq[q] = fmax3f(mq[q], __uint_as_float(r[q][c]), __uint_as_float(r[q][c + 1]));
      }
      const float mx = fmax3f(m, fmax3f(mq[0], mq[1], mq[2]), mq[3]);
      if (mx > m) {  // exact running max (see kLazy in qem_forward.cuh)
        s *= ex2(m - mx);
        m = mx;
      }
    }
    const float2 nm = f2(-m);
    float2 acc[4] = {f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        float2 e = add2(make_float2(__uint_as_float(r[q][c]), __uint_as_float(r[q][c + 1])), nm);
        if (QEM_FWD_LAZY && c >= 16 - kPolyExpFwd)  // the software exponent add would wrap past 2^128
          e = make_float2(fminf(e.x, 128.f), fminf(e.y, 128.f));
        const float2 x = c >= 16 - kPolyExpFwd ? exp2_poly2(e) : make_float2(ex2(e.x), ex2(e.y));
        acc[q] = add2(acc[q], x);
      }
    const float2 t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
    const float sn = s + (t.x + t.y);
    if (!QEM_FWD_LAZY || !nomax || !__any_sync(0xffffffffu, !(sn <= redo_thr))) {
      s = sn;
      return;
    }
    nomax = false;  // near overflow / NaN (the aux merge adds 4 slices' sums): the exact pass
    redo = true;  // QEM_FWD_REDO_COUNT builds count it per epilogue warp at the end of the kernel
  }
}

// Forward epilogue, polynomial mode: acc += sum P (2^v - 1), v = log2e D' = c2.w + g2 S.
template <int N, int NC16>
__device__ __forceinline__ void fwd_epi_poly(uint32_t taddr, const float* pp, float& acc) {
  float2 a2[2] = {f2(0.f), f2(0.f)};
  tmem_pipeline16<NC16>(taddr, [&](int c16, uint32_t(&r)[16]) {
    float p[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = reinterpret_cast<const float4*>(pp + c16 * 16)[q];
      p[4 * q] = v.x;
      p[4 * q + 1] = v.y;
      p[4 * q + 2] = v.z;
      p[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const float2 dp = make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1]));
      a2[(c >> 1) & 1] = fma2(make_float2(p[c], p[c + 1]), expm1_2_poly<N>(dp), a2[(c >> 1) & 1]);
    }
  });
  const float2 t = add2(a2[0], a2[1]);
  acc += t.x + t.y;
}

// The polynomial modes' epilogues (out of line was measured 3 % slower on the online mode too)
__device__ __forceinline__ void fwd_epi_poly_any(int md, uint32_t taddr, const float* pp, float& acc) {
  switch (md) {
    case 0: fwd_epi_poly<3, 4>(taddr, pp, acc); break;
    case 1: fwd_epi_poly<4, 4>(taddr, pp, acc); break;
    case 2: fwd_epi_poly<5, 4>(taddr, pp, acc); break;
    case 3: fwd_epi_poly<7, 4>(taddr, pp, acc); break;
    default: fwd_epi_poly<9, 4>(taddr, pp, acc); break;
  }
}

// Tile walk of a persistent CTA (no integer division in the loop): group j (instance i =
// blockIdx.x + j gridDim.x), outer block cb, inner block rb; T = tile count, J = (group, outer block) count.
struct TileWalk {
  int64_t T, J, j, i;
  int t, cb, rb, nin, nout;
  __device__ TileWalk(int n_in, int n_out)
      : T(0), J(0), j(0), i(blockIdx.x), t(0), cb(0), rb(0), nin(n_in), nout(n_out) {}
  __device__ __forceinline__ void next() {
    ++T;
    ++t;
    if (++rb == nin) {
      rb = 0;
      ++J;
      if (++cb == nout) {
        cb = 0;
        t = 0;
        ++j;
        i += gridDim.x;
      }
    }
  }
};

// ------------------------------------------------------------------ forward
#ifndef QEM_FWD_SA
#define QEM_FWD_SA 3
#endif
#ifndef QEM_FWD_FS
#define QEM_FWD_FS 8
#endif
template <int D>
struct FwdTcL {
  static constexpr int SA = QEM_FWD_SA;                              // row-block stages
  static constexpr uint32_t A_C = 128 * TcGeo<D>::CB;                // 12 KB (split) / 4 KB (compact)
  static constexpr uint32_t A_STAGE = A_C + 128 * kTcRowXBytes;      // 16 KB / 8 KB
  static constexpr uint32_t B_STAGE = 256 * TcGeo<D>::COL;           // 32 KB / 16 KB
  static constexpr uint32_t P_STAGE = 256 * 4;                       // P of the block's columns
  static constexpr size_t a() { return 0; }
  static constexpr size_t b() { return a() + SA * A_STAGE; }
  static constexpr size_t p() { return b() + 2 * B_STAGE; }
  static constexpr int FS = QEM_FWD_FS;                               // row-block hand-over stages
  static constexpr size_t fin() { return p() + 2 * P_STAGE; }         // [FS][4][128] float2
  static constexpr size_t bars() { return fin() + FS * 4 * 128 * 8; }  // 2*SA + 8 + 2*FS mbarriers
  static constexpr int NBARS = 2 * SA + 8 + 2 * FS;
  static size_t __host__ __device__ st0(int) { return bars() + NBARS * 8; }
  static size_t __host__ __device__ st1(int K) { return st0(K) + (size_t)4 * K * 4; }
  static size_t __host__ __device__ g(int K) { return st1(K) + (size_t)4 * K * 4; }
  static size_t __host__ __device__ bytes(int K) { return g(K) + (size_t)K * 8; }
};

constexpr int kFwdAuxWarps = 2;  // row finalisers of the forward
constexpr int kFwdThreads = kTcThreads + 32 * kFwdAuxWarps;

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1) k_forward_tc(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  using L = FwdTcL<D>;
  using G = TcGeo<D>;
  constexpr int SA = L::SA;
  const int K = a.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = K / 256, RB = K / 128, TPG = NB * RB;
  unsigned char* s_a = smem + L::a();
  unsigned char* s_b = smem + L::b();
  float* s_p = reinterpret_cast<float*>(smem + L::p());
  float2* s_fin = reinterpret_cast<float2*>(smem + L::fin());
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars());
  uint64_t* a_full = bars;           // [SA]
  uint64_t* a_empty = bars + SA;     // [SA]
  uint64_t* b_full = bars + 2 * SA;  // [2]
  uint64_t* b_empty = b_full + 2;    // [2]  MMA commit + 16 epilogue warps
  uint64_t* t_full = b_empty + 2;    // [2]
  uint64_t* t_empty = t_full + 2;    // [2]  16 epilogue warps
  uint64_t* f_full = t_empty + 2;    // [FS] 16 epilogue warps: a row block's slice states are in s_fin
  uint64_t* f_empty = f_full + L::FS;  // [FS] aux warps: s_fin stage merged
  float* s_st0 = reinterpret_cast<float*>(smem + L::st0(K));
  float* s_st1 = reinterpret_cast<float*>(smem + L::st1(K));
  double* s_g = reinterpret_cast<double*>(smem + L::g(K));
  __shared__ uint32_t s_tmem;

  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t ntiles = ngroups * TPG;

  if (tid == 0) {
    for (int b = 0; b < SA; ++b) {
      mbar_init(&a_full[b], 1);
      mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&b_full[b], 1);
      mbar_init(&b_empty[b], 1 + kTcEpiWarps);
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], kTcEpiWarps);
    }
    for (int b = 0; b < L::FS; ++b) {
      mbar_init(&f_full[b], kTcEpiWarps);
      mbar_init(&f_empty[b], kFwdAuxWarps);
    }
    fence_mbar_init();
  }
  if (warp == kTcEpiWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int k = tid; k < K; k += blockDim.x) s_g[k] = 0.0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  double csum = 0.0;

  if (warp == kTcEpiWarps) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const unsigned char* colop = reinterpret_cast<const unsigned char*>(a.ws.colop);
      const unsigned char* rowc = reinterpret_cast<const unsigned char*>(a.ws.rowop);
      const unsigned char* rowx = reinterpret_cast<const unsigned char*>(a.ws.rowop_x);
      for (TileWalk tw(RB, NB); tw.T < ntiles; tw.next()) {
        const int64_t T = tw.T, j = tw.j;
        const int t = tw.t, cb = tw.cb, rb = tw.rb;
        const int64_t i = tw.i;
        if (rb == 0) {
          const int64_t J = tw.J;
          const int st = (int)(J & 1);
          if (J >= 2) mbar_wait(&b_empty[st], (uint32_t)(((J >> 1) - 1) & 1));
          mbar_expect_tx(&b_full[st], L::B_STAGE + L::P_STAGE);
          tma_bulk_g2s(s_b + st * L::B_STAGE, colop + ((size_t)i * K + (size_t)cb * 256) * G::COL, L::B_STAGE,
                       &b_full[st]);
          tma_bulk_g2s(s_p + st * 256, a.ws.colaux + (size_t)i * 2 * K + (size_t)cb * 256, L::P_STAGE, &b_full[st]);
        }
        const int sa = (int)(T % SA);
        const int64_t ua = T / SA;
        if (ua >= 1) mbar_wait(&a_empty[sa], (uint32_t)((ua - 1) & 1));
        mbar_expect_tx(&a_full[sa], L::A_STAGE);
        tma_bulk_g2s(s_a + sa * L::A_STAGE, rowc + (size_t)rb * L::A_C, L::A_C, &a_full[sa]);
        tma_bulk_g2s(s_a + sa * L::A_STAGE + L::A_C, rowx + (size_t)rb * 128 * kTcRowXBytes, 128 * kTcRowXBytes,
                     &a_full[sa]);
      }
    }
  } else if (warp == kTcEpiWarps + 1) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(128, 256);
      for (TileWalk tw(RB, NB); tw.T < ntiles; tw.next()) {
        const int64_t T = tw.T, j = tw.j;
        const int t = tw.t, cb = tw.cb, rb = tw.rb;
        const int64_t J = tw.J;
        const int sa = (int)(T % SA), tb = (int)(T & 1);
        mbar_wait(&a_full[sa], (uint32_t)((T / SA) & 1));
        if (rb == 0) mbar_wait(&b_full[J & 1], (uint32_t)((J >> 1) & 1));
        if (T >= 2) mbar_wait(&t_empty[tb], (uint32_t)(((T >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t A = smem_u32(s_a + sa * L::A_STAGE), B = smem_u32(s_b + (J & 1) * L::B_STAGE);
        umma_tile<D>(tmem + (uint32_t)tb * 256, A, 8 * G::CB, B, 8 * G::COL, A + L::A_C, 256, B + 8 * G::CB,
                     8 * G::COL, idesc);
        umma_commit(&t_full[tb]);
        umma_commit(&a_empty[sa]);
        if (rb == RB - 1) umma_commit(&b_empty[J & 1]);
      }
    }
  } else if (warp >= kTcEpiWarps + 2) {
    // ------------------------------------------- aux: merge the 4 column slices of each row, finalise
    // h, dg = alpha' + h and the plate sum (one row block of 128 rows at a time, behind the epilogue)
    const int atid = tid - kTcThreads;
    constexpr int NTA = 32 * kFwdAuxWarps;
    int md = 5;
    double mi[D];  // u0_i = m_i - mu_ref of the group, formed once per group (not per row)
    double M2 = 0.0;
    int64_t j = 0, i = blockIdx.x;
    int rb = 0;
    for (int64_t u = 0; u < ngroups * RB; ++u) {
      if (rb == 0) {
        md = a.ws.gmode[i];
        M2 = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) {  // u0_i = m_i - mu_ref, exact in fp64
          mi[r] = (double)a.q_m[i * D + r] - (double)a.ws.ref->mu_ref[r];
          M2 = fma(mi[r], mi[r], M2);
        }
        if (atid == 0) {
          atomicAdd(&a.cnt->mode_hist[md], 1ull);
          csum += a.ws.cvec[i];
        }
      }
      const int st = (int)(u % L::FS);
      mbar_wait(&f_full[st], (uint32_t)((u / L::FS) & 1));
      const float2* fin = s_fin + st * 512;
      for (int rr = atid; rr < 128; rr += NTA) {
        const int k = rb * 128 + rr;
        double h;
        if (md == 5) {
          float mx = -CUDART_INF_F;
#pragma unroll
          for (int c = 0; c < 4; ++c) mx = fmaxf(mx, fin[c * 128 + rr].x);
          float sm = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 f = fin[c * 128 + rr];
            sm += f.y * ex2(f.x - mx);
          }
          // log2 -> natural units in fp64: the fp32 ln 2 (relative error 2.8e-9) times an h of tens
          // would be a bias of ~1e-7 per group on every row but k_ref (whose h is 0), coherent over the
          // plate sum (1e-4 in the root log-weights at 1000 groups)
          h = ((double)mx + log2((double)sm)) * kLn2D;  // fp64 log: log2f's ~1-ulp error is not zero-mean
        } else {
          float sm = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) sm += fin[c * 128 + rr].x;
          h = log1p((double)sm);
        }
        // alpha'_ik = D_k(m_i) = alpha_k + gamma_k |u0_i|^2 + c_k . u0_i in fp64 (u = z - mu_ref rows)
        const double* cd = a.ws.coef_d + (size_t)k * (D + 1);  // (gamma, c[D]) as fp64: no conversions
        double ap = fma(cd[0], M2, a.ws.alpha_d[k]);
#pragma unroll
        for (int r = 0; r < D; ++r) ap = fma(cd[1 + r], mi[r], ap);
        const double dgd = ap + h;
        a.ws.hmsg[(size_t)i * K + k] = (float)h;  // re-centred message, the backward's row constant
        a.ws.dg[(size_t)i * K + k] = (float)dgd;
        s_g[k] += dgd;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&f_empty[st]);
      if (++rb == RB) {
        rb = 0;
        ++j;
        i += gridDim.x;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3, cq = warp >> 2;
    int md = 5;
    bool redo = false;  // some chunk of this warp took the exact redo (R41)
    int64_t u = 0;  // finalised row blocks so far
    for (TileWalk tw(RB, NB); tw.T < ntiles; tw.next()) {
      const int64_t T = tw.T, J = tw.J;
      const int t = tw.t, cb = tw.cb, rb = tw.rb;
      const int64_t i = tw.i;
      if (t == 0) md = a.ws.gmode[i];
      const int k = rb * 128 + q * 32 + lane;
      float st0, st1 = 0.f;
      if (cb == 0)
        st0 = md == 5 ? -CUDART_INF_F : 0.f;
      else {
        st0 = s_st0[cq * K + k];
        st1 = s_st1[cq * K + k];
      }
      mbar_wait(&t_full[T & 1], (uint32_t)((T >> 1) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem + (uint32_t)(T & 1) * 256 + (uint32_t)(cq * 64) + ((uint32_t)(q * 32) << 16);
      const float* pp = s_p + (J & 1) * 256 + cq * 64;
      if (md != 5 || kLpEpi) mbar_wait(&b_full[J & 1], (uint32_t)((J >> 1) & 1));  // P / lP of this block in SMEM
      if (md == 5) {
        fwd_epi_online(taddr, pp, st0, st1, cb > 0, a.redo_thr, redo);
      } else {
        fwd_epi_poly_any(md, taddr, pp, st0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&t_empty[T & 1]);
        if (rb == RB - 1) mbar_arrive(&b_empty[J & 1]);
      }
      if (cb < NB - 1) {
        s_st0[cq * K + k] = st0;
        s_st1[cq * K + k] = st1;
      } else {
        // ---- row k complete in this slice: hand (max, sum) to the aux warps
        const int fs = (int)(u % L::FS);
        if (u >= L::FS) mbar_wait(&f_empty[fs], (uint32_t)(((u / L::FS) - 1) & 1));
        s_fin[fs * 512 + cq * 128 + q * 32 + lane] = make_float2(st0, st1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_full[fs]);
        ++u;
      }
    }
    if (QEM_FWD_REDO_COUNT && redo && lane == 0) atomicAdd(&a.cnt->mode_hist[7], 1ull);
  }

  // ---- teardown, per-CTA partial plate sums, last-CTA fixed-order reduce
  tc_fence_before();
  __syncthreads();
  if (warp == kTcEpiWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  // the CTA's plate sums (fixed order within the CTA: its static group stride) go to the (K + 1) x
  // {h, m} accumulators k_root_prep zeroed, split on fixed grids (Fx2, R39) so that the
  // atomics' order cannot change a bit; no CTA walks the 148 CTAs' partials at the end
  double* acc_h = a.ws.partial;
  double* acc_m = a.ws.partial + (K + 1);
  for (int k = tid; k < K; k += blockDim.x) {
    Fx2 f;
    f.add(s_g[k]);
    atomicAdd(&acc_h[k], f.h);
    atomicAdd(&acc_m[k], f.m);
  }
  if (tid == kTcThreads) {  // the first aux thread accumulated sum_i c_i
    Fx2 f;
    f.add(csum);
    atomicAdd(&acc_h[K], f.h);
    atomicAdd(&acc_m[K], f.m);
  }
  __threadfence();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) s_last = (atomicAdd(&a.cnt->ticket_fwd, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int k = tid; k <= K; k += blockDim.x) a.ws.red[k] = __ldcg(acc_h + k) + __ldcg(acc_m + k);
    if (tid == 0) a.cnt->ticket_fwd = 0;
  }
}

// ----------------------------------------------------------------- backward
constexpr int kBwdAuxWarps = 2;  // per-group row-slab builders of the backward

template <int D>
struct BwdTcL {
  static constexpr int SB = 3;                                  // row-block stages
  static constexpr uint32_t A_STAGE = 128 * TcGeo<D>::COL;      // 16 KB / 8 KB: 128 columns
  static constexpr uint32_t B_STAGE = 256 * TcGeo<D>::CB;       // 24 KB / 8 KB: 256 rows of Eb (k*-differenced)
  static constexpr size_t a() { return 0; }
  static constexpr size_t b() { return a() + 2 * A_STAGE; }
  static constexpr size_t wp() { return b() + SB * B_STAGE; }            // [2][4][128] float
  static constexpr size_t bars() { return wp() + 2 * 4 * 128 * 4; }      // 24 mbarriers (20 used)
  static size_t __host__ __device__ bx(int) { return (bars() + 24 * 8 + 1023) & ~(size_t)1023; }
  static size_t __host__ __device__ bytes(int K) { return bx(K) + (size_t)2 * K * kTcRowXBytes; }
};
constexpr int kBwdThreads = kTcThreads + 32 * kBwdAuxWarps;

// ------------------------------------------------- backward column constants (K4a)
// Backward reference:
//   log P(k'|k) = log P(k'|k*) + E_k(k') - (l_k - l_*),  E_k = B(k,.) - B(k*,.).
// Per group: the column constants L*(k') = log2e log P(k'|k*), a softmax over the group's
// columns of the fp64 logits t_ref(k') + B(k*,k') - B(k_ref,k'), into colaux's second slot
// (the forward's ln P is not needed any more).  One CTA per SM, persistent over groups;
// each group's z (16 x K fp32, contiguous) and t_ref (K fp64) arrive in SMEM by one
// cp.async.bulk each into a 2-stage ring, so HBM streams while the previous group computes.
struct GroupStage {  // shared by k_bwd_cols_tc and k_moments_tc (z of D dims + t_ref or w)
  static constexpr int THREADS = 256;
  __host__ __device__ static size_t z_bytes(int K, int D) { return (size_t)D * K * 4; }
  __host__ __device__ static size_t stage(int K, int D) { return z_bytes(K, D) + (size_t)K * 8; }
  __host__ __device__ static size_t bytes(int K, int D) { return 2 * stage(K, D) + 64 * 8 + 4 * 8; }
};

__device__ __forceinline__ double block_max256(double v, double* scr) {
  v = warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scr[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = scr[0];
#pragma unroll
  for (int w = 1; w < GroupStage::THREADS / 32; ++w) m = fmax(m, scr[w]);
  return m;
}
__device__ __forceinline__ double block_sum256(double v, double* scr) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scr[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = 0.0;
#pragma unroll
  for (int w = 0; w < GroupStage::THREADS / 32; ++w) m += scr[w];
  return m;
}

template <int D>
__global__ void __launch_bounds__(GroupStage::THREADS, 1) k_bwd_cols_tc(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int K = a.K, tid = threadIdx.x;
  const size_t SZ = GroupStage::stage(K, D);
  double* scr = reinterpret_cast<double*>(smem + 2 * SZ);
  uint64_t* full = reinterpret_cast<uint64_t*>(scr + 64);
  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t zb = (uint32_t)GroupStage::z_bytes(K, D), tb = (uint32_t)K * 8;
  auto issue = [&](int64_t j) {
    const int64_t i = blockIdx.x + j * gridDim.x;
    unsigned char* st = smem + (size_t)(j & 1) * SZ;
    mbar_expect_tx(&full[j & 1], zb + tb);
    tma_bulk_g2s(st, a.z + (size_t)i * D * K, zb, &full[j & 1]);
    tma_bulk_g2s(st + zb, a.ws.tA + (size_t)i * K, tb, &full[j & 1]);
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t j = 0; j < 2 && j < ngroups; ++j) issue(j);
  float mus[D], mur[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    mus[r] = a.ws.ref->mu_star[r];
    mur[r] = a.ws.ref->mu_ref[r];
  }
  const double es = a.ws.ref->e_star, bs = a.ws.ref->bstar_const;
  const double er = a.ws.ref->e_ref, br = a.ws.ref->bref_const;
  const int c4 = tid * 4;
  const bool act = c4 < K;
  for (int64_t j = 0; j < ngroups; ++j) {
    const int64_t i = blockIdx.x + j * gridDim.x;
    const unsigned char* st = smem + (size_t)(j & 1) * SZ;
    mbar_wait(&full[j & 1], (uint32_t)((j >> 1) & 1));
    double t[4] = {-CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF};
    double mx = -CUDART_INF;
    if (act) {
      const float* zs = reinterpret_cast<const float*>(st);
      double d[4] = {0.0, 0.0, 0.0, 0.0}, g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const float4 zv = *reinterpret_cast<const float4*>(zs + (size_t)r * K + c4);
        const double zz[4] = {(double)zv.x, (double)zv.y, (double)zv.z, (double)zv.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double ds = zz[c] - (double)mus[r], dr = zz[c] - (double)mur[r];
          d[c] = fma(ds, ds, d[c]);
          g[c] = fma(dr, dr, g[c]);
        }
      }
      const double* tr = reinterpret_cast<const double*>(st + zb);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        t[c] = (bs - 0.5 * es * d[c]) - (br - 0.5 * er * g[c]) + tr[c4 + c];
        mx = fmax(mx, t[c]);
      }
    }
    mx = block_max256(mx, scr);
    double se = 0.0;
    if (act) {
#pragma unroll
      for (int c = 0; c < 4; ++c) se += (double)expf((float)(t[c] - mx));
    }
    const double lse = mx + log(block_sum256(se, scr + 8));
    __syncthreads();  // every thread is done with this stage
    if (tid == 0 && j + 2 < ngroups) issue(j + 2);
    if (act) {
      // L*(k') into the lP slots of the column operand's extra slab (the forward's ln P is no longer
      // needed): the backward's MMA adds it to every tile element (row slab lP switch on), so the
      // epilogue does not
      unsigned char* cop = reinterpret_cast<unsigned char*>(a.ws.colop) + (size_t)i * K * kTcColBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 x0, x1;
        extra_col(0.f, (float)((t[c] - lse) * kLog2eD), x0, x1);
        *reinterpret_cast<uint4*>(cop + tc_col_offset(c4 + c, 56)) = x1;  // chunk 7: 1 L*0 L*1 L*2 0...
      }
    }
  }
}

// ------------------------------------------------------------ moments (K4c)
// After the backward: E z = c + S1/S0, Var z = S2/S0 - (S1/S0)^2, S_p = sum_k' w (z - c)^p in
// fp64 (self-normalised, shifted by the Q mean c = m_i; R24).  One CTA per SM over groups,
// z and w of a group staged by cp.async.bulk (2-stage ring); warp q handles dims 2q, 2q+1.
template <int D>
__global__ void __launch_bounds__(GroupStage::THREADS, 1) k_moments_tc(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int K = a.K, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t SZ = GroupStage::stage(K, D);
  double* scr = reinterpret_cast<double*>(smem + 2 * SZ);
  uint64_t* full = reinterpret_cast<uint64_t*>(scr + 64);
  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t zb = (uint32_t)GroupStage::z_bytes(K, D), wb = (uint32_t)K * 4;
  auto issue = [&](int64_t j) {
    const int64_t i = blockIdx.x + j * gridDim.x;
    unsigned char* st = smem + (size_t)(j & 1) * SZ;
    mbar_expect_tx(&full[j & 1], zb + wb);
    tma_bulk_g2s(st, a.z + (size_t)i * D * K, zb, &full[j & 1]);
    tma_bulk_g2s(st + zb, a.w + (size_t)i * K, wb, &full[j & 1]);
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t j = 0; j < 2 && j < ngroups; ++j) issue(j);
  for (int64_t j = 0; j < ngroups; ++j) {
    const int64_t i = blockIdx.x + j * gridDim.x;
    const unsigned char* st = smem + (size_t)(j & 1) * SZ;
    mbar_wait(&full[j & 1], (uint32_t)((j >> 1) & 1));
    const float* zs = reinterpret_cast<const float*>(st);
    const float* ws = reinterpret_cast<const float*>(st + zb);
    const int r0 = 2 * warp;  // 8 warps x 2 dims (dims >= D: the warp idles)
    const int r1 = r0 + 1 < D ? r0 + 1 : r0;
    const bool act = r0 < D;
    const double c0 = act ? a.q_m[i * D + r0] : 0.0, c1 = act ? a.q_m[i * D + r1] : 0.0;
    double s0 = 0.0, a1 = 0.0, a2 = 0.0, b1 = 0.0, b2 = 0.0;
    for (int c4 = lane * 4; act && c4 < K; c4 += 128) {
      const float4 wv = *reinterpret_cast<const float4*>(ws + c4);
      const float4 za = *reinterpret_cast<const float4*>(zs + (size_t)r0 * K + c4);
      const float4 zb4 = *reinterpret_cast<const float4*>(zs + (size_t)r1 * K + c4);
      const double w4[4] = {wv.x, wv.y, wv.z, wv.w};
      const double e4[4] = {za.x - c0, za.y - c0, za.z - c0, za.w - c0};
      const double f4[4] = {zb4.x - c1, zb4.y - c1, zb4.z - c1, zb4.w - c1};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        s0 += w4[c];
        const double pe = w4[c] * e4[c], pf = w4[c] * f4[c];
        a1 += pe;
        a2 = fma(pe, e4[c], a2);
        b1 += pf;
        b2 = fma(pf, f4[c], b2);
      }
    }
    s0 = warp_sum(s0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    b1 = warp_sum(b1);
    b2 = warp_sum(b2);
    if (lane == 0 && act) {
      const double ma = a1 / s0, mb = b1 / s0;
      a.m1[i * D + r0] = c0 + ma;
      a.v[i * D + r0] = a2 / s0 - ma * ma;
      if (r1 != r0) {
        a.m1[i * D + r1] = c1 + mb;
        a.v[i * D + r1] = b2 / s0 - mb * mb;
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0 && j + 2 < ngroups) issue(j + 2);
  }
}

// Backward row extra slab of group i (K x 32 B) into `bx`, built by the aux warps two groups
// ahead: [Eg pattern | 0 0 0 | rho], rho_k = log2 w_root(k) - log2e (h_k - h_*) (h = the
// forward's re-centred message; -1e30 where w_root = 0).
__device__ __forceinline__ void bwd_bx(const TLArgs& a, int64_t i, unsigned char* bx, int atid) {
  constexpr int NT = 32;  // one aux warp builds the slabs
  const int K = a.K;
  const float hs = a.ws.hmsg[(size_t)i * K + a.ws.ref->k_star];
#pragma unroll 2
  for (int k4 = atid * 4; k4 < K; k4 += NT * 4) {
    const float4 wr = *reinterpret_cast<const float4*>(a.w_root + k4);
    const float4 hm = *reinterpret_cast<const float4*>(a.ws.hmsg + (size_t)i * K + k4);
    const float4 bg = *reinterpret_cast<const float4*>(a.ws.bgam + k4);
    const float w4[4] = {wr.x, wr.y, wr.z, wr.w}, h4[4] = {hm.x, hm.y, hm.z, hm.w}, g4[4] = {bg.x, bg.y, bg.z, bg.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float rho = w4[c] > 0.f ? log2f(w4[c]) - (h4[c] - hs) * kLog2e : -1e30f;
      uint4 c0, c1;
      extra_row(g4[c], 1.f, rho, c0, c1);  // lP switch on: the column slab holds L* (k_bwd_cols_tc)
      *reinterpret_cast<uint4*>(bx + tc_rowx_offset(k4 + c, 0)) = c0;
      *reinterpret_cast<uint4*>(bx + tc_rowx_offset(k4 + c, 8)) = c1;
    }
  }
  fence_proxy_async();  // generic-proxy SMEM writes -> visible to the tensor core (async proxy)
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1) k_backward_tc(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  using L = BwdTcL<D>;
  using G = TcGeo<D>;
  constexpr int SB = L::SB;
  const int K = a.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int CB = K / 128, RB = K / 256, TPG = CB * RB;
  unsigned char* s_a = smem + L::a();
  unsigned char* s_b = smem + L::b();
  float* s_wp = reinterpret_cast<float*>(smem + L::wp());
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars());
  uint64_t* a_full = bars;            // [2]
  uint64_t* a_empty = bars + 2;       // [2]
  uint64_t* b_full = bars + 4;        // [SB]
  uint64_t* b_empty = b_full + SB;    // [SB]
  uint64_t* t_full = b_empty + SB;    // [2]
  uint64_t* t_empty = t_full + 2;     // [2]  16 epilogue warps
  uint64_t* bx_full = t_empty + 2;    // [2]  aux warps: row extra slab of a group ready (MMA waits)
  uint64_t* g_done = bx_full + 2;     // [2]  16 epilogue warps: group finished (its slab stage is free)
  uint64_t* wp_full = g_done + 2;     // [2]  16 epilogue warps: a column block's 4 slice sums are in s_wp
  uint64_t* wp_empty = wp_full + 2;   // [2]  merger warp: s_wp stage merged
  unsigned char* s_bx = smem + L::bx(K);
  __shared__ uint32_t s_tmem;

  const int64_t n = a.n_local;
  const int64_t ngroups = n > blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t ntiles = ngroups * TPG;

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], 1);
      mbar_init(&a_empty[b], 1);
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], kTcEpiWarps);
      mbar_init(&bx_full[b], 1);  // the slab-builder warp
      mbar_init(&g_done[b], kTcEpiWarps);
      mbar_init(&wp_full[b], kTcEpiWarps);
      mbar_init(&wp_empty[b], 1);
    }
    for (int b = 0; b < SB; ++b) {
      mbar_init(&b_full[b], 1);
      mbar_init(&b_empty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == kTcEpiWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == kTcEpiWarps) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const unsigned char* colop = reinterpret_cast<const unsigned char*>(a.ws.colop);
      const unsigned char* rowc = reinterpret_cast<const unsigned char*>(a.ws.rowop_b);
      for (TileWalk tw(RB, CB); tw.T < ntiles; tw.next()) {
        const int64_t T = tw.T;
        const int cb = tw.cb, rb = tw.rb;
        const int64_t i = tw.i;
        if (rb == 0) {
          const int64_t J = tw.J;
          const int st = (int)(J & 1);
          if (J >= 2) mbar_wait(&a_empty[st], (uint32_t)(((J >> 1) - 1) & 1));
          mbar_expect_tx(&a_full[st], L::A_STAGE);
          tma_bulk_g2s(s_a + st * L::A_STAGE, colop + ((size_t)i * K + (size_t)cb * 128) * G::COL, L::A_STAGE,
                       &a_full[st]);
        }
        const int sb = (int)(T % SB);
        const int64_t ub = T / SB;
        if (ub >= 1) mbar_wait(&b_empty[sb], (uint32_t)((ub - 1) & 1));
        mbar_expect_tx(&b_full[sb], L::B_STAGE);
        tma_bulk_g2s(s_b + sb * L::B_STAGE, rowc + (size_t)rb * L::B_STAGE, L::B_STAGE, &b_full[sb]);
      }
    }
  } else if (warp == kTcEpiWarps + 1) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(128, 256);
      for (TileWalk tw(RB, CB); tw.T < ntiles; tw.next()) {
        const int64_t T = tw.T, j = tw.j, J = tw.J;
        const int t = tw.t, rb = tw.rb;
        const int sb = (int)(T % SB), tb = (int)(T & 1);
        if (t == 0) mbar_wait(&bx_full[j & 1], (uint32_t)((j >> 1) & 1));
        if (rb == 0) mbar_wait(&a_full[J & 1], (uint32_t)((J >> 1) & 1));
        mbar_wait(&b_full[sb], (uint32_t)((T / SB) & 1));
        if (T >= 2) mbar_wait(&t_empty[tb], (uint32_t)(((T >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t A = smem_u32(s_a + (J & 1) * L::A_STAGE), B = smem_u32(s_b + sb * L::B_STAGE);
        const uint32_t BX = smem_u32(s_bx + (size_t)(j & 1) * K * kTcRowXBytes + (size_t)rb * 256 * kTcRowXBytes);
        umma_tile<D>(tmem + (uint32_t)tb * 256, A, 8 * G::COL, B, 8 * G::CB, A + 8 * G::CB, 8 * G::COL, BX, 256,
                     idesc);
        umma_commit(&t_full[tb]);
        umma_commit(&b_empty[sb]);
        if (rb == RB - 1) umma_commit(&a_empty[J & 1]);
      }
    }
  } else if (warp == kTcEpiWarps + 2) {
    // ------------------------------- aux 1: row extra slabs two groups ahead of the MMAs
    const int atid = lane;
    for (int64_t jj = 0; jj < 2 && jj < ngroups; ++jj) {
      bwd_bx(a, blockIdx.x + jj * gridDim.x, s_bx + (size_t)jj * K * kTcRowXBytes, atid);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bx_full[jj]);
    }
    for (int64_t j = 0; j + 2 < ngroups; ++j) {
      const int st = (int)(j & 1);
      mbar_wait(&g_done[st], (uint32_t)((j >> 1) & 1));  // group j's MMAs all complete: its stage is free
      bwd_bx(a, blockIdx.x + (j + 2) * gridDim.x, s_bx + (size_t)st * K * kTcRowXBytes, atid);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bx_full[st]);
    }
  } else if (warp == kTcEpiWarps + 3) {
    // ------------------------------- aux 2: merge the 4 row-slice sums of each column block -> w
    int64_t i = blockIdx.x;
    int cb = 0;
    for (int64_t u = 0; u < ngroups * CB; ++u) {
      const int st = (int)(u & 1);
      mbar_wait(&wp_full[st], (uint32_t)((u >> 1) & 1));
      const float* wpb = s_wp + st * 512;
#pragma unroll
      for (int c = lane; c < 128; c += 32) {
        const float wv = wpb[c] + wpb[128 + c] + wpb[256 + c] + wpb[384 + c];
        a.w[(size_t)i * K + cb * 128 + c] = wv;
        if (isnan(wv)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&wp_empty[st]);
      if (++cb == CB) {
        cb = 0;
        i += gridDim.x;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3, cq = warp >> 2;
    float acc = 0.f;
    for (TileWalk tw(RB, CB); tw.T < ntiles; tw.next()) {
      const int64_t T = tw.T, j = tw.j;
      const int t = tw.t, cb = tw.cb, rb = tw.rb;
      if (rb == 0) acc = 0.f;
      mbar_wait(&t_full[T & 1], (uint32_t)((T >> 1) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem + (uint32_t)(T & 1) * 256 + (uint32_t)(cq * 64) + ((uint32_t)(q * 32) << 16);
      float2 wp[2] = {f2(0.f), f2(0.f)};
      // 16-column chunks with the next chunk's TMEM load in flight (measured faster here than one
      // 64-column load: the SFU work of a chunk overlaps the next load)
      tmem_pipeline16<4>(taddr, [&](int, uint32_t(&r)[16]) {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          // v = rho_k + E_k(k') + L*(k') in log2 units, all from the MMA (extra slab)
          const float2 x = make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1]));
          const float2 e = c >= 16 - kPolyExpBwd ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          wp[(c >> 1) & 1] = add2(wp[(c >> 1) & 1], e);
        }
      });
      wp[0] = add2(wp[0], wp[1]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&t_empty[T & 1]);
        if (t == TPG - 1) mbar_arrive(&g_done[j & 1]);
      }
      acc += wp[0].x + wp[0].y;
      if (rb == RB - 1) {
        // hand the column block's slice sum to the merger warp (no epilogue barrier)
        const int64_t u = tw.J;
        const int st = (int)(u & 1);
        if (u >= 2) mbar_wait(&wp_empty[st], (uint32_t)(((u >> 1) - 1) & 1));
        s_wp[st * 512 + cq * 128 + q * 32 + lane] = acc;
        __syncwarp();
        if (lane == 0) mbar_arrive(&wp_full[st]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTcEpiWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
