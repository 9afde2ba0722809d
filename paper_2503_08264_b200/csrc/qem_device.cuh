// qem_device.cuh -- device helpers for the sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace qem {

constexpr double kLn2Pi = 1.8378770664093454835606594728112;
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLog2eD = 1.4426950408889634074;
constexpr double kLn2D = 0.69314718055994530942;

__device__ __forceinline__ float ex2(float x) {
#ifdef QEM_EXACT_EX2  // diagnostics: the libm 2^x instead of the SFU's ex2.approx
  return exp2f(x);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// 2^x on the FMA pipe for two values (FFMA2/FADD2), to share the exp load with the SFU
// (MUFU.EX2 is the binding pipe of the pair epilogues): x = n + f, n = rint(x) by the
// 1.5*2^23 shifter, 2^f by a degree-5 polynomial fitted on [-1/2, 1/2] (max relative error
// 2.3e-7 in fp32, vs ~1.7e-7 for ex2.approx), 2^n added into the exponent field.
// Inputs below -127 are clamped (2^-127: negligible wherever it is used).
// Order-independent sum of fp64 terms (the FFMA forward's plate sums: which CTA adds which group
// differs from launch to launch with its dynamic group queue).  Each term x is split, with two
// round-to-grid steps (add and subtract a power-of-two-scaled 1.5), into h = x on the 2^-20 grid and
// m = (x - h) on the 2^-57 grid (the rest, < 2^-58, is dropped); sums of h are exact while |sum h| <
// 2^33 and sums of m while fewer than 2^17 terms meet (|m| <= 2^-21), so the totals do not depend
// on the order.  Only DADDs (FP64 pipe): nothing lands on the XU pipe the pair tiles' ex2 saturate.
// Past those bounds the sums stay fp64-accurate but order-dependent in the last bits.
struct Fx2 {
  double h = 0.0, m = 0.0;
  __device__ __forceinline__ void add(Fx2 t) {
    h += t.h;
    m += t.m;
  }
  __device__ __forceinline__ void add(double x) {
    const double th = __dsub_rn(__dadd_rn(x, 0x1.8p32), 0x1.8p32);  // x on the 2^-20 grid
    const double r = __dsub_rn(x, th);                                // exact
    const double tm = __dsub_rn(__dadd_rn(r, 0x1.8p-5), 0x1.8p-5);    // r on the 2^-57 grid
    h += th;
    m += tm;
  }
  __device__ __forceinline__ double value() const { return h + m; }
};

// ln x in fp64 for a positive normal fp32 x, branch-free: x = 2^e m with m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh(s), s = (m - 1)/(m + 1) (|s| <= 0.1716), the atanh series to s^21 (next term
// < 3e-17); 1/(m + 1) from the fp32 reciprocal and two fp64 Newton steps.  Absolute error
// <= 2e-15 for x up to 2^24 (checked against math.log on 2e5 points).  The fp64 logs of the
// pair tiles' sums go through this instead of the library log (a third of the instructions).
__device__ __forceinline__ double log_pos_f32(float x) {
  const int ix = __float_as_int(x);
  int e = ((ix >> 23) & 0xff) - 127;
  int mi = (ix & 0x7fffff) | 0x3f800000;
  if (mi > 0x3fb504f3) {
    mi -= 0x00800000;
    e += 1;
  }
  const double f = (double)__int_as_float(mi) - 1.0;  // exact
  const double d = 2.0 + f;
  double r;
  {
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)d));
    r = rf;
  }
  r = r * fma(-d, r, 2.0);
  r = r * fma(-d, r, 2.0);
  const double s = f * r, s2 = s * s;
  double p = 1.0 / 21;
#pragma unroll
  for (int k = 19; k >= 1; k -= 2) p = fma(p, s2, 1.0 / k);
  return fma((double)e, 0.69314718055994530942, 2.0 * s * p);
}

__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 t = add2(x, f2(12582912.f));
  const float2 nf = add2(t, f2(-12582912.f));
  const float2 fr = add2(x, make_float2(-nf.x, -nf.y));
  float2 p = f2(0.001327647129073739f);
  p = fma2(p, fr, f2(0.009675540961325169f));
  p = fma2(p, fr, f2(0.05550713092088699f));
  p = fma2(p, fr, f2(0.24022120237350464f));
  p = fma2(p, fr, f2(0.6931469440460205f));
  p = fma2(p, fr, f2(1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Philox4x32-10 (Salmon et al., SC'11).  Same counter/key convention as the
// DESIGN.md "Sampler" section; integer-exact.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// r = sqrt(-2 ln u), u = (m + 1/2) 2^-23, m a 23-bit integer.  Near u = 1 (v = 1 - u < 2^-5,
// exact in fp32) -ln u = v + v^2/2 + ... + v^6/6 (error < v^7/7 < 1e-11); elsewhere
// ln u = ln2 lg2.approx(u) (absolute error ~1.7e-7, i.e. <= 7e-7 on r >= 0.25 there).
__device__ __forceinline__ float bm_radius(uint32_t m) {
  const float u = ((float)m + 0.5f) * 1.1920928955078125e-07f;
  float nl;
  if (m >= 8126464u) {  // u > 1 - 2^-5
    const float v = ((float)(8388607u - m) + 0.5f) * 1.1920928955078125e-07f;
    nl = v * fmaf(v, fmaf(v, fmaf(v, fmaf(v, fmaf(v, 1.f / 6.f, 0.2f), 0.25f), 1.f / 3.f), 0.5f), 1.f);
  } else {
    float l2;
    asm("lg2.approx.f32 %0, %1;" : "=f"(l2) : "f"(u));
    nl = -0.69314718055994531f * l2;
  }
  const float x = 2.f * nl;
  float rs;
  asm("rsqrt.approx.f32 %0, %1;" : "=f"(rs) : "f"(x));
  return x * rs;
}
// (sin, cos) of 2 pi u, u = (m + 1/2) 2^-23: quadrant from the top two bits, reflection to
// [0, pi/4] exact in fp32, Taylor polynomials (sin to x^9, cos to x^10; error < 3e-8).
__device__ __forceinline__ void bm_sincos2pi(uint32_t m, float& sn, float& cs) {
  const uint32_t q = m >> 21;                                          // quadrant
  float f = ((float)(m & 0x1FFFFFu) + 0.5f) * 4.76837158203125e-07f;  // in (0, 1): angle f pi/2
  const bool hi = f > 0.5f;
  if (hi) f = 1.f - f;  // exact (Sterbenz)
  const float x = f * 1.5707963267948966f, x2 = x * x;
  const float sa = x * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.7557319e-6f, -1.9841270e-4f), 8.3333333e-3f),
                                     -1.6666667e-1f), 1.f);
  const float ca = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, -2.7557319e-7f, 2.4801587e-5f), -1.3888889e-3f),
                                           4.1666667e-2f), -0.5f), 1.f);
  const float s1 = hi ? ca : sa, c1 = hi ? sa : ca;  // sin, cos of the in-quadrant angle
  switch (q) {
    case 0: sn = s1; cs = c1; break;
    case 1: sn = c1; cs = -s1; break;
    case 2: sn = -s1; cs = -c1; break;
    default: sn = -c1; cs = s1; break;
  }
}

// Four N(0,1) draws of one Philox4x32-10 call: Box-Muller on
// u = ((x >> 9) + 0.5) 2^-23, radius and angle evaluated from the integer bits (bm_radius,
// bm_sincos2pi: ~3x fewer instructions than sqrtf(-2 logf(u)) and sincospif(2u); absolute error
// <= ~1e-6 on eps vs the fp64 transform).  The sampler (k_sample) and the fused column prep
// (k_colprep_tc) both draw through this, so their samples are bit-identical.
__device__ __forceinline__ float4 philox_normal4(uint4 ctr, uint2 key) {
  const uint4 o = philox4x32_10(ctr, key);
  const float r0 = bm_radius(o.x >> 9), r1 = bm_radius(o.z >> 9);
  float s0, c0, s1, c1;
  bm_sincos2pi(o.y >> 9, s0, c0);
  bm_sincos2pi(o.w >> 9, s1, c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

// ------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bulk (non-tensor) TMA copy global -> shared, completion signalled on `bar`.
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bulk prefetch of a global range into L2 (bytes % 16 == 0).
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// cp.async (LDGSTS) 16 bytes global -> shared, L2 only; groups committed / waited per thread.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Named barrier `id` (1..15) over `n` threads (a multiple of 32).
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// three-input max (FMNMX3 on sm_100a)
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware (woken when the phase
// completes) instead of spinning and taking issue slots from the epilogue warps.
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t a, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(a), "r"(parity), "r"(1000000u)
      : "memory");
  return done;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait for the phase of `bar` with the given parity.  A wait longer than 10 s traps (a protocol
// bug then fails the launch with an error instead of hanging the GPU).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const uint64_t t0 = global_ns();
  while (!mbar_try_wait(a, parity))
    if (global_ns() - t0 > 10000000000ull) __trap();
}

// ------------------------------------------- tcgen05 operand helpers (d = 16)
// Tensor-core operands hold a 16-dim fp32 vector per row as three bf16 terms
// (x = x0 + x1 + x2, each round-to-nearest), i.e. 48 bf16 = 96 bytes per row,
// in the K-major SWIZZLE_NONE canonical layout: 8-row x 16-byte core matrices,
// chunks of 8 bf16 along K 128 B apart (LBO), 8-row groups 768 B apart (SBO).
constexpr int kTcRowBytes = 96;
__host__ __device__ __forceinline__ int tc_offset(int row, int kk) {
  return (row >> 3) * 768 + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2;
}
__device__ __forceinline__ void split3_bf16(float x, __nv_bfloat16 (&s)[3]) {
  s[0] = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(s[0]);
  s[1] = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(s[1]);
  s[2] = __float2bfloat16_rn(r2);
}
// Column operand of the restructured tensor-core path: 128 B per column =
// the 3 x 16 bf16 split of u (chunks 0-5) + one 16-entry "extra" K-slab
// (chunks 6-7); 8-row groups 1024 B apart.
constexpr int kTcColBytes = 128;
// Row-extra operand (forward A-extra / backward B-extra): one 16-entry slab,
// 32 B per row, 8-row groups 256 B apart.
constexpr int kTcRowXBytes = 32;
__host__ __device__ __forceinline__ int tc_col_offset(int row, int kk) {
  return (row >> 3) * 1024 + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2;
}
__host__ __device__ __forceinline__ int tc_rowx_offset(int row, int kk) {
  return (row >> 3) * 256 + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2;
}
// Any K-major no-swizzle operand of `rb` bytes per row (8-row groups 8 rb apart).
__host__ __device__ __forceinline__ int tc_off(int row, int kk, int rb) {
  return (row >> 3) * (8 * rb) + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2;
}
__device__ __forceinline__ uint32_t pack_bf16x2(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
// 8 bf16 (as floats already representable in bf16, or rounded) -> one 16-byte core-matrix row
__device__ __forceinline__ uint4 pack8_bf16(const __nv_bfloat16 (&v)[8]) {
  return make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                    pack_bf16x2(v[6], v[7]));
}
// UMMA shared-memory descriptor: start address, LBO, SBO (bytes), version 1, no swizzle.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// Instruction descriptor kind::f16: fp32 accumulate, bf16 A/B, K-major, N, M.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// D += A_split . B_split over the 3-term splits, small products first (measured
// max error 1e-7 of sum|a_r b_r|, unbiased: tools/tc_probe.cu).
__device__ __forceinline__ void umma_bf16x3(uint32_t tmem_d, uint32_t a_saddr, uint32_t b_saddr, uint32_t idesc) {
  const int pa[6] = {2, 1, 0, 1, 0, 0}, pb[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
  for (int q = 0; q < 6; ++q)
    umma_bf16(tmem_d, umma_desc(a_saddr + pa[q] * 256, 128, 768), umma_desc(b_saddr + pb[q] * 256, 128, 768), idesc,
              q > 0);
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 lanes x 32 columns of fp32 from TMEM (each thread: its lane, 32 consecutive columns).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// 32 lanes x 16 columns, asynchronous: the registers are valid only after tmem_wait().
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// Wait for all outstanding tcgen05.ld; the registers of `r` are threaded through
// the asm so no use of them can be scheduled before the wait.
__device__ __forceinline__ void tmem_wait16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

// Read-only 128-bit global loads as volatile asm: issued in program order and never
// sunk next to their first use, so a batch of them is in flight together.
__device__ __forceinline__ float4 ldg_nc_v4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldg_nc_v2d(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_d(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Register-dependency fence: no use of `r` is scheduled before this point (pairs with a
// preceding tcgen05.wait::ld, since volatile asm statements keep their relative order).
__device__ __forceinline__ void reg_fence16(uint32_t (&r)[16]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
// 32 lanes x 64 columns from TMEM in one go: four x16 loads in flight, one wait.
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[4][16]) {
  tmem_ld16_async(taddr, r[0]);
  tmem_ld16_async(taddr + 16, r[1]);
  tmem_ld16_async(taddr + 32, r[2]);
  tmem_ld16_async(taddr + 48, r[3]);
  tmem_wait16(r[0]);
  reg_fence16(r[1]);
  reg_fence16(r[2]);
  reg_fence16(r[3]);
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions; `scratch` holds >= 32 doubles; all threads get the
// result.  Fixed order (deterministic).  Contains __syncthreads().
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += scratch[w];
  return t;
}
__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = -CUDART_INF;
  for (int w = 0; w < nw; ++w) t = fmax(t, scratch[w]);
  return t;
}

// log N(x; m, v) in fp64.
__device__ __forceinline__ double lnN(double x, double m, double v) {
  const double r = x - m;
  return -0.5 * (kLn2Pi + log(v)) - 0.5 * r * r / v;
}

// log Poisson(y; exp(eta)), fp64.
__device__ __forceinline__ double log_pois(double y, double eta, double lgy1) {
  return y * eta - exp(eta) - lgy1;
}

// Iteration number: explicit (>0) or the device counter (graph mode).
__device__ __forceinline__ int resolve_iter(int t_host, const int32_t* d_iter) {
  return t_host > 0 ? t_host : *d_iter;
}

}  // namespace qem
