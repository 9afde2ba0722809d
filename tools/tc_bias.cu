// tc_bias.cu -- accumulation error of tcgen05 kind::f16 MMAs (bf16 inputs, fp32 TMEM accumulator)
// for the compact (d = 1) operand arrangements of qem_tc.cuh: is the sum of the 16 exact bf16
// products of one MMA (and of several MMAs into one accumulator) rounded to nearest, or biased?
// The products themselves are exact, so any error is the tensor core's accumulation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tc_bias.cu -o tools/tc_bias
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// slab q of a K-major operand: rows x 16 bf16, 32 B per row, 8-row groups 256 B apart
__device__ __forceinline__ int slab_off(int rows, int q, int row, int kk) {
  return q * rows * 32 + (row >> 3) * 256 + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2;
}

// A [128][16 NM], B [256][16 NM] bf16 (row-major, MMA q uses entries 16q..16q+15); D [128][256]
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int NM) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;
  unsigned char* sb = smem + 128 * 32 * NM;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 16 * NM; e += blockDim.x) {
    const int row = e / (16 * NM), k = e % (16 * NM);
    *(__nv_bfloat16*)(sa + slab_off(128, k / 16, row, k % 16)) = A[e];
  }
  for (int e = tid; e < 256 * 16 * NM; e += blockDim.x) {
    const int row = e / (16 * NM), k = e % (16 * NM);
    *(__nv_bfloat16*)(sb + slab_off(256, k / 16, row, k % 16)) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    for (int q = 0; q < NM; ++q) {
      const uint64_t ad = make_desc(smem_u32(sa) + q * 128 * 32, 128, 256);
      const uint64_t bd = make_desc(smem_u32(sb) + q * 256 * 32, 128, 256);
      const uint32_t acc = q > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < 256; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[row * 256 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static void split3(float x, __nv_bfloat16* s) {
  s[0] = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(s[0]);
  s[1] = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(s[1]);
  s[2] = __float2bfloat16_rn(r2);
}

// arrangement: 0 = compact (one 12-product slab), 1 = three slabs by magnitude class (small first),
// 2 = compact with the large pair (c0 w0, g0 S0) moved to a second slab after the rest;
// with lp != 0 a log-probability lP ~ -U(0, lpmax) per column joins as three split entries (x 1):
// 3 = the c-region slab then an lP slab (the forward's layout), 4 = lP slab first, 5 = lP inside the
// c-region slab (entries 12-14)
static void run(int arr, float cscale, float gscale, float wscale, float m, float lpmax = 0.f) {
  const int NM = (arr == 0 || arr == 5) ? 1 : (arr == 1 ? 3 : 2);
  std::mt19937 rng(7);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<__nv_bfloat16> A(128 * 16 * NM, __float2bfloat16_rn(0.f)), B(256 * 16 * NM, __float2bfloat16_rn(0.f));
  auto put = [&](std::vector<__nv_bfloat16>& X, int row, int q, int k, __nv_bfloat16 v) { X[row * 16 * NM + 16 * q + k] = v; };
  // (slab, entry) of the 12 products (a_term, b_term, which): which 0 = c w, 1 = g S
  struct P { int ia, ib, which; };
  const P prods[12] = {{2, 0, 0}, {1, 1, 0}, {0, 2, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 0},
                       {0, 0, 1}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}, {1, 1, 1}};
  int slab[12], ent[12];
  for (int p = 0; p < 12; ++p) {
    const int order = prods[p].ia + prods[p].ib;
    if (arr == 0 || arr >= 3) { slab[p] = arr == 4 ? 1 : 0; ent[p] = p; }
    else if (arr == 1) { slab[p] = 2 - order; ent[p] = p; }  // order 2 first (slab 0), order 0 last
    else { slab[p] = order == 0 ? 1 : 0; ent[p] = p; }
  }
  const int lslab = arr == 3 ? 1 : 0, lent = arr == 5 ? 12 : 0;  // where the 3 lP entries go (arr >= 3)
  for (int r = 0; r < 128; ++r) {
    __nv_bfloat16 cs[3], gs[3];
    split3(cscale * nd(rng), cs);
    split3(gscale * nd(rng), gs);
    for (int p = 0; p < 12; ++p) put(A, r, slab[p], ent[p], prods[p].which ? gs[prods[p].ia] : cs[prods[p].ia]);
    if (arr >= 3)
      for (int q = 0; q < 3; ++q) put(A, r, lslab, lent + q, __float2bfloat16_rn(1.f));
  }
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  for (int c = 0; c < 256; ++c) {
    const float w = wscale * nd(rng);
    const float S = fmaf(2.f, m * w, w * w);
    __nv_bfloat16 ws[3], ss[3];
    split3(w, ws);
    split3(S, ss);
    for (int p = 0; p < 12; ++p) put(B, c, slab[p], ent[p], prods[p].which ? ss[prods[p].ib] : ws[prods[p].ib]);
    if (arr >= 3) {
      __nv_bfloat16 ls[3];
      split3(-lpmax * ud(rng), ls);
      for (int q = 0; q < 3; ++q) put(B, c, lslab, lent + q, ls[q]);
    }
  }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (128 + 256) * 32 * NM;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dD, NM);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return; }
  std::vector<float> D(128 * 256);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double bias = 0, mabs = 0, mx = 0, bias_ulp = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 256; ++c) {
      double s = 0, pmax = 0;
      for (int k = 0; k < 16 * NM; ++k) {
        const double p = (double)__bfloat162float(A[r * 16 * NM + k]) * (double)__bfloat162float(B[c * 16 * NM + k]);
        s += p;
        pmax = fmax(pmax, fabs(p));
      }
      const double err = (double)D[r * 256 + c] - s;
      const double ulp = std::ldexp(1.0, std::ilogb(fmax(fabs(s), 1e-30)) - 23);  // fp32 ulp of the result
      bias += err / pmax;
      bias_ulp += err / ulp;
      mabs += fabs(err) / pmax;
      mx = fmax(mx, fabs(err) / pmax);
    }
  const double N = 128.0 * 256.0;
  printf("arr=%d cs=%.2g gs=%.2g ws=%.2g m=%.2g: mean signed err/max|prod| %+.3e  mean signed err in result ulps %+.3f  "
         "mean |err|/max|prod| %.3e  max %.3e\n", arr, cscale, gscale, wscale, m, bias / N, bias_ulp / N, mabs / N, mx);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

int main() {
  for (int arr = 0; arr < 3; ++arr) {
    run(arr, 1.f, 0.3f, 0.3f, -0.65f);
    run(arr, 3.f, 1.f, 1.f, -0.65f);
  }
  for (int arr = 3; arr < 6; ++arr) {
    run(arr, 1.f, 0.3f, 0.3f, -0.65f, 15.f);
    run(arr, 3.f, 1.f, 1.f, -0.65f, 15.f);
    run(arr, 10.f, 3.f, 1.f, -0.65f, 30.f);
  }
  return 0;
}
