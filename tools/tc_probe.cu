// tc_probe.cu -- validates the tcgen05 building blocks used by the d=16 pair
// kernels: K-major SWIZZLE_NONE smem descriptors, kind::f16 (bf16) MMA
// M=128 N=256 K=16, 3-way bf16 split with 6 partial products (~fp32-exact
// dot products), TMEM alloc / tcgen05.ld.32x32b / commit-to-mbarrier.
// D[m][n] = sum_r A[m][r] * B[n][r], r < 16, compared with fp64 on the host.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tc_probe.cu -o tools/tc_probe
//        (add -DTC_PROBE_SMALL_FIRST for the partial-product order the library uses).
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element (row, kk) of a K-major no-swizzle operand with 6 chunks of 8 bf16 per row:
// byte offset = (row/8)*768 + (kk/8)*128 + (row%8)*16 + (kk%8)*2
__device__ __forceinline__ int op_off(int row, int kk) { return (row >> 3) * 768 + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2; }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int split) {
  // A: [128][16] fp32, B: [256][16] fp32, D: [128][256]
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;               // 128 rows * 96 B = 12 KB
  unsigned char* sb = smem + 128 * 96;    // 256 rows * 96 B = 24 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 3-way bf16 split: x = x0 + x1 + x2
  for (int e = tid; e < 128 * 16; e += blockDim.x) {
    int row = e / 16, r = e % 16;
    float x = A[e];
    __nv_bfloat16 x0 = __float2bfloat16_rn(x);
    float r1 = x - __bfloat162float(x0);
    __nv_bfloat16 x1 = __float2bfloat16_rn(r1);
    float r2 = r1 - __bfloat162float(x1);
    __nv_bfloat16 x2 = __float2bfloat16_rn(r2);
    *(__nv_bfloat16*)(sa + op_off(row, r)) = x0;
    *(__nv_bfloat16*)(sa + op_off(row, 16 + r)) = x1;
    *(__nv_bfloat16*)(sa + op_off(row, 32 + r)) = x2;
  }
  for (int e = tid; e < 256 * 16; e += blockDim.x) {
    int row = e / 16, r = e % 16;
    float x = B[e];
    __nv_bfloat16 x0 = __float2bfloat16_rn(x);
    float r1 = x - __bfloat162float(x0);
    __nv_bfloat16 x1 = __float2bfloat16_rn(r1);
    float r2 = r1 - __bfloat162float(x1);
    __nv_bfloat16 x2 = __float2bfloat16_rn(r2);
    *(__nv_bfloat16*)(sb + op_off(row, r)) = x0;
    *(__nv_bfloat16*)(sb + op_off(row, 16 + r)) = x1;
    *(__nv_bfloat16*)(sb + op_off(row, 32 + r)) = x2;
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
  // instruction descriptor: F32 accum (bit4), A=BF16 (bits 7-9 = 1), B=BF16 (bits 10-12 = 1),
  // K-major A and B, N>>3 at bits 17-22, M>>4 at bits 24-28
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    // (split_a, split_b) products: 00 01 10 02 11 20 (or only 00 when split == 0)
#ifdef TC_PROBE_SMALL_FIRST  // the order the library uses (qem_tc.cuh umma_tile7): smallest products first
    const int pa[6] = {2, 1, 0, 1, 0, 0}, pb[6] = {0, 1, 2, 0, 1, 0};
#else
    const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
#endif
    const int np = split ? 6 : 1;
    for (int q = 0; q < np; ++q) {
      uint64_t ad = make_desc(a0 + pa[q] * 256, 128, 768);
      uint64_t bd = make_desc(b0 + pb[q] * 256, 128, 768);
      uint32_t acc = q > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for MMA completion
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 TMEM lanes (rows 32w..32w+31), 32 columns at a time
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[row * 256 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(128 * 16), B(256 * 16), D(128 * 256);
  srand(1);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX - 0.5) * 0.01f;
  for (auto& x : B) x = (float)(rand() / (double)RAND_MAX - 0.5) * 3.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  int smem = 128 * 96 + 256 * 96;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int split = 0; split < 2; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxabs = 0, maxrel = 0, scale = 0, sumsigned = 0, sumabsrel = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double s = 0, sa = 0;
        for (int r = 0; r < 16; ++r) {
          s += (double)A[m * 16 + r] * (double)B[n * 16 + r];
          sa += fabs((double)A[m * 16 + r] * (double)B[n * 16 + r]);
        }
        double err = fabs(s - D[m * 256 + n]);
        maxabs = fmax(maxabs, err);
        maxrel = fmax(maxrel, err / sa);
        sumsigned += (D[m * 256 + n] - s) / sa;
        sumabsrel += err / sa;
        scale = fmax(scale, sa);
      }
    printf("mean signed rel err %.3e  mean |rel err| %.3e\n", sumsigned / (128 * 256), sumabsrel / (128 * 256));
    printf("split=%d  max|err|=%.3e  max err/sum|terms|=%.3e  (term scale %.3e)  D[0][0]=%.7e D[127][255]=%.7e\n",
           split, maxabs, maxrel, scale, D[0], D[127 * 256 + 255]);
  }
  return 0;
}
