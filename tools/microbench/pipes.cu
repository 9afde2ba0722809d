// K7 microbenchmarks: FFMA, FFMA2 (f32x2), MUFU.EX2, DFMA throughput per SM-clock.
// Measures the roofline denominators DESIGN.md uses for the pair-tile kernels.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
  float2 x4 = make_float2(8, 9), x5 = make_float2(10, 11), x6 = make_float2(12, 13), x7 = make_float2(14, 15);
  float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = __ffma2_rn(x0, A, B); x1 = __ffma2_rn(x1, A, B); x2 = __ffma2_rn(x2, A, B); x3 = __ffma2_rn(x3, A, B);
      x4 = __ffma2_rn(x4, A, B); x5 = __ffma2_rn(x5, A, B); x6 = __ffma2_rn(x6, A, B); x7 = __ffma2_rn(x7, A, B);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x4.y + x5.y + x6.y + x7.y;
}
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k_ex2(float* out, float a) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f, x4 = x0+.4f, x5=x0+.5f, x6=x0+.6f, x7=x0+.7f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = ex2(x0) ; x1 = ex2(x1); x2 = ex2(x2); x3 = ex2(x3); x4 = ex2(x4); x5 = ex2(x5); x6 = ex2(x6); x7 = ex2(x7);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// Mixed: 1 ex2 + N ffma per element, to see whether MUFU and FMA overlap.
template <int NF>
__global__ void k_mix(float* out, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  float y0 = 0, y1 = 0, y2 = 0, y3 = 0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float e0 = ex2(x0), e1 = ex2(x1), e2 = ex2(x2), e3 = ex2(x3);
#pragma unroll
      for (int f = 0; f < NF; ++f) { y0 = fmaf(y0, a, e0); y1 = fmaf(y1, a, e1); y2 = fmaf(y2, a, e2); y3 = fmaf(y3, a, e3); }
      x0 = e0 * b; x1 = e1 * b; x2 = e2 * b; x3 = e3 * b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1 + y2 + y3 + x0;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  float* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256;  // 2048 threads per SM? (8x256) -> clamp by occupancy
  auto run = [&](const char* name, auto launch, double ops_per_thread) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = ops_per_thread * blocks * threads * 5;
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    printf("%-10s %.3f ms  %.3e ops/s  %.2f ops/clk/SM at max clock %d MHz\n", name, ms, ops / (ms * 1e-3),
           ops / (ms * 1e-3) / (sms * clk_khz * 1e3), clk_khz / 1000);
  };
  run("ffma", [&] { k_ffma<<<blocks, threads>>>(out, 1.0000001f, 1e-7f); }, 32.0 * ITERS);
  run("ffma2", [&] { k_ffma2<<<blocks, threads>>>(out, 1.0000001f, 1e-7f); }, 64.0 * ITERS);
  run("ex2", [&] { k_ex2<<<blocks, threads>>>(out, 1.0f); }, 32.0 * ITERS);
  run("mix1", [&] { k_mix<1><<<blocks, threads>>>(out, 0.5f, 1e-3f); }, 16.0 * ITERS);
  run("mix4", [&] { k_mix<4><<<blocks, threads>>>(out, 0.5f, 1e-3f); }, 16.0 * ITERS);
  run("mix8", [&] { k_mix<8><<<blocks, threads>>>(out, 0.5f, 1e-3f); }, 16.0 * ITERS);
  run("dfma", [&] { k_dfma<<<blocks, threads>>>((double*)out, 1.0000001, 1e-7); }, 8.0 * ITERS);
  printf("sms=%d\n", sms);
  return 0;
}
