#include <cstdio>
#include <cuda_fp16.h>
#include <cstdint>
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t v[16]; float f[16];
  for (int i = 0; i < 16; ++i) { v[i] = 0x3c003c00u ^ (threadIdx.x + i); f[i] = threadIdx.x * 1e-6f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) v[i] = ex2h2(v[i]) ^ 0x80008000u;
      else if (MODE == 1) v[i] = ex2bf2(v[i]) ^ 0x80008000u;
      else f[i] = ex2f(f[i]) * -0.5f;
    }
  }
  uint32_t s = 0; for (int i = 0; i < 16; ++i) s ^= v[i] ^ __float_as_uint(f[i]);
  if (s == 0x1234567u) out[threadIdx.x] = s;
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4096 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"ex2.approx.f16x2", "ex2.approx.ftz.bf16x2", "ex2.approx.ftz.f32"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      const int iters = 4096, wps = 16;
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      kern<<<sms, 32 * wps>>>(out, 16);
      cudaEventRecord(a); kern<<<sms, 32 * wps>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double elems = double(sms) * 32 * wps * iters * 16 * (mode < 2 ? 2 : 1);
      if (rep) printf("%s: %.2f elements/clk/SM (%.2f instr/clk/SM)\n", names[mode], elems / (ms * 1e-3) / sms / (clk * 1e3),
                      elems / (mode < 2 ? 2 : 1) / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  return 0;
}
