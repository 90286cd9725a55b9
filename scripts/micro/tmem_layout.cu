// Probe of the tcgen05.ld/st 16x128b and 16x64b thread <-> (lane, column) mappings on this GPU.
#include <cstdio>
#include <cstdint>

__global__ void k(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  // warp q (0..3) writes lanes 32q..32q+31, cols 0..31 with value (lane << 16) | col  (32x32b: thread t <-> lane 32q+t)
  if (warp < 4) {
    uint32_t v[8];
    for (int c0 = 0; c0 < 32; c0 += 8) {
      for (int e = 0; e < 8; ++e) v[e] = ((32 * warp + lane) << 16) | (c0 + e);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + ((32 * warp) << 16) + c0),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp 1 (quadrant 1) loads at lane base 32 + 16 with 16x128b.x2 (8 cols): 4 regs per thread
  if (warp == 1) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(tb + ((32 + 16) << 16) + 0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int e = 0; e < 4; ++e) out[lane * 4 + e] = r[e];
    uint32_t s[2];
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(s[0]), "=r"(s[1]) : "r"(tb + ((32 + 16) << 16) + 4));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int e = 0; e < 2; ++e) out[128 + lane * 2 + e] = s[e];
    uint32_t q[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
                 : "r"(tb + ((32 + 16) << 16) + 8));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int e = 0; e < 4; ++e) out[192 + lane * 4 + e] = q[e];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4096 * 4);
  cudaMemset(d, 0xff, 4096 * 4);
  k<<<1, 128>>>(d);
  uint32_t h[320];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  printf("16x128b.x2 at lane 48 col 0: thread: (lane,col) per reg\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int r = 0; r < 4; ++r) printf(" (%u,%u)", h[t * 4 + r] >> 16, h[t * 4 + r] & 0xffff);
    printf("\n");
  }
  printf("16x64b.x2 at lane 48 col 4:\n");
  for (int t = 0; t < 32; ++t) printf("t%2d: (%u,%u) (%u,%u)\n", t, h[128 + t * 2] >> 16, h[128 + t * 2] & 0xffff, h[129 + t * 2] >> 16, h[129 + t * 2] & 0xffff);
  printf("16x256b.x1 at lane 48 col 8:\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int r = 0; r < 4; ++r) printf(" (%u,%u)", h[192 + t * 4 + r] >> 16, h[192 + t * 4 + r] & 0xffff);
    printf("\n");
  }
  return 0;
}
