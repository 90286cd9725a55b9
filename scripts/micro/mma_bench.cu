// Microbenchmark: issue cost and execution time of the attention kernel's tcgen05.mma shapes on this GPU.
// One CTA per SM, one thread issues `n` MMAs back to back (operands: garbage smem / TMEM), commits, waits.
// Reports clocks per MMA for issue (time until the issuing thread is past the last MMA) and completion.
#include <cstdio>
#include <cstdint>
#include "../../paper_2110_10221_b200/csrc/ptx.cuh"
using namespace cora;

__global__ void __launch_bounds__(128, 1) k(int n, int shape, long long* out, int issuers) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((warp == 1 || (issuers == 2 && warp == 2)) && (shape >= 4 || lane == 0)) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t tb = tbase + (warp == 2 ? 256 : 0);
    const uint32_t idesc_s = make_idesc_bf16(128, 128), idesc_o = make_idesc_bf16(128, 64, true),
                   idesc_256 = make_idesc_bf16(128, 256);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (shape == 6) {  // S shape, 2 accumulators interleaved (unrolled: constant TMEM offsets)
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc_s, i & 3);
        umma_bf16_ss(tb + 128, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc_s, i & 3);
        ++i;
      } else if (shape == 7) {  // N64, 4 accumulators interleaved
        const uint32_t id = make_idesc_bf16(128, 64);
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), id, i & 3);
        umma_bf16_ss(tb + 64, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), id, i & 3);
        umma_bf16_ss(tb + 128, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), id, i & 3);
        umma_bf16_ss(tb + 192, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), id, i & 3);
        i += 3;
      } else if (shape == 8) {  // S (acc 0) and PV (acc 192) interleaved: the attention pair of independent chains
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc_s, i & 3);
        umma_bf16_ts(tb + 192, tb + 128 + (i & 7) * 8, make_sdesc_sw128(b + (i & 7) * 2048, 16384, 1024), idesc_o, i & 7);
        ++i;
      }
      else if (shape == 0)  // S: SS, M128 N128 K16
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc_s, i & 3);
      else if (shape == 1)  // PV: TS, M128 N64 K16, B MN-major
        umma_bf16_ts(tb + 192, tb + 128 + (i & 7) * 8, make_sdesc_sw128(b + (i & 7) * 2048, 16384, 1024), idesc_o, i & 7);
      else if (shape == 2)  // SS M128 N64
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), make_idesc_bf16(128, 64), i & 3);
      else if (shape == 3)  // SS M128 N256
        umma_bf16_ss(tb, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), make_sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc_256, i & 3);
      else if (shape == 4) {  // S shape, whole warp, elected issue
        const uint64_t ad = make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), bd = make_sdesc_sw128(b + (i & 3) * 32, 16, 1024);
        if (elect_one()) umma_bf16_ss(tb, ad, bd, idesc_s, i & 3);
        __syncwarp();
      } else {  // PV shape, whole warp, elected issue
        const uint64_t vd = make_sdesc_sw128(b + (i & 7) * 2048, 16384, 1024);
        if (elect_one()) umma_bf16_ts(tb + 192, tb + 128 + (i & 7) * 8, vd, idesc_o, i & 7);
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if (lane == 0) umma_commit(warp == 2 ? &bar2 : &bar);
    mbar_wait<false>(warp == 2 ? &bar2 : &bar, 0);
    long long t2 = clock64();
    if (lane == 0 && warp == 1) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMallocManaged(&out, sms * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* names[] = {"SS M128 N128 K16 (S)", "TS M128 N64 K16 (PV)", "SS M128 N64 K16", "SS M128 N256 K16", "S warp-elect", "PV warp-elect", "S 2 accumulators", "N64 4 accumulators", "PV N32 2 accumulators"};
  for (int issuers = 1; issuers <= 1; ++issuers)
  for (int shape : {0, 1, 3, 6, 7, 8})
    for (int n : {8, 512}) {
      k<<<sms, 128, 65536>>>(n, shape, out, issuers);
      k<<<sms, 128, 65536>>>(n, shape, out, issuers);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      double is = 0, co = 0;
      for (int i = 0; i < sms; ++i) is += out[2 * i], co += out[2 * i + 1];
      printf("{\"issuers\": %d, \"mma\": \"%s\", \"n\": %d, \"issue_clk_per_mma\": %.1f, \"complete_clk_per_mma\": %.1f, \"first_complete_clk\": %.0f}\n",
             issuers, names[shape], n, is / sms / n, co / sms / n, co / sms);
    }
  return 0;
}
