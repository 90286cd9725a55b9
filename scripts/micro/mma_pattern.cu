// Microbenchmark: tensor-pipe time of the attention kernel's tcgen05.mma issue PATTERNS on this GPU.
// One elected thread per CTA issues `reps` repetitions of a fixed pattern of MMAs (zeroed smem operands,
// descriptors computed in the loop as in the kernels), commits once, waits.  1 or 2 CTAs per SM.
// Output (one JSON line per pattern x CTAs/SM): clocks per MMA of one CTA's stream, and per MMA of the SM.
// Question answered: is an MMA stream slowed by switching accumulator / form / shape between groups?
#include <cstdio>
#include <cstdint>
#include "../../paper_2110_10221_b200/csrc/ptx.cuh"
using namespace cora;

constexpr int kSmem = 96 * 1024;  // 2 CTAs per SM fit

__device__ __forceinline__ void ss(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc, uint32_t acc, uint32_t lbo = 16) {
  umma_bf16_ss(d, make_sdesc_sw128(a, 16, 1024), make_sdesc_sw128(b, lbo, 1024), idesc, acc);
}

template <int P>
__device__ __forceinline__ int body(uint32_t tb, uint32_t a, uint32_t b, int r) {
  constexpr uint32_t n128 = make_idesc_bf16(128, 128), n64 = make_idesc_bf16(128, 64), n256 = make_idesc_bf16(128, 256),
                     n64mn = make_idesc_bf16(128, 64, true);
  const uint32_t acc = r != 0;
  if constexpr (P == 0) {  // S only: 4 x SS N128 into one accumulator
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n128, acc | (k != 0));
    return 4;
  } else if constexpr (P == 1) {  // PV only: 8 x TS N64, B MN-major (P in TMEM cols 128..191, O at 192)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ts(tb + 192, tb + 128 + k * 8, make_sdesc_sw128(b + k * 2048, 16384, 1024), n64mn, acc | (k != 0));
    return 8;
  } else if constexpr (P == 2) {  // 8 x SS N64 K-major, one accumulator
#pragma unroll
    for (int k = 0; k < 8; ++k) ss(tb, a + (k & 3) * 32, b + (k & 3) * 32, n64, acc | (k != 0));
    return 8;
  } else if constexpr (P == 3) {  // the attention step: 4 x SS N128 (S) then 8 x TS N64 (PV)
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n128, k != 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ts(tb + 192, tb + 128 + k * 8, make_sdesc_sw128(b + k * 2048, 16384, 1024), n64mn, acc | (k != 0));
    return 12;
  } else if constexpr (P == 4) {  // two accumulators, groups of 4 (same shape)
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n128, k != 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb + 128, a + k * 32, b + k * 32, n128, k != 0);
    return 8;
  } else if constexpr (P == 5) {  // two accumulators, alternating every MMA
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ss(tb, a + k * 32, b + k * 32, n128, k != 0);
      ss(tb + 128, a + k * 32, b + k * 32, n128, k != 0);
    }
    return 8;
  } else if constexpr (P == 6) {  // 4 x SS N256 into one accumulator
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n256, acc | (k != 0));
    return 4;
  } else if constexpr (P == 7) {  // PV as SS: 8 x SS N64, B MN-major
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ss(tb + 192, make_sdesc_sw128(a + (k & 3) * 32, 16, 1024), make_sdesc_sw128(b + k * 2048, 16384, 1024),
                   n64mn, acc | (k != 0));
    return 8;
  } else if constexpr (P == 8) {  // attention step with an SS-form PV
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n128, k != 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ss(tb + 192, make_sdesc_sw128(a + (k & 3) * 32, 16, 1024), make_sdesc_sw128(b + k * 2048, 16384, 1024),
                   n64mn, acc | (k != 0));
    return 12;
  } else if constexpr (P == 9) {  // 8 x TS N64 with B K-major (isolates the MN-major B)
#pragma unroll
    for (int k = 0; k < 8; ++k) umma_bf16_ts(tb + 192, tb + 128 + k * 8, make_sdesc_sw128(b + (k & 3) * 32, 16, 1024), n64, acc | (k != 0));
    return 8;
  } else if constexpr (P == 10) {  // 8 x SS N128 one accumulator, accumulate always on (no zeroing)
#pragma unroll
    for (int k = 0; k < 8; ++k) ss(tb, a + (k & 3) * 32, b + (k & 3) * 32, n128, 1);
    return 8;
  } else {  // P == 11: two S accumulators and two PV accumulators, FA4-like order S0 S1 PV0 PV1
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb, a + k * 32, b + k * 32, n128, k != 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) ss(tb + 128, a + k * 32, b + k * 32, n128, k != 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ts(tb + 384, tb + 256 + k * 8, make_sdesc_sw128(b + k * 2048, 16384, 1024), n64mn, acc | (k != 0));
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_bf16_ts(tb + 448, tb + 320 + k * 8, make_sdesc_sw128(b + k * 2048, 16384, 1024), n64mn, acc | (k != 0));
    return 24;
  }
}

__device__ volatile int g_stop;
template <int P, int COLS, int BG>
__global__ void __launch_bounds__(512, 1) kern(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSmem / 4; i += blockDim.x) {
    // zeros, or random bf16 pairs in (-2, 2) (BG >= 8: data-dependent tensor-core cost)
    uint32_t h = (i + 1) * 2654435761u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    const uint32_t lo = 0x3f80u | ((h & 0x7f) << 0) | ((h >> 7) & 1u) << 15, hi = 0x3f80u | ((h >> 8) & 0x7f) | ((h >> 15) & 1u) << 15;
    reinterpret_cast<uint32_t*>(smem)[i] = (BG & 8) ? (lo | (hi << 16)) : 0u;
  }
  if (warp == 0) tmem_alloc<COLS>(&tbase);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if ((BG & 16) && warp >= 4) {
    // background MUFU / FMA work (like softmax warps in their exponential phase): 12 warps
    float x[16];
    for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 0.001f + c;
    int it = 0;
    while (!stop && it < 200000) {
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = ex2_approx(fmaf(x[c], 0.999f, -0.5f)) + x[c] * 0.25f;
      ++it;
    }
    if (x[3] == 12345.f) out[0] = 0;
  }
  if ((BG & 3) != 0 && warp >= 4) {
    // background TMEM traffic on columns the MMAs do not touch (lanes of this warp's quadrant)
    const uint32_t ta = tbase + (((warp & 3) * 32) << 16) + (COLS == 512 ? 256 : 0);
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = c;
    int it = 0;
    while (!stop && it < 1000000) {
      if ((BG & 3) == 1) {
        CORA_TMEM_LD_32X32B_X32(ta + (it & 3) * 32, r);
        tmem_ld_wait();
      } else {
        CORA_TMEM_ST_32X32B_X32(ta + (it & 3) * 32, r);
        tmem_st_wait();
      }
      ++it;
    }
    if (r[0] == 12345) out[0] = 0;
  }
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t tb = tbase;
    int n = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) n += body<P>(tb, a, b, r);
    const long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait<false>(&bar, 0);
    const long long t2 = clock64();
    out[blockIdx.x * 3] = t1 - t0;
    out[blockIdx.x * 3 + 1] = t2 - t0;
    out[blockIdx.x * 3 + 2] = n;
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(tbase);
}

template <int P, int BG = 0>
void run(const char* name, int sms, long long* out) {
  for (int per_sm : {1, 2}) {
    if ((BG & 19) && per_sm == 2) continue;
    auto k = per_sm == 1 ? kern<P, 512, BG> : kern<P, 256, BG>;
    if (per_sm == 2 && P == 11) continue;  // needs 512 columns
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    const int reps = 2048 / (P == 11 ? 24 : 8);
    for (int it = 0; it < 2; ++it) k<<<sms * per_sm, (BG & 16) ? 512 : (BG & 3) ? 256 : 128, kSmem>>>(reps, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"error\": \"%s\", \"pattern\": \"%s\"}\n", cudaGetErrorString(e), name);
      exit(1);
    }
    double is = 0, co = 0, n = 0;
    for (int i = 0; i < sms * per_sm; ++i) is += out[3 * i], co += out[3 * i + 1], n += out[3 * i + 2];
    const double per = n / (sms * per_sm);
    printf("{\"pattern\": \"%s\", \"ctas_per_sm\": %d, \"mma_per_cta\": %.0f, \"issue_clk_per_mma\": %.1f, "
           "\"complete_clk_per_mma_cta\": %.1f, \"complete_clk_per_mma_sm\": %.1f}\n",
           name, per_sm, per, is / (sms * per_sm) / per, co / (sms * per_sm) / per, co / (sms * per_sm) / per / per_sm);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMallocManaged(&out, sms * 2 * 3 * sizeof(long long));
  run<0>("S only: SS M128 N128 K16 x4, one acc (nominal 64 clk)", sms, out);
  run<10>("SS M128 N128 K16 x8, accumulate on", sms, out);
  run<6>("SS M128 N256 K16 x4, one acc (nominal 128)", sms, out);
  run<2>("SS M128 N64 K16 x8 K-major, one acc (nominal 32)", sms, out);
  run<1>("PV only: TS M128 N64 K16 x8, B MN-major (nominal 32)", sms, out);
  run<9>("TS M128 N64 K16 x8, B K-major", sms, out);
  run<7>("SS M128 N64 K16 x8, B MN-major", sms, out);
  run<3>("attention step: S (4 SS N128) + PV (8 TS N64)", sms, out);
  run<8>("attention step, PV as SS: S (4 SS N128) + PV (8 SS N64 MN-major)", sms, out);
  run<4>("two accumulators, groups of 4 SS N128", sms, out);
  run<5>("two accumulators alternating every SS N128", sms, out);
  run<11>("FA4 order S0 S1 PV0 PV1 (1 CTA, 512 cols)", sms, out);
  run<3, 16>("attention step + 12 warps of MUFU/FMA work", sms, out);
  run<1, 16>("PV only + 12 warps of MUFU/FMA work", sms, out);
  run<11, 16>("FA4 order + 12 warps of MUFU/FMA work", sms, out);
  run<0, 8>("S only, random operands", sms, out);
  run<1, 8>("PV only, random operands", sms, out);
  run<3, 8>("attention step, random operands", sms, out);
  run<11, 8>("FA4 order, random operands", sms, out);
  run<3, 1>("attention step + 4 warps of tcgen05.ld x32 on other columns", sms, out);
  run<3, 2>("attention step + 4 warps of tcgen05.st x32 on other columns", sms, out);
  run<0, 1>("S only + 4 warps of tcgen05.ld", sms, out);
  run<1, 1>("PV only + 4 warps of tcgen05.ld", sms, out);
  run<1, 2>("PV only + 4 warps of tcgen05.st", sms, out);
  return 0;
}
