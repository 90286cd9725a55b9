// Steps a2 / a4 / a6 / a7: the packed ("vloop-fused") linear operators of the encoder layer.
//
// CoRa implements QKV Proj, Linear Proj, FF1 and FF2 as GEMMs over the fused token loop
// ("We use vloop fusion ... to implement the linear transformation
// operators ... with minimal padding"), with the bias / activation / residual add fused into
// the GEMM (Table ap_op_times).  CoRa additionally bulk-pads sum L to a
// multiple of 64; here no padding exists at all: the M tail is zero-filled
// by TMA on load and clipped by TMA on store.
//
// sm_100a design: persistent, warp-specialised, one CTA per SM
//   warp 0      : TMA producer (A 128x64 and B BNx64 bf16 tiles, SWIZZLE_128B, mbarrier ring)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  : epilogue, one TMEM lane quadrant each: tcgen05.ld -> +bias -> act ->
//                 +residual -> bf16 -> swizzled smem -> TMA store (per warp, 32 rows x 64 cols)
//   TMEM holds two BN-column fp32 accumulators so the epilogue of tile i overlaps the
//   main loop of tile i+1.
#include <cuda_bf16.h>

#include <cstdint>

#include "cora_internal.h"
#include "ptx.cuh"

namespace cora {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiRows = 32;                      // rows per epilogue warp
constexpr int kEpiBufBytes = kEpiRows * BK * 2;   // 4 KB staging buffer (32 rows x 128 B)

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + STAGES * kABytes;
  static constexpr int kOffC = kOffB + STAGES * kBBytes;
  static constexpr int kOffBar = kOffC + kEpiWarps * 2 * kEpiBufBytes;
  // full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2], tmem ptr
  static constexpr int kBytes = kOffBar + (2 * STAGES + 4) * 8 + 16;
  static constexpr int kAlloc = kBytes + 1024;  // manual 1024-B alignment (SWIZZLE_128B atoms)
  static constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
};

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float apply_act(float x, int act) {
  if (act == CORA_ACT_RELU) return fmaxf(x, 0.f);
  if (act == CORA_ACT_GELU_ERF) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
  return x;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                        const __grid_constant__ CUtensorMap tm_c, const __nv_bfloat16* __restrict__ bias,
                        const __nv_bfloat16* __restrict__ residual, int32_t M, int32_t N, int32_t K, int32_t act) {
  using S = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int m_blocks = (M + BM - 1) / BM;
  const int n_blocks = (N + BN - 1) / BN;
  const int num_tiles = m_blocks * n_blocks;
  const int k_blocks = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_c);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<S::kTmemCols>(tmem_ptr);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m0 = (t / n_blocks) * BM, n0 = (t % n_blocks) * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + S::kOffA + stage * S::kABytes;
          uint8_t* sb = smem + S::kOffB + stage * S::kBBytes;
          mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
          tma_load_2d(sa, &tm_a, &full[stage], kb * BK, m0);
          tma_load_2d(sb, &tm_b, &full[stage], kb * BK, n0);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + S::kOffA + stage * S::kABytes);
          const uint32_t b_addr = smem_u32(smem + S::kOffB + stage * S::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(b_addr + k * 32, 16, 1024);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        umma_commit(&tmem_full[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    const uint32_t q = warp & 3;  // TMEM lane quadrant accessible to this warp
    uint8_t* cbuf = smem + S::kOffC + (warp - 2) * 2 * kEpiBufBytes;
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int m0 = (t / n_blocks) * BM, n0 = (t % n_blocks) * BN;
      const int row = m0 + q * 32 + lane;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int n_chunks = min(BN, N - n0 + BK - 1) / BK;  // 64-col chunks that intersect [0, N)
#pragma unroll 1
      for (int c = 0; c < n_chunks; ++c) {
        const int nc = n0 + c * BK;
        uint32_t r[64];
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN + c * BK;
        CORA_TMEM_LD_32X32B_X32(taddr, r);
        CORA_TMEM_LD_32X32B_X32(taddr + 32, (r + 32));
        tmem_ld_wait();
        if (c == n_chunks - 1) {
          // all TMEM reads of this accumulator are done: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tmem_empty[acc]);
        }
        float v[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]);
        if (bias != nullptr) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (nc + g * 8 < N) {
              const uint4 bw = __ldg(reinterpret_cast<const uint4*>(bias + nc + g * 8));
              const uint32_t w[4] = {bw.x, bw.y, bw.z, bw.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                v[g * 8 + 2 * i] += bf16_lo(w[i]);
                v[g * 8 + 2 * i + 1] += bf16_hi(w[i]);
              }
            }
          }
        }
        if (act != CORA_ACT_NONE) {
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = apply_act(v[j], act);
        }
        if (residual != nullptr && row < M) {
          const __nv_bfloat16* rp = residual + static_cast<size_t>(row) * N + nc;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (nc + g * 8 < N) {
              const uint4 rw = *reinterpret_cast<const uint4*>(rp + g * 8);
              const uint32_t w[4] = {rw.x, rw.y, rw.z, rw.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                v[g * 8 + 2 * i] += bf16_lo(w[i]);
                v[g * 8 + 2 * i + 1] += bf16_hi(w[i]);
              }
            }
          }
        }
        // staging buffer `buf` was last read by the TMA store issued two chunks ago
        if (lane == 0) tma_store_wait_read<1>();
        __syncwarp();
        uint8_t* sbuf = cbuf + buf * kEpiBufBytes;
        const uint32_t sbase = smem_u32(sbuf);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          st_shared_v4(sbase + sw128_offset(lane, ch), pack_bf16x2(v[ch * 8 + 0], v[ch * 8 + 1]),
                       pack_bf16x2(v[ch * 8 + 2], v[ch * 8 + 3]), pack_bf16x2(v[ch * 8 + 4], v[ch * 8 + 5]),
                       pack_bf16x2(v[ch * 8 + 6], v[ch * 8 + 7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tm_c, sbuf, nc, m0 + q * 32);
          tma_store_commit();
        }
        buf ^= 1;
      }
      if (n_chunks == 0) {  // cannot happen for a valid tile, kept for safety
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      }
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<S::kTmemCols>(tmem_base);
}

template <int BN, int STAGES>
cudaError_t run_gemm(const GemmArgs& g, cudaStream_t stream) {
  using S = GemmSmem<BN, STAGES>;
  CUtensorMap ta, tb, tc;
  if (!make_tmap_2d_bf16(&ta, g.a, g.k, g.m, static_cast<uint64_t>(g.k) * 2, BK, BM, true) ||
      !make_tmap_2d_bf16(&tb, g.b, g.k, g.n, static_cast<uint64_t>(g.k) * 2, BK, BN, true) ||
      !make_tmap_2d_bf16(&tc, g.c, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
    return cudaErrorInvalidValue;
  auto kern = gemm_bf16_tn_kernel<BN, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN);
  const int grid = tiles < device_sm_count() ? tiles : device_sm_count();
  kern<<<grid, kThreads, S::kAlloc, stream>>>(ta, tb, tc, static_cast<const __nv_bfloat16*>(g.bias),
                                               static_cast<const __nv_bfloat16*>(g.residual), g.m, g.n, g.k, g.act);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.m == 0 || g.n == 0) return cudaSuccess;
  return run_gemm<256, 4>(g, stream);
}

}  // namespace cora
