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
//   warps 2..5  : epilogue, one TMEM lane quadrant each: tcgen05.ld -> +bias (smem) -> act ->
//                 +residual (TMA-loaded into the swizzled staging buffer) -> bf16 in place -> TMA
//                 store (per warp, 32 rows x 64 cols per chunk)
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

template <int BN, int STAGES, int EPI_BUFS>
struct GemmSmem {
  static constexpr int kChunks = BN / BK;          // 64-column epilogue chunks per tile
  static constexpr int kBufs = EPI_BUFS;           // staging buffers per epilogue warp
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + STAGES * kABytes;
  static constexpr int kOffC = kOffB + STAGES * kBBytes;  // per warp: kBufs staging buffers
  static constexpr int kOffBias = kOffC + kEpiWarps * kBufs * kEpiBufBytes;  // per warp: BN bf16
  static constexpr int kOffBar = kOffBias + kEpiWarps * BN * 2;
  // full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2], res[kEpiWarps][kBufs], tmem ptr
  static constexpr int kNumBars = 2 * STAGES + 4 + kEpiWarps * kBufs;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  static constexpr int kAlloc = kBytes;
  static constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
};

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float apply_act(float x, int act) {
  if (act == CORA_ACT_RELU) return fmaxf(x, 0.f);
  if (act == CORA_ACT_GELU_ERF) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
  return x;
}

// RESIDUAL: the residual tile of chunk c is TMA-loaded into staging buffer c % EPI_BUFS as soon as that
// buffer is free (all of them at tile start when EPI_BUFS >= BN/64) and the output is written over it in
// place; otherwise the EPI_BUFS buffers rotate as plain output staging.
template <int BN, int STAGES, int EPI_BUFS, bool RESIDUAL>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                        const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_r,
                        const __nv_bfloat16* __restrict__ bias, int32_t has_residual, int32_t M, int32_t N,
                        int32_t K, int32_t act) {
  using S = GemmSmem<BN, STAGES, EPI_BUFS>;
  // SWIZZLE_128B atoms need 1024-B alignment; the dynamic smem window is declared so aligned
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* res_bar = tmem_empty + 2;  // [kEpiWarps][kBufs]
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(res_bar + kEpiWarps * S::kBufs);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int m_blocks = (M + BM - 1) / BM;
  const int n_blocks = (N + BN - 1) / BN;
  const int num_tiles = m_blocks * n_blocks;
  const int k_blocks = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_c);
    if (has_residual) tma_prefetch_desc(&tm_r);
    for (int i = 0; i < kEpiWarps * S::kBufs; ++i) mbar_init(&res_bar[i], 1);
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
    // Per warp: 32 rows (its TMEM lane quadrant) x BN columns in kChunks chunks of 64.  Chunk c has its
    // own 4 KB swizzled smem buffer: the residual tile is TMA-loaded into it at the start of the tile,
    // the output is written over it in place and TMA-stored from it (clipped at M and N).
    const uint32_t q = warp & 3;  // TMEM lane quadrant accessible to this warp
    const uint32_t ew = warp - 2;
    uint8_t* cbuf = smem + S::kOffC + ew * S::kBufs * kEpiBufBytes;
    __nv_bfloat16* sbias = reinterpret_cast<__nv_bfloat16*>(smem + S::kOffBias + ew * BN * 2);
    uint64_t* rbar = res_bar + ew * S::kBufs;
    int acc = 0;
    uint32_t acc_phase = 0, res_phase = 0;  // res_phase: one parity bit per staging-buffer barrier
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int m0 = (t / n_blocks) * BM, n0 = (t % n_blocks) * BN;
      const int row0 = m0 + q * 32;
      const int n_chunks = min(BN, N - n0 + BK - 1) / BK;  // 64-col chunks that intersect [0, N)
      if (RESIDUAL) {
        // the previous tile's stores must have finished reading the staging buffers
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
      }
      if (RESIDUAL && lane == 0) {
        for (int c = 0; c < n_chunks && c < S::kBufs; ++c) {
          mbar_arrive_expect_tx(&rbar[c], kEpiBufBytes);
          tma_load_2d(cbuf + c * kEpiBufBytes, &tm_r, &rbar[c], n0 + c * BK, row0);
        }
      }
      // bias of this tile's columns -> smem (one 16-B load per lane), read back as broadcasts
      for (int g = lane; g < BN / 8; g += 32) {
        uint4 bw = make_uint4(0u, 0u, 0u, 0u);
        if (bias != nullptr && n0 + g * 8 < N) bw = __ldg(reinterpret_cast<const uint4*>(bias + n0 + g * 8));
        *reinterpret_cast<uint4*>(sbias + g * 8) = bw;
      }
      __syncwarp();
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < n_chunks; ++c) {
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
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(sbias + c * BK);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t b2 = bw[j];
          v[2 * j] = __uint_as_float(r[2 * j]) + bf16_lo(b2);
          v[2 * j + 1] = __uint_as_float(r[2 * j + 1]) + bf16_hi(b2);
        }
        if (act != CORA_ACT_NONE) {
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = apply_act(v[j], act);
        }
        uint8_t* buf = cbuf + (c % S::kBufs) * kEpiBufBytes;
        if (!RESIDUAL) {
          // buffer (c % kBufs) was last read by the store issued kBufs chunks ago
          if (lane == 0) tma_store_wait_read<S::kBufs - 1>();
          __syncwarp();
        }
        const uint32_t sbase = smem_u32(buf);
        if (RESIDUAL) {
          const int j = c % S::kBufs;
          mbar_wait(&rbar[j], (res_phase >> j) & 1u);
          res_phase ^= 1u << j;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            uint32_t w0, w1, w2, w3;
            ld_shared_v4(sbase + sw128_offset(lane, ch), w0, w1, w2, w3);
            const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              v[ch * 8 + 2 * i] += bf16_lo(w[i]);
              v[ch * 8 + 2 * i + 1] += bf16_hi(w[i]);
            }
          }
        }
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          st_shared_v4(sbase + sw128_offset(lane, ch), pack_bf16x2(v[ch * 8 + 0], v[ch * 8 + 1]),
                       pack_bf16x2(v[ch * 8 + 2], v[ch * 8 + 3]), pack_bf16x2(v[ch * 8 + 4], v[ch * 8 + 5]),
                       pack_bf16x2(v[ch * 8 + 6], v[ch * 8 + 7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tm_c, buf, n0 + c * BK, row0);
          tma_store_commit();
          if (RESIDUAL && c + S::kBufs < n_chunks) {
            // refill this buffer with the residual of chunk c + kBufs once the store has read it
            tma_store_wait_read<0>();
            mbar_arrive_expect_tx(&rbar[c % S::kBufs], kEpiBufBytes);
            tma_load_2d(buf, &tm_r, &rbar[c % S::kBufs], n0 + (c + S::kBufs) * BK, row0);
          }
        }
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

template <int BN, int STAGES, int EPI_BUFS, bool RESIDUAL>
cudaError_t run_gemm(const GemmArgs& g, cudaStream_t stream) {
  using S = GemmSmem<BN, STAGES, EPI_BUFS>;
  CUtensorMap ta, tb, tc, tr;
  if (!make_tmap_2d_bf16(&ta, g.a, g.k, g.m, static_cast<uint64_t>(g.k) * 2, BK, BM, true) ||
      !make_tmap_2d_bf16(&tb, g.b, g.k, g.n, static_cast<uint64_t>(g.k) * 2, BK, BN, true) ||
      !make_tmap_2d_bf16(&tc, g.c, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
    return cudaErrorInvalidValue;
  if (g.residual != nullptr) {
    if (!make_tmap_2d_bf16(&tr, g.residual, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
      return cudaErrorInvalidValue;
  } else {
    tr = tc;  // unused
  }
  auto kern = gemm_bf16_tn_kernel<BN, STAGES, EPI_BUFS, RESIDUAL>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN);
  const int grid = tiles < device_sm_count() ? tiles : device_sm_count();
  kern<<<grid, kThreads, S::kAlloc, stream>>>(ta, tb, tc, tr, static_cast<const __nv_bfloat16*>(g.bias),
                                               g.residual != nullptr ? 1 : 0, g.m, g.n, g.k, g.act);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.m == 0 || g.n == 0) return cudaSuccess;
  // residual GEMMs: a short K loop (out-proj, K = d) is epilogue-bound -> 4 staging buffers per warp
  // with every residual chunk prefetched at tile start (3 stages, 210 KB); a long K loop (FF2,
  // K = d_ff) keeps 4 pipeline stages and refills 2 staging buffers just in time (226 KB)
  if (g.residual != nullptr) {
    if (g.k < 1024) return run_gemm<256, 3, 4, true>(g, stream);
    return run_gemm<256, 4, 2, true>(g, stream);
  }
  return run_gemm<256, 4, 2, false>(g, stream);
}

}  // namespace cora
