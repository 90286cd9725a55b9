// Steps a2 / a4 / a6 / a7: the packed ("vloop-fused") linear operators of the encoder layer.
//
// CoRa implements QKV Proj, Linear Proj, FF1 and FF2 as GEMMs over the fused token loop
// ("We use vloop fusion ... to implement the linear transformation
// operators ... with minimal padding"), with the bias / activation / residual add fused into
// the GEMM (Table ap_op_times).  CoRa additionally bulk-pads sum L to a
// multiple of 64; here no padding exists at all: the M tail is zero-filled
// by TMA on load and clipped by TMA on store.
//
// sm_100a design: persistent, warp-specialised, one CTA per SM; by default a CTA PAIR (cluster of
// 2, cta_group::2) computes 256 x BN tiles: each CTA holds 128 rows of A and BN/2 rows of B per
// stage, the leader CTA issues M=256 tcgen05.mma for both, and each CTA's TMEM receives its own
// 128 accumulator rows.  Per SM that is A + B/2 bytes per k-block instead of A + B -- the loads in
// flight (smem stages) cover the ~2 us TMA latency with half the bytes.
//   warp 0      : TMA producer (both CTAs; the leader's `full` barrier collects both CTAs' bytes)
//   warp 1      : TMEM allocator (both CTAs) + single-thread tcgen05.mma issuer (leader only)
//   warps 2..9  : epilogue, two warps per TMEM lane quadrant (column halves): tcgen05.ld -> +bias
//                 (smem) -> act -> +residual (TMA-loaded into the swizzled staging buffer) -> bf16 in
//                 place -> TMA store (32 rows x 64 cols per chunk)
//   TMEM holds two BN-column fp32 accumulators so the epilogue of tile i overlaps the main loop of
//   tile i+1.  A single m-block (M <= 128) runs the 1-CTA variant (cta_group::1, M=128).
#include <cuda_bf16.h>

#include <cstdint>

#include "cora_internal.h"
#include "ptx.cuh"

namespace cora {
namespace {

constexpr int BM = 128;  // accumulator rows per CTA
constexpr int BK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, each owning half of the tile's columns
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiRows = 32;                      // rows per epilogue warp
constexpr int kEpiBufBytes = kEpiRows * BK * 2;   // 4 KB staging buffer (32 rows x 128 B)

template <int BN, int STAGES, int CL>
struct GemmSmem {
  static constexpr int kChunks = BN / BK;             // 64-column epilogue chunks per tile
  static constexpr int kWarpCols = BN / 2;            // columns per epilogue warp
  static constexpr int kBufs = kWarpCols / BK;        // staging buffers per epilogue warp (one per chunk)
  static constexpr int kABytes = BM * BK * 2;         // this CTA's A rows
  static constexpr int kBBytes = (BN / CL) * BK * 2;  // this CTA's share of the B tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + STAGES * kABytes;
  static constexpr int kOffC = kOffB + STAGES * kBBytes;  // per warp: kBufs staging buffers
  static constexpr int kOffBias = kOffC + kEpiWarps * kBufs * kEpiBufBytes;  // per warp: kWarpCols bf16
  static constexpr int kOffBar = kOffBias + kEpiWarps * kWarpCols * 2;
  // full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2], res[kEpiWarps][kBufs], tmem ptr
  static constexpr int kNumBars = 2 * STAGES + 4 + kEpiWarps * kBufs;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  static constexpr int kAlloc = kBytes;
  static constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static_assert(kBytes <= 232448, "shared memory budget");
};

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float apply_act(float x, int act) {
  if (act == CORA_ACT_RELU) return fmaxf(x, 0.f);
  if (act == CORA_ACT_GELU_ERF) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
  return x;
}

// Epilogue: warp (quadrant q, half hf) owns rows [32 q, 32 q + 32) x columns [hf BN/2, (hf+1) BN/2) of the
// CTA's accumulator, one 4 KB staging buffer per 64-column chunk.  RESIDUAL: the residual chunks are
// TMA-loaded into the staging buffers at tile start and the output is written over them in place.
// CL: 1 = one CTA computes a 128 x BN tile (cta_group::1); 2 = a CTA pair computes a 256 x BN tile
// (cta_group::2), rank r owning rows [128 r, 128 r + 128) of it.
template <int BN, int STAGES, bool RESIDUAL, int CL>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                        const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_r,
                        const __nv_bfloat16* __restrict__ bias, int32_t M, int32_t N, int32_t K, int32_t act) {
  using S = GemmSmem<BN, STAGES, CL>;
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
  const int k_blocks = (K + BK - 1) / BK;
  // work units: 128-row tiles (CL = 1) or 256-row tile pairs (CL = 2), strided over CTAs / clusters
  const uint32_t rank = CL > 1 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit0 = CL > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int unit_step = CL > 1 ? static_cast<int>(num_clusters_x()) : static_cast<int>(gridDim.x);
  const int num_units = ((m_blocks + CL - 1) / CL) * n_blocks;
  auto unit_m0 = [&](int u) { return ((u / n_blocks) * CL + static_cast<int>(rank)) * BM; };
  auto unit_n0 = [&](int u) { return (u % n_blocks) * BN; };
  constexpr uint16_t kPairMask = (1u << CL) - 1u;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_c);
    if (RESIDUAL) tma_prefetch_desc(&tm_r);
    for (int i = 0; i < kEpiWarps * S::kBufs; ++i) mbar_init(&res_bar[i], 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // (leader) one expect_tx arrive; both CTAs' bytes complete it
      mbar_init(&empty[s], 1);  // one (multicast) MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], kEpiWarps * CL);  // (leader) the epilogue warps of every CTA
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CL > 1)
      tmem_alloc_cg2<S::kTmemCols>(tmem_ptr);
    else
      tmem_alloc<S::kTmemCols>(tmem_ptr);
  }
  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();  // barrier inits visible cluster-wide before any remote complete_tx / arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_wait();  // the previous kernel's outputs (our A / residual) are complete and visible
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (every CTA)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit0; u < num_units; u += unit_step) {
        const int m0 = unit_m0(u), n0 = unit_n0(u);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + S::kOffA + stage * S::kABytes;
          uint8_t* sb = smem + S::kOffB + stage * S::kBBytes;
          if (CL > 1) {
            // both CTAs' A rows and B halves complete the LEADER's full barrier
            const uint32_t bar = mapa_shared(&full[stage], 0);
            if (leader) mbar_arrive_expect_tx(&full[stage], CL * S::kStageBytes);
            tma_load_2d_cg2(sa, &tm_a, bar, kb * BK, m0);
            tma_load_2d_cg2(sb, &tm_b, bar, kb * BK, n0 + static_cast<int>(rank) * (BN / CL));
          } else {
            mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
            tma_load_2d(sa, &tm_a, &full[stage], kb * BK, m0);
            tma_load_2d(sb, &tm_b, &full[stage], kb * BK, n0);
          }
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader, one thread)
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc_bf16(BM * CL, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = unit0; u < num_units; u += unit_step) {
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
            if (CL > 1)
              umma_bf16_ss_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else
              umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          // frees the smem stage (of every CTA of the pair) once these MMAs retire
          if (CL > 1)
            umma_commit_cg2_mcast(&empty[stage], kPairMask);
          else
            umma_commit(&empty[stage]);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        // accumulator ready for the epilogue of every CTA
        if (CL > 1)
          umma_commit_cg2_mcast(&tmem_full[acc], kPairMask);
        else
          umma_commit(&tmem_full[acc]);
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps (every CTA)
    const uint32_t q = warp & 3;  // TMEM lane quadrant accessible to this warp
    const uint32_t ew = warp - 2;
    const int hf = static_cast<int>(ew) / 4;  // column half of the tile
    uint8_t* cbuf = smem + S::kOffC + ew * S::kBufs * kEpiBufBytes;
    __nv_bfloat16* sbias = reinterpret_cast<__nv_bfloat16*>(smem + S::kOffBias + ew * S::kWarpCols * 2);
    uint64_t* rbar = res_bar + ew * S::kBufs;
    const uint32_t tmem_empty_lead0 = CL > 1 ? mapa_shared(&tmem_empty[0], 0) : 0u;
    int acc = 0;
    uint32_t acc_phase = 0, res_phase = 0;
    for (int u = unit0; u < num_units; u += unit_step) {
      const int m0 = unit_m0(u);
      const int nw = unit_n0(u) + hf * S::kWarpCols;  // first column of this warp
      const int row0 = m0 + q * 32;
      // 64-col chunks of this warp that intersect [0, N)
      const int n_chunks = N > nw ? min(S::kBufs, (N - nw + BK - 1) / BK) : 0;
      // the previous tile's stores must have finished reading the staging buffers
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      if (RESIDUAL && lane == 0) {
        for (int c = 0; c < n_chunks; ++c) {
          mbar_arrive_expect_tx(&rbar[c], kEpiBufBytes);
          tma_load_2d(cbuf + c * kEpiBufBytes, &tm_r, &rbar[c], nw + c * BK, row0);
        }
      }
      // bias of this warp's columns -> smem (one 16-B load per lane), read back as broadcasts
      for (int g = lane; g < S::kWarpCols / 8; g += 32) {
        uint4 bw = make_uint4(0u, 0u, 0u, 0u);
        if (bias != nullptr && nw + g * 8 < N) bw = __ldg(reinterpret_cast<const uint4*>(bias + nw + g * 8));
        *reinterpret_cast<uint4*>(sbias + g * 8) = bw;
      }
      __syncwarp();
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < S::kBufs; ++c) {
        if (c < n_chunks) {
          uint32_t r[64];
          const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN + hf * S::kWarpCols + c * BK;
          CORA_TMEM_LD_32X32B_X32(taddr, r);
          CORA_TMEM_LD_32X32B_X32(taddr + 32, (r + 32));
          tmem_ld_wait();
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
          uint8_t* buf = cbuf + c * kEpiBufBytes;
          const uint32_t sbase = smem_u32(buf);
          if (RESIDUAL) {
            mbar_wait(&rbar[c], (res_phase >> c) & 1u);
            res_phase ^= 1u << c;
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
            tma_store_2d(&tm_c, buf, nw + c * BK, row0);
            tma_store_commit();
          }
        }
        if (c == S::kBufs - 1) {
          // all TMEM reads of this accumulator are done: hand it back to the (leader's) MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CL > 1)
              mbar_arrive_cluster(tmem_empty_lead0 + acc * 8);
            else
              mbar_arrive(&tmem_empty[acc]);
          }
        }
      }
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();  // the peer may still complete_tx / arrive on this CTA's barriers until here
  else
    __syncthreads();
  if (warp == 1) {
    if (CL > 1)
      tmem_dealloc_cg2<S::kTmemCols>(tmem_base);
    else
      tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

template <int BN, int STAGES, bool RESIDUAL, int CL>
cudaError_t run_gemm(const GemmArgs& g, cudaStream_t stream) {
  using S = GemmSmem<BN, STAGES, CL>;
  CUtensorMap ta, tb, tc, tr;
  if (!make_tmap_2d_bf16(&ta, g.a, g.k, g.m, static_cast<uint64_t>(g.k) * 2, BK, BM, true) ||
      !make_tmap_2d_bf16(&tb, g.b, g.k, g.n, static_cast<uint64_t>(g.k) * 2, BK, BN / CL, true) ||
      !make_tmap_2d_bf16(&tc, g.c, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
    return cudaErrorInvalidValue;
  if (RESIDUAL) {
    if (!make_tmap_2d_bf16(&tr, g.residual, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
      return cudaErrorInvalidValue;
  } else {
    tr = tc;  // unused
  }
  auto kern = gemm_bf16_tn_kernel<BN, STAGES, RESIDUAL, CL>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int m_blocks = (g.m + BM - 1) / BM, n_blocks = (g.n + BN - 1) / BN;
  const int units = ((m_blocks + CL - 1) / CL) * n_blocks;
  const int max_units = device_sm_count() / CL;
  const int grid = (units < max_units ? units : max_units) * CL;
  return launch_pdl(kern, dim3(grid), dim3(kThreads), S::kAlloc, stream, CL, ta, tb, tc, tr,
                    static_cast<const __nv_bfloat16*>(g.bias), g.m, g.n, g.k, g.act);
}

}  // namespace

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.m == 0 || g.n == 0) return cudaSuccess;
  const bool pair = ((g.m + BM - 1) / BM) >= 2;  // a single m-block runs on one CTA
  // smem per SM: CTA pair -> 32 KB per stage (A 16 KB + half of B) -> 5 stages; 1 CTA -> 48 KB -> 3
  if (g.residual != nullptr)
    return pair ? run_gemm<256, 5, true, 2>(g, stream) : run_gemm<256, 3, true, 1>(g, stream);
  return pair ? run_gemm<256, 5, false, 2>(g, stream) : run_gemm<256, 3, false, 1>(g, stream);
}

}  // namespace cora
