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
//   warps 2..9  : epilogue (2..17 for the staged LN), two (four) warps per TMEM lane quadrant: tcgen05.ld -> +bias
//                 (smem) -> act -> +residual (TMA-loaded into the swizzled staging buffer) -> bf16 in
//                 place -> TMA store (32 rows x 64 cols per chunk)
//   TMEM holds two BN-column fp32 accumulators so the epilogue of tile i overlaps the main loop of
//   tile i+1.  A single m-block (M <= 128) runs the 1-CTA variant (cta_group::1, M=128).
// The mainloop is bound by the bytes in flight (stages x stage bytes / TMA latency): non-residual GEMMs
// keep one reused staging buffer per epilogue warp and 6 stages.
// LN (N = 512, steps a4+a5 / a7+a8): two CTA pairs of one 4-CTA cluster hold the two 256-column halves
// of the same 256 rows and combine LayerNorm row statistics over DSMEM.  Short K (out-proj, bound by
// shared-memory bandwidth): residual TMA-staged, 4 stages, 16 epilogue warps (64 columns each).  Long K
// (FF2, mainloop-bound): LNREG -- row segments in registers, 32-B residual loads and output stores,
// 6 stages.  The LN kernels have no activation variants (one epilogue body),
// the plain GEMM takes the activation as a template parameter.
// PDL: the producer issues the weight (B) tiles of its first stages before griddepcontrol.wait -- no
// kernel of the layer writes the weights -- and A / residual only after it.
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "cora_internal.h"
#include "prelude_impl.cuh"
#include "ptx.cuh"

#ifdef CORA_GEMM_TRACE
// profiling build only: %globaltimer stamps of the phases of every CTA of the last launch
__device__ unsigned long long g_gemm_trace[2048 * 16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// CORA_GEMM_TRACE = 1: FF2 + LN2 (register LN), 2: out-proj + LN1 (staged LN), 3: plain GEMMs (last: FF1)
#define GTRACE_ON ((CORA_GEMM_TRACE == 1 && LNREG) || (CORA_GEMM_TRACE == 2 && LN && !LNREG) || (CORA_GEMM_TRACE == 3 && !LN))
#define GTRACE(k) (GTRACE_ON ? (void)(g_gemm_trace[blockIdx.x * 16 + (k)] = gtime()) : (void)0)
extern "C" int cora_debug_gemm_trace(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_gemm_trace, sizeof(unsigned long long) * (n < 2048 * 16 ? n : 2048 * 16)) ==
                 cudaSuccess ? 0 : 1;
}
// per-CTA wait totals (clock64 cycles) of the traced launch: [0] producer waiting for free stages, [1] MMA
// waiting for loaded stages, [2] MMA waiting for a free accumulator, [3] MMA role total, [4] epilogue warp 0
// waiting for its accumulator, [5] epilogue warp 0 total, [6] units of this CTA
__device__ long long g_gemm_waits[2048][8];
extern "C" int cora_debug_gemm_waits(long long* host) {
  return cudaMemcpyFromSymbol(host, g_gemm_waits, sizeof(g_gemm_waits)) == cudaSuccess ? 0 : 1;
}
#define GW_DECL long long gw_t0 = clock64(), gw_w = 0, gw_w2 = 0, gw_n = 0
#define GW_WAIT(acc, stmt) do { const long long t_ = clock64(); stmt; acc += clock64() - t_; } while (0)
#define GW_STORE(i, v) do { if (GTRACE_ON) g_gemm_waits[blockIdx.x][i] = (v); } while (0)
#else
#define GTRACE(k) ((void)0)
#define GW_DECL
#define GW_WAIT(acc, stmt) stmt
#define GW_STORE(i, v) ((void)0)
#endif

CORA_KSPAN_DEFINE(gemm)

namespace cora {
namespace {

constexpr int BM = 128;  // accumulator rows per CTA
constexpr int BK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, each owning half of the tile's columns
#ifndef CORA_LN_EW
#define CORA_LN_EW 16
#endif
// epilogue warps: 8, or 16 (four per quadrant, a quarter of the columns each) for the staged-residual LN
// epilogue of the short-K out-projection, which is epilogue-bound
template <bool LN, bool LNREG>
constexpr int epi_warps() { return (LN && !LNREG) ? CORA_LN_EW : kEpiWarps; }
constexpr int kEpiRows = 32;                      // rows per epilogue warp
constexpr int kEpiBufBytes = kEpiRows * BK * 2;   // 4 KB staging buffer (32 rows x 128 B)

// NBUF: staging buffers per epilogue warp -- one per 64-column chunk when a residual is TMA-prefetched into
// them (RESIDUAL / LN), else one reused buffer, which frees 32 KB for a sixth pipeline stage (the mainloop
// is bound by the bytes in flight: stages x stage bytes / TMA latency)
template <int BN, int STAGES, int CL, bool LN, int NBUF = 2, int EW = kEpiWarps>
struct GemmSmem {
  static constexpr int kChunks = BN / BK;             // 64-column epilogue chunks per tile
  static constexpr int kWarpCols = BN * 4 / EW;       // columns per epilogue warp
  static constexpr int kBufs = kWarpCols / BK;        // staging buffers per epilogue warp (one per chunk)
  static constexpr int kABytes = BM * BK * 2;         // this CTA's A rows
  // this CTA's share of the B tile: half of it in a CTA pair (cta_group::2); all of it for one CTA or a
  // DUO (LN with CL = 2: two single CTAs holding the two column halves of the same 128 rows)
  static constexpr int kBBytes = ((CL == 4 || (CL == 2 && !LN)) ? BN / 2 : BN) * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + STAGES * kABytes;
  static constexpr int kNBuf = NBUF;
  static constexpr int kOffC = kOffB + STAGES * kBBytes;  // per warp: NBUF staging buffers
  static constexpr int kOffBias = kOffC + EW * NBUF * kEpiBufBytes;  // per warp: kWarpCols bf16
  // LN mode: this CTA's column half of gamma / beta (fp32), per-warp row partials and the partner's
  static constexpr int kOffGamma = kOffBias + EW * kWarpCols * 2;
  static constexpr int kOffBeta = kOffGamma + (LN ? BN * 4 : 0);
  static constexpr int kOffPart = kOffBeta + (LN ? BN * 4 : 0);  // float2 [2 acc][EW / 4 groups][128 rows]
  static constexpr int kOffRecv = kOffPart + (LN ? 2 * (EW / 4) * BM * 8 : 0);  // float2 [2 acc][128 rows]
  static constexpr int kOffBar = kOffRecv + (LN ? 2 * BM * 8 : 0);
  // full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2], res[EW][kBufs], xch[2], tmem ptr
  static constexpr int kNumBars = 2 * STAGES + 4 + EW * kBufs + 2;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  static constexpr int kAlloc = kBytes;
  static constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static_assert(kBytes <= 232448, "shared memory budget");
};

// LayerNorm row statistics of the fused epilogues as (mean, M2 = sum (v - mean)^2) pairs, merged across
// column segments and CTAs with the pairwise formula of Chan et al.: no E[v^2] - mean^2 cancellation, so
// rows whose |mean| is large against their spread keep an accurate variance.
// Segment of n values with shifted sums s1 = sum (v - K), s2 = sum (v - K)^2:
__device__ __forceinline__ float2 seg_moments(float K, float s1, float s2, float n) {
  return make_float2(K + s1 / n, fmaxf(s2 - s1 * (s1 / n), 0.f));
}
// Merge a (na = k * n values) with b (n values); k = 1 (equal halves) by default.  For k = 1 the result is
// symmetric in a and b (both CTAs of a row compute bitwise the same statistics).
__device__ __forceinline__ float2 merge_moments(float2 a, float2 b, float n, int k = 1) {
  const float na = n * static_cast<float>(k), nc = na + n;
  const float d = b.x - a.x;
  if (k == 1) return make_float2((a.x + b.x) * 0.5f, (a.y + b.y) + d * d * (n * 0.5f));
  return make_float2(a.x + d * (n / nc), (a.y + b.y) + d * d * (na * n / nc));
}

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
// (cta_group::2), pair rank r owning rows [128 r, 128 r + 128) of it; 4 (LN only) = two CTA pairs compute
// the two BN-column halves of the same 256 rows (N = 2 BN), so every row of the output lives in one
// cluster and its LayerNorm statistics are combined across the pairs (section "LN epilogue" below).
// DUO (LN with CL = 2): two single CTAs (cta_group::1) of a 2-CTA cluster compute the two BN-column halves
// of the same 128 rows, so the LN GEMM tiles all 148 SMs (clusters of 4 strand 16 at GPC boundaries) in
// units of half the rows; each CTA's epilogue is the pair CTA's (the same 128 x BN accumulator and row
// segments), only the statistics partner differs (rank ^ 1 instead of rank ^ 2).
template <int BN, int STAGES, bool RESIDUAL, int CL, bool LN, bool LNREG, int ACT>
__global__ void __launch_bounds__(64 + 32 * epi_warps<LN, LNREG>(), 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                        const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_r,
                        const __nv_bfloat16* __restrict__ bias, const float* __restrict__ ln_gamma,
                        const float* __restrict__ ln_beta, float ln_eps, const __nv_bfloat16* __restrict__ res_ptr,
                        __nv_bfloat16* __restrict__ out_ptr, int32_t M, int32_t N, int32_t K, int32_t act,
                        int32_t late_wait, const PreludeArgs pre) {
  // staging buffers per epilogue warp: the residual is TMA-prefetched into one per chunk (RESIDUAL,
  // staged LN), or the row segment lives in registers (LNREG) / there is no residual: one reused buffer
  constexpr int EW = epi_warps<LN, LNREG>();
  using S = GemmSmem<BN, STAGES, CL, LN, (RESIDUAL && !LNREG) ? BN * 4 / EW / BK : (LNREG ? 0 : 1), EW>;
  static_assert(!LN || ((CL == 4 || CL == 2) && RESIDUAL), "the LayerNorm epilogue runs on 2 CTA pairs or a DUO with a residual");
  // SWIZZLE_128B atoms need 1024-B alignment; the dynamic smem window is declared so aligned
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* res_bar = tmem_empty + 2;  // [EW][kBufs]
  uint64_t* xch_bar = res_bar + EW * S::kBufs;  // [2 acc] partner's row partials landed (LN)
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(xch_bar + 2);
  if (threadIdx.x == 0) GTRACE(0);
  constexpr int kSpanSlot = LN ? (LNREG ? 5 : 3) : (ACT != CORA_ACT_NONE ? 4 : 2);
  KSPAN_ENTRY(gemm, kSpanSlot);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int m_blocks = (M + BM - 1) / BM;
  const int n_blocks = (N + BN - 1) / BN;
  const int k_blocks = (K + BK - 1) / BK;
  // work units: 128-row tiles (CL = 1), 256-row tiles of one BN-column block (CL = 2) or 256 full rows
  // (CL = 4), strided over CTAs / clusters
  constexpr bool DUO = LN && CL == 2;        // two single CTAs (cta_group::1), one per column half
  constexpr bool PAIR = CL > 1 && !DUO;      // cta_group::2 CTA pairs
  constexpr bool CLUSTER = CL > 1;
  const uint32_t rank = CLUSTER ? cluster_ctarank() : 0u;
  const uint32_t prank = PAIR ? (rank & 1u) : 0u;       // rank inside the CTA pair
  const uint32_t lead_rank = PAIR ? (rank & ~1u) : rank;  // the pair's leader (issues the MMAs)
  const int half = LN ? static_cast<int>(DUO ? rank : rank >> 1) : 0;  // LN: which BN-column half of the rows
  const uint32_t ln_partner = DUO ? (rank ^ 1u) : (rank ^ 2u);  // LN: the CTA holding the other half
  const bool leader = prank == 0;
  const int unit0 = CLUSTER ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int unit_step = CLUSTER ? static_cast<int>(num_clusters_x()) : static_cast<int>(gridDim.x);
  const int nb_units = LN ? 1 : n_blocks;
  const int num_units = ((m_blocks + (PAIR ? 1 : 0)) / (PAIR ? 2 : 1)) * nb_units;
  auto unit_m0 = [&](int u) { return ((u / nb_units) * (PAIR ? 2 : 1) + static_cast<int>(prank)) * BM; };
  auto unit_n0 = [&](int u) { return LN ? half * BN : (u % nb_units) * BN; };
  const uint16_t kPairMask = static_cast<uint16_t>(3u << lead_rank);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_c);
    if (RESIDUAL) tma_prefetch_desc(&tm_r);
    for (int i = 0; i < EW * S::kBufs; ++i) mbar_init(&res_bar[i], 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // (leader) one expect_tx arrive; both CTAs' bytes complete it
      mbar_init(&empty[s], 1);  // one (multicast) MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], EW * (PAIR ? 2 : 1));  // (leader) the epilogue warps of both CTAs
      mbar_init(&xch_bar[a], 1);                               // LN: local arm + the partner's st.async bytes
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR)
      tmem_alloc_cg2<S::kTmemCols>(tmem_ptr);
    else
      tmem_alloc<S::kTmemCols>(tmem_ptr);
  }
  tc_fence_before();
  if (CLUSTER)
    cluster_sync_all();  // barrier inits visible cluster-wide before any remote complete_tx / arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  // late_wait: the operands were complete before the previous kernel (the prelude) started, so wait for
  // that kernel only at the end -- this grid then still completes after it (its dependents see both)
  if (threadIdx.x == 0) GTRACE(1);
  // The weights (B) are never written by another kernel of the layer: the producer issues the B tiles of
  // its first stages before griddepcontrol.wait, so they are in flight while the previous kernel drains
  int pre_b = 0;
  if (warp == 0 && lane == 0 && unit0 < num_units) {
    pre_b = STAGES < k_blocks ? STAGES : k_blocks;
    const int n0 = unit_n0(unit0);
    for (int kb = 0; kb < pre_b; ++kb) {
      uint8_t* sb = smem + S::kOffB + kb * S::kBBytes;
      if (PAIR) {
        const uint32_t bar = mapa_shared(&full[kb], lead_rank);
        if (leader) mbar_arrive_expect_tx(&full[kb], 2 * S::kStageBytes);
        tma_load_2d_cg2(sb, &tm_b, bar, kb * BK, n0 + static_cast<int>(prank) * (BN / 2));
      } else {
        mbar_arrive_expect_tx(&full[kb], S::kStageBytes);
        tma_load_2d(sb, &tm_b, &full[kb], kb * BK, n0);
      }
    }
  }
  if (!late_wait) pdl_wait();  // the previous kernel's outputs (our A / residual) are complete and visible
  if (!late_wait) KSPAN_WAITED(gemm, kSpanSlot);
  if (threadIdx.x == 0) GTRACE(2);
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (every CTA)
    if (lane == 0) {
      GW_DECL;
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit0; u < num_units; u += unit_step) {
        const int m0 = unit_m0(u), n0 = unit_n0(u);
        for (int kb = 0; kb < k_blocks; ++kb) {
          const bool b_issued = u == unit0 && kb < pre_b;  // fresh stage, B already in flight
          if (!b_issued) GW_WAIT(gw_w, mbar_wait(&empty[stage], phase ^ 1));
          uint8_t* sa = smem + S::kOffA + stage * S::kABytes;
          uint8_t* sb = smem + S::kOffB + stage * S::kBBytes;
          if (PAIR) {
            // both CTAs' A rows and B halves complete the pair leader's full barrier
            const uint32_t bar = mapa_shared(&full[stage], lead_rank);
            if (leader && !b_issued) mbar_arrive_expect_tx(&full[stage], 2 * S::kStageBytes);
            tma_load_2d_cg2(sa, &tm_a, bar, kb * BK, m0);
            if (!b_issued) tma_load_2d_cg2(sb, &tm_b, bar, kb * BK, n0 + static_cast<int>(prank) * (BN / 2));
          } else {
            if (!b_issued) mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
            tma_load_2d(sa, &tm_a, &full[stage], kb * BK, m0);
            if (!b_issued) tma_load_2d(sb, &tm_b, &full[stage], kb * BK, n0);
          }
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
      GW_STORE(0, gw_w);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader, one thread)
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc_bf16(BM * (PAIR ? 2 : 1), BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      GW_DECL;
      for (int u = unit0; u < num_units; u += unit_step) {
        GW_WAIT(gw_w2, mbar_wait(&tmem_empty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          GW_WAIT(gw_w, mbar_wait(&full[stage], phase));
          if (u == unit0 && kb == 0) GTRACE(3);
          if (u == unit0 && kb == k_blocks / 2) GTRACE(4);
          if (u == unit0 && kb == k_blocks - 1) GTRACE(5);
#if defined(CORA_GEMM_TRACE)
          if (u == unit0 + unit_step && kb == 0) GTRACE(13);
          if (u == unit0 + unit_step && kb == k_blocks - 1) GTRACE(14);
#endif
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + S::kOffA + stage * S::kABytes);
          const uint32_t b_addr = smem_u32(smem + S::kOffB + stage * S::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(b_addr + k * 32, 16, 1024);
            if (PAIR)
              umma_bf16_ss_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else
              umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          // frees the smem stage (of every CTA of the pair) once these MMAs retire
          if (PAIR)
            umma_commit_cg2_mcast(&empty[stage], kPairMask);
          else
            umma_commit(&empty[stage]);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        // accumulator ready for the epilogue of every CTA
        if (PAIR)
          umma_commit_cg2_mcast(&tmem_full[acc], kPairMask);
        else
          umma_commit(&tmem_full[acc]);
        if (++acc == 2) acc = 0, acc_phase ^= 1;
#ifdef CORA_GEMM_TRACE
        ++gw_n;
#endif
      }
      GW_STORE(1, gw_w);
      GW_STORE(2, gw_w2);
#ifdef CORA_GEMM_TRACE
      GW_STORE(3, clock64() - gw_t0);
      GW_STORE(6, gw_n);
#endif
    }
  } else if (LN && LNREG) {
    // ------------------------------------------------------------ LN epilogue (every CTA)
    // Warp (q, hf) owns rows [32 q, 32 q + 32) x columns [hf 128, hf 128 + 128) of this CTA's BN-column
    // half; one thread = one row segment of 128 columns, held in REGISTERS (64 bf16 pairs) from the
    // residual load to the normalised store, so the epilogue needs a single 4 KB staging buffer per warp
    // (for the TMA store) and the shared memory this frees holds a fifth pipeline stage.
    // The residual segment is loaded (16-B global loads) before the accumulator is waited for; pass 1:
    // v = bf16(acc + bias + residual) in place (the rounding point of the unfused path, Y1 / Y2) and per-row
    // (sum v, sum v^2); the two column quarters of a row are combined in smem, the CTA partial is sent with
    // st.async to the CTA holding the row's other column half (rank ^ 2), whose bytes complete this CTA's
    // xch_bar; pass 2: (v - mean) * rstd * gamma + beta (reading c2/c3: post-LN, biased variance) ->
    // staging -> TMA store, chunk by chunk.
    const uint32_t q = warp & 3;
    const uint32_t ew = warp - 2;
    const int hf = static_cast<int>(ew) / 4;
    const int row = static_cast<int>(q) * 32 + static_cast<int>(lane);  // accumulator row of this thread
    uint8_t* cbuf = smem + S::kOffC + ew * S::kNBuf * kEpiBufBytes;
    __nv_bfloat16* sbias = reinterpret_cast<__nv_bfloat16*>(smem + S::kOffBias);  // [BN] this CTA's half
    float* sgamma = reinterpret_cast<float*>(smem + S::kOffGamma);
    float* sbeta = reinterpret_cast<float*>(smem + S::kOffBeta);
    float2* part = reinterpret_cast<float2*>(smem + S::kOffPart);  // [acc][hf][row]
    float2* recv = reinterpret_cast<float2*>(smem + S::kOffRecv);  // [acc][row]
    const uint32_t tmem_empty_lead0 = mapa_shared(&tmem_empty[0], lead_rank);
    const uint32_t partner = ln_partner;
    const uint32_t recv_remote0 = mapa_shared(recv, partner);
    const uint32_t xch_remote0 = mapa_shared(&xch_bar[0], partner);
    const int n_half0 = half * BN;
    // this CTA's column half of bias / gamma / beta, once
    for (int c = static_cast<int>(threadIdx.x) - 64; c < BN; c += 32 * EW) {
      sbias[c] = bias != nullptr ? bias[n_half0 + c] : __float2bfloat16_rn(0.f);
      sgamma[c] = ln_gamma[n_half0 + c];
      sbeta[c] = ln_beta[n_half0 + c];
    }
    named_bar_sync(1, 32 * EW);
    const float inv_n = 1.0f / static_cast<float>(N);
    constexpr int kSeg = S::kWarpCols;  // 128 columns per thread
    const bool v8_ok = ((reinterpret_cast<uintptr_t>(res_ptr) | reinterpret_cast<uintptr_t>(out_ptr)) & 31u) == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit0; u < num_units; u += unit_step) {
      const int m0 = unit_m0(u);
      const int nw = n_half0 + hf * kSeg;
      const int row0 = m0 + static_cast<int>(q) * 32;
      const int grow = m0 + row;  // global row of this thread
      uint32_t vv[kSeg / 2];      // the row segment as bf16 pairs: residual, then v
      {
        // 32-B loads: each lane reads whole sectors of its row (residual base 32-B aligned; else 16-B loads)
        const __nv_bfloat16* src = res_ptr + static_cast<size_t>(grow) * N + nw;
#pragma unroll
        for (int g = 0; g < kSeg / 16; ++g) {
          uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          if (grow < M) {
            if (v8_ok) {
              ld_global_nc_v8(src + g * 16, w);
            } else {
              const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + g * 16));
              const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + g * 16 + 8));
              w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
            }
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) vv[8 * g + e] = w[e];
        }
      }
      if (ew == 0 && lane == 0) mbar_arrive_expect_tx(&xch_bar[acc], BM * 8);  // the partner's 128 row partials
      mbar_wait(&tmem_full[acc], acc_phase);
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(6);
      if (u != unit0 && ew == 0 && lane == 0 && (u - unit0) / unit_step <= 2) GTRACE(10 + (u - unit0) / unit_step);
      tc_fence_after();
      // shifted sums (shift K = the segment's first value): no cancellation when |mean| >> sigma; the pair
      // of columns of a bf16x2 word on the paired fp32 pipe (FADD2 / FFMA2)
      float2 s1v = make_float2(0.f, 0.f), s2v = s1v, nK = s1v;
#pragma unroll
      for (int c = 0; c < kSeg / BK; ++c) {
        uint32_t r[64];
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN + hf * kSeg + c * BK;
        CORA_TMEM_LD_32X32B_X32(taddr, r);
        CORA_TMEM_LD_32X32B_X32(taddr + 32, (r + 32));
        tmem_ld_wait();
        if (c == kSeg / BK - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_lead0 + acc * 8);
        }
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(sbias + hf * kSeg + c * BK);
#pragma unroll
        for (int p2 = 0; p2 < 32; ++p2) {
          const uint32_t b2 = bw[p2];
          const float v0 = __uint_as_float(r[2 * p2]) + bf16_lo(b2);
          const float v1 = __uint_as_float(r[2 * p2 + 1]) + bf16_hi(b2);
          const uint32_t rw = vv[c * 32 + p2];
          const uint32_t o = pack_bf16x2(v0 + bf16_lo(rw), v1 + bf16_hi(rw));
          vv[c * 32 + p2] = o;
          const float2 y = make_float2(bf16_lo(o), bf16_hi(o));  // statistics of the rounded values
          if (c == 0 && p2 == 0) nK = make_float2(-y.x, -y.x);
          const float2 dv = __fadd2_rn(y, nK);
          s1v = __fadd2_rn(s1v, dv);
          s2v = __ffma2_rn(dv, dv, s2v);
        }
      }
      float2* pa = part + acc * 2 * BM;
      pa[hf * BM + row] = seg_moments(-nK.x, s1v.x + s1v.y, s2v.x + s2v.y, static_cast<float>(kSeg));
      named_bar_sync(1, 32 * EW);  // both column quarters of every row are in `part`
      const float2 cm = merge_moments(pa[row], pa[BM + row], static_cast<float>(kSeg));  // this CTA's 256 columns
      if (hf == 0)
        st_async_v2f32(recv_remote0 + (acc * BM + row) * 8, cm.x, cm.y, xch_remote0 + acc * 8);
      mbar_wait(&xch_bar[acc], acc_phase);
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(7);
      const float2 rm = merge_moments(cm, recv[acc * BM + row], static_cast<float>(N / 2));
      const float mean = rm.x;
      const float rstd = rsqrtf(rm.y * inv_n + ln_eps);
      // straight from registers to the row in global memory (16-B stores; no staging buffer, whose 32 KB
      // hold a sixth pipeline stage instead)
      __nv_bfloat16* dst = out_ptr + static_cast<size_t>(grow) * N + nw;
#pragma unroll
      for (int c = 0; c < kSeg / BK; ++c) {
        const float* gm = sgamma + hf * kSeg + c * BK;
        const float* bt = sbeta + hf * kSeg + c * BK;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {  // 16 columns = one 32-B sector per store
          uint32_t w[8];
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) {
            const int col = ch * 16 + 2 * i2;
            const uint32_t vw = vv[c * 32 + ch * 8 + i2];
            w[i2] = pack_bf16x2((bf16_lo(vw) - mean) * rstd * gm[col] + bt[col],
                                (bf16_hi(vw) - mean) * rstd * gm[col + 1] + bt[col + 1]);
          }
          if (grow < M) {
            if (v8_ok) {
              st_global_v8(dst + c * BK + ch * 16, w);
            } else {
              uint4* d4 = reinterpret_cast<uint4*>(dst + c * BK + ch * 16);
              d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
              d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
          }
        }
      }
      (void)row0;
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(8);
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
  } else if (LN) {
    // ------------------------------------------------------------ LN epilogue, staged residual (every CTA)
    // Warp (q, hf) owns rows [32 q, 32 q + 32) x columns [hf 128, hf 128 + 128) of this CTA's BN-column
    // half.  pass 1: v = bf16(acc + bias + residual) into the staging buffers (the rounding point of
    // the unfused path, Y1 / Y2) and per-row (sum v, sum v^2); the two column quarters of a row are
    // combined in smem, the CTA partial is sent with st.async to the CTA holding the row's other
    // column half (rank ^ 2), whose bytes complete this CTA's xch_bar; pass 2: normalise
    // (v - mean) * rstd * gamma + beta (reading c2/c3: post-LN, biased variance) in place, TMA store.
    const uint32_t q = warp & 3;
    const uint32_t ew = warp - 2;
    const int hf = static_cast<int>(ew) / 4;
    const int row = static_cast<int>(q) * 32 + static_cast<int>(lane);  // accumulator row of this thread
    uint8_t* cbuf = smem + S::kOffC + ew * S::kNBuf * kEpiBufBytes;
    uint64_t* rbar = res_bar + ew * S::kBufs;
    __nv_bfloat16* sbias = reinterpret_cast<__nv_bfloat16*>(smem + S::kOffBias);  // [BN] this CTA's half
    float* sgamma = reinterpret_cast<float*>(smem + S::kOffGamma);
    float* sbeta = reinterpret_cast<float*>(smem + S::kOffBeta);
    float2* part = reinterpret_cast<float2*>(smem + S::kOffPart);  // [acc][hf][row]
    float2* recv = reinterpret_cast<float2*>(smem + S::kOffRecv);  // [acc][row]
    const uint32_t tmem_empty_lead0 = mapa_shared(&tmem_empty[0], lead_rank);
    const uint32_t partner = ln_partner;
    const uint32_t recv_remote0 = mapa_shared(recv, partner);
    const uint32_t xch_remote0 = mapa_shared(&xch_bar[0], partner);
    const int n_half0 = half * BN;
    // this CTA's column half of bias / gamma / beta, once
    for (int c = static_cast<int>(threadIdx.x) - 64; c < BN; c += 32 * EW) {
      sbias[c] = bias != nullptr ? bias[n_half0 + c] : __float2bfloat16_rn(0.f);
      sgamma[c] = ln_gamma[n_half0 + c];
      sbeta[c] = ln_beta[n_half0 + c];
    }
    named_bar_sync(1, 32 * EW);
    const float inv_n = 1.0f / static_cast<float>(N);
    int acc = 0;
    uint32_t acc_phase = 0, res_phase = 0;
    for (int u = unit0; u < num_units; u += unit_step) {
      const int m0 = unit_m0(u);
      const int nw = n_half0 + hf * S::kWarpCols;
      const int row0 = m0 + static_cast<int>(q) * 32;
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < S::kBufs; ++c) {
          mbar_arrive_expect_tx(&rbar[c], kEpiBufBytes);
          tma_load_2d(cbuf + c * kEpiBufBytes, &tm_r, &rbar[c], nw + c * BK, row0);
        }
        if (ew == 0) mbar_arrive_expect_tx(&xch_bar[acc], BM * 8);  // the partner's 128 row partials
      }
      mbar_wait(&tmem_full[acc], acc_phase);
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(6);
      if (u != unit0 && ew == 0 && lane == 0 && (u - unit0) / unit_step <= 2) GTRACE(10 + (u - unit0) / unit_step);
      tc_fence_after();
      // shifted sums (shift K = the segment's first value): no cancellation when |mean| >> sigma; the pair
      // of columns of a bf16x2 word on the paired fp32 pipe (FADD2 / FFMA2)
      float2 s1v = make_float2(0.f, 0.f), s2v = s1v, nK = s1v;
#pragma unroll 1
      for (int c = 0; c < S::kBufs; ++c) {
        uint32_t r[64];
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN + hf * S::kWarpCols + c * BK;
        CORA_TMEM_LD_32X32B_X32(taddr, r);
        CORA_TMEM_LD_32X32B_X32(taddr + 32, (r + 32));
        tmem_ld_wait();
        if (c == S::kBufs - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_lead0 + acc * 8);
        }
        const uint32_t sbase = smem_u32(cbuf + c * kEpiBufBytes);
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(sbias + hf * S::kWarpCols + c * BK);
        mbar_wait(&rbar[c], (res_phase >> c) & 1u);
        res_phase ^= 1u << c;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t w[4];
          ld_shared_v4(sbase + sw128_offset(lane, ch), w[0], w[1], w[2], w[3]);
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t b2 = bw[ch * 4 + i];
            const float v0 = __uint_as_float(r[ch * 8 + 2 * i]) + bf16_lo(b2);
            const float v1 = __uint_as_float(r[ch * 8 + 2 * i + 1]) + bf16_hi(b2);
            o[i] = pack_bf16x2(v0 + bf16_lo(w[i]), v1 + bf16_hi(w[i]));
            const float2 y = make_float2(bf16_lo(o[i]), bf16_hi(o[i]));  // statistics of the rounded values
            if (ch == 0 && i == 0 && c == 0) nK = make_float2(-y.x, -y.x);
            const float2 dv = __fadd2_rn(y, nK);
            s1v = __fadd2_rn(s1v, dv);
            s2v = __ffma2_rn(dv, dv, s2v);
          }
          st_shared_v4(sbase + sw128_offset(lane, ch), o[0], o[1], o[2], o[3]);
        }
      }
      float2* pa = part + acc * (EW / 4) * BM;
      pa[hf * BM + row] = seg_moments(-nK.x, s1v.x + s1v.y, s2v.x + s2v.y, static_cast<float>(S::kWarpCols));
      named_bar_sync(1, 32 * EW);  // every column group of every row is in `part`
      float2 cm = pa[row];         // this CTA's 256-column (mean, M2)
#pragma unroll
      for (int g = 1; g < EW / 4; ++g) cm = merge_moments(cm, pa[g * BM + row], static_cast<float>(S::kWarpCols), g);
      if (hf == 0)
        st_async_v2f32(recv_remote0 + (acc * BM + row) * 8, cm.x, cm.y, xch_remote0 + acc * 8);
      mbar_wait(&xch_bar[acc], acc_phase);
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(7);
      const float2 rm = merge_moments(cm, recv[acc * BM + row], static_cast<float>(N / 2));
      const float mean = rm.x;
      const float rstd = rsqrtf(rm.y * inv_n + ln_eps);
#pragma unroll 1
      for (int c = 0; c < S::kBufs; ++c) {
        uint8_t* buf = cbuf + c * kEpiBufBytes;
        const uint32_t sbase = smem_u32(buf);
        const float* gm = sgamma + hf * S::kWarpCols + c * BK;
        const float* bt = sbeta + hf * S::kWarpCols + c * BK;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t w[4];
          ld_shared_v4(sbase + sw128_offset(lane, ch), w[0], w[1], w[2], w[3]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int col = ch * 8 + 2 * i;
            w[i] = pack_bf16x2((bf16_lo(w[i]) - mean) * rstd * gm[col] + bt[col],
                               (bf16_hi(w[i]) - mean) * rstd * gm[col + 1] + bt[col + 1]);
          }
          st_shared_v4(sbase + sw128_offset(lane, ch), w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tm_c, buf, nw + c * BK, row0);
          tma_store_commit();
        }
      }
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(8);
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps (every CTA)
    const uint32_t q = warp & 3;  // TMEM lane quadrant accessible to this warp
    const uint32_t ew = warp - 2;
    const int hf = static_cast<int>(ew) / 4;  // column half of the tile
    uint8_t* cbuf = smem + S::kOffC + ew * S::kNBuf * kEpiBufBytes;
    __nv_bfloat16* sbias = reinterpret_cast<__nv_bfloat16*>(smem + S::kOffBias + ew * S::kWarpCols * 2);
    uint64_t* rbar = res_bar + ew * S::kBufs;
    const uint32_t tmem_empty_lead0 = PAIR ? mapa_shared(&tmem_empty[0], lead_rank) : 0u;
    GW_DECL;
    if constexpr (EW == 256 / 32 && !RESIDUAL) {
      if (pre.nparts > 0) {
        // the prelude (step a1) in the 8 epilogue warps, while the first unit's mainloop runs: its scratch is
        // the staging buffers (free until the first accumulator), so no extra shared memory and no extra kernel
        static_assert(sizeof(PreludeSmem<256>) + sizeof(int32_t) * (kPreludeInGemmMaxBatch + 1) <=
                          static_cast<size_t>(S::kOffBias - S::kOffC), "prelude scratch in the staging buffers");
        auto& psm = *reinterpret_cast<PreludeSmem<256>*>(smem + S::kOffC);
        int32_t* s_off = reinterpret_cast<int32_t*>(smem + S::kOffC + sizeof(PreludeSmem<256>));
        const WarpTeam team{64, 256, 2};
        for (int part = static_cast<int>(blockIdx.x); part < pre.nparts; part += static_cast<int>(gridDim.x)) {
          prelude_part<256>(team, psm, s_off, pre, part, pre.nparts);
          team.sync();  // the scratch is reused by the next part, then by the staging buffers
        }
      }
    }
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
#ifdef CORA_GEMM_TRACE
      GW_WAIT(gw_w, mbar_wait(&tmem_full[acc], acc_phase));
#else
      mbar_wait(&tmem_full[acc], acc_phase);
#endif
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(6);
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
          if constexpr (ACT != CORA_ACT_NONE) {  // a compile-time variant: one epilogue body per kernel
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = apply_act(v[j], ACT);
          }
          uint8_t* buf = cbuf + (c % S::kNBuf) * kEpiBufBytes;
          if (S::kNBuf == 1 && c > 0) {  // the reused buffer: the previous chunk's store has read it
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
          }
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
            if (PAIR)
              mbar_arrive_cluster(tmem_empty_lead0 + acc * 8);
            else
              mbar_arrive(&tmem_empty[acc]);
          }
        }
      }
      if (u == unit0 && ew == 0 && lane == 0) GTRACE(8);
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
#ifdef CORA_GEMM_TRACE
    if (ew == 0 && lane == 0) {
      GW_STORE(4, gw_w);
      GW_STORE(5, clock64() - gw_t0);
    }
#endif
  }

  if (late_wait) pdl_wait();
  if (late_wait) KSPAN_WAITED(gemm, kSpanSlot);
  if (threadIdx.x == 64) GTRACE(9);
  tc_fence_before();
  if (CLUSTER)
    cluster_sync_all();  // the peers may still complete_tx / arrive on this CTA's barriers until here
  else
    __syncthreads();
  if (threadIdx.x == 64) GTRACE(10);
  if (warp == 1) {
    if (PAIR)
      tmem_dealloc_cg2<S::kTmemCols>(tmem_base);
    else
      tmem_dealloc<S::kTmemCols>(tmem_base);
  }
  KSPAN_EXIT(gemm, kSpanSlot);
}

template <int BN, int STAGES, bool RESIDUAL, int CL, bool LN = false, bool LNREG = false, int ACT = CORA_ACT_NONE>
cudaError_t run_gemm(const GemmArgs& g, cudaStream_t stream) {
  constexpr int EW = epi_warps<LN, LNREG>();
  constexpr int kThreads = 64 + 32 * EW;
  using S = GemmSmem<BN, STAGES, CL, LN, (RESIDUAL && !LNREG) ? BN * 4 / EW / BK : (LNREG ? 0 : 1), EW>;
  constexpr bool PAIR = CL == 4 || (CL == 2 && !LN);  // cta_group::2 (else single CTAs, DUO included)
  CUtensorMap ta, tb, tc, tr;
  if (!make_tmap_2d_bf16(&ta, g.a, g.k, g.m, static_cast<uint64_t>(g.k) * 2, BK, BM, true) ||
      !make_tmap_2d_bf16(&tb, g.b, g.k, g.n, static_cast<uint64_t>(g.k) * 2, BK, PAIR ? BN / 2 : BN, true) ||
      !make_tmap_2d_bf16(&tc, g.c, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
    return cudaErrorInvalidValue;
  if (RESIDUAL) {
    if (!make_tmap_2d_bf16(&tr, g.residual, g.n, g.m, static_cast<uint64_t>(g.n) * 2, BK, kEpiRows, true))
      return cudaErrorInvalidValue;
  } else {
    tr = tc;  // unused
  }
  auto kern = gemm_bf16_tn_kernel<BN, STAGES, RESIDUAL, CL, LN, LNREG, ACT>;
  static bool attr_set[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kAlloc);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  const int m_blocks = (g.m + BM - 1) / BM, n_blocks = (g.n + BN - 1) / BN;
  const int units = ((m_blocks + (PAIR ? 1 : 0)) / (PAIR ? 2 : 1)) * (LN ? 1 : n_blocks);
  // persistent grid = the clusters that can be co-resident (clusters of 4 cannot use every SM: GPC
  // boundaries strand some), so no cluster waits for a second wave
  static int max_clusters_dev[kMaxDevices] = {};
  int& max_clusters = max_clusters_dev[dev];
  if (max_clusters == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * (device_sm_count() / CL));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = S::kAlloc;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = device_sm_count() / CL;
    max_clusters = n;
    if (getenv("CORA_DEBUG") != nullptr)
      fprintf(stderr, "cora gemm<BN=%d,ST=%d,RES=%d,CL=%d,LN=%d>: %d co-resident clusters, smem %d B\n", BN, STAGES,
              int(RESIDUAL), CL, int(LN), n, S::kAlloc);
  }
  const int grid = (units < max_clusters ? units : max_clusters) * CL;
  return launch_pdl(kern, dim3(grid), dim3(kThreads), S::kAlloc, stream, CL, ta, tb, tc, tr,
                    static_cast<const __nv_bfloat16*>(g.bias), g.ln_gamma, g.ln_beta, g.ln_eps,
                    static_cast<const __nv_bfloat16*>(g.residual), static_cast<__nv_bfloat16*>(g.c), g.m, g.n, g.k,
                    g.act, g.late_wait ? 1 : 0, g.prelude);
}

}  // namespace

#ifndef CORA_GEMM_STAGES
#define CORA_GEMM_STAGES 6
#endif
namespace {
template <int ACT>
cudaError_t launch_gemm_act(const GemmArgs& g, bool pair, cudaStream_t stream) {
  if (g.residual != nullptr)
    return pair ? run_gemm<256, 5, true, 2, false, false, ACT>(g, stream)
                : run_gemm<256, 3, true, 1, false, false, ACT>(g, stream);
  return pair ? run_gemm<256, CORA_GEMM_STAGES, false, 2, false, false, ACT>(g, stream)
              : run_gemm<256, 3, false, 1, false, false, ACT>(g, stream);
}
}  // namespace

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.m == 0 || g.n == 0) return cudaSuccess;
  const bool pair = ((g.m + BM - 1) / BM) >= 2;  // a single m-block runs on one CTA
  // smem per SM: CTA pair -> 32 KB per stage (A 16 KB + half of B) -> 5 stages; 1 CTA -> 48 KB -> 3
  switch (g.act) {
    case CORA_ACT_NONE:
      return launch_gemm_act<CORA_ACT_NONE>(g, pair, stream);
    case CORA_ACT_RELU:
      return launch_gemm_act<CORA_ACT_RELU>(g, pair, stream);
    case CORA_ACT_GELU_ERF:
      return launch_gemm_act<CORA_ACT_GELU_ERF>(g, pair, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

// 128-row units from which the short-K LN GEMM runs as DUOs (74 two-CTA clusters)
constexpr int kLnDuoMinBlocks = 128;

bool gemm_ln_supported(const GemmArgs& g) {
  // act NONE only (the layer's a4 / a7): with the activation variants compiled in, the fully unrolled
  // epilogue is 4x the code and a one-unit-per-CTA launch stalls on cold instruction fetches
  return g.n == 512 && g.act == CORA_ACT_NONE && g.residual != nullptr && g.ln_gamma != nullptr &&
         g.ln_beta != nullptr && ((g.m + BM - 1) / BM) >= 2;
}

cudaError_t launch_gemm_ln(const GemmArgs& g, cudaStream_t stream) {
  if (g.m == 0) return cudaSuccess;
  if (!gemm_ln_supported(g)) return cudaErrorInvalidValue;
  // 2 CTA pairs per cluster.  Long K (FF2): row segments in registers, one staging buffer, 5 stages --
  // the mainloop is bound by the bytes in flight.  Short K (out-proj): the epilogue is the critical path,
  // so the residual is TMA-prefetched into two staging buffers per warp (4 stages fit beside them).
  // Long K (FF2) stays on 2 CTA pairs: a DUO CTA fills 48 KB of smem per k-block instead of 32 and its
  // mainloop, bound by the bytes in flight, runs slower than the 16 SMs it gains (C4 FF2 + LN2 80 -> 83 us).
  // Short K (out-proj, epilogue-bound) runs as DUOs once there are enough 128-row units to fill the
  // 148 SMs in several waves (C4 out-proj + LN1 41.5 -> 36.9 us; at T ~ 1.5-6k the 4-CTA clusters are
  // 0.2-0.5 us faster).  Both give bitwise the same output (test_ln_gemm_duo_bitwise).
  // CORA_LN_DUO=0 / 1 forces the short-K choice (A/B runs).
  static const int duo_env = getenv("CORA_LN_DUO") != nullptr ? atoi(getenv("CORA_LN_DUO")) : -1;
  const int m_blocks = (g.m + BM - 1) / BM;
  const bool duo = duo_env >= 0 ? duo_env != 0 : m_blocks >= kLnDuoMinBlocks;
  if (g.k >= 1024) return run_gemm<256, 6, true, 4, true, true>(g, stream);
  if (duo) return run_gemm<256, 3, true, 2, true, false>(g, stream);
  return run_gemm<256, 4, true, 4, true, false>(g, stream);
}

}  // namespace cora
