// Step a3: fused ragged multi-head attention (QK^T -> softmax -> .V) per (sequence, head, q-tile).
//
// Paper: the SDPA sub-module is where CoRa beats FasterTransformer, because
// it computes only (partially padded) per-sequence L_b x L_b score blocks instead of a fully
// padded B x L_max x L_max tensor; thread blocks are ordered
// longest-sequence-first.  CoRa runs QK^T, softmax and AttnV as three
// kernels with the ragged score tensor X[b,i,h,j] in HBM.
//
// sm_100a design: nothing of S or P touches HBM.  A persistent CTA walks the
// longest-first tile list built by the prelude (static stride over the list).  For one work
// tile (b, h, qt): Q = 128 query rows of sequence b, head h; K_j / V_j = 128-key tiles,
// j < ceil(L_b / 128).
//   warp 0     : TMA producers from QKV[T, 3d], 128x64 SWIZZLE_128B boxes: lane 0 Q (2 slots) + K (3-deep
//                ring), lane 1 V (2-deep ring)
//   warp 1     : TMEM allocator + single-thread tcgen05.mma issuer
//                  S_j = Q K_j^T  (M128 N128 K64, SS form, fp32 in TMEM cols [0,128))
//                  O  += P_j V_j  (M128 N64 K128, TS form: P read from TMEM cols [128,192) as bf16
//                                  pairs, V an MN-major smem operand; O in TMEM cols [192,256))
//                the S MMAs run one KV step ahead of the PV MMAs over the CTA's whole work list, so the
//                next tile's S_0 is issued before this tile's last PV
//   warps 4..7 : softmax / correction, one query row per thread (TMEM lane = row):
//                  S_j is read from TMEM in one pass and the buffer released at once (so S_{j+1}
//                  overlaps the exponentials), online softmax in the exp2 domain with a lazily
//                  moved reference max, masking keys >= L_b with -inf in the tail tile only
//                  (reading c18), P_j -> bf16 pairs -> TMEM (tcgen05.st; A operand of the PV MMA);
//                  O accumulates in TMEM across KV tiles (rescaled in place only when the
//                  reference max moves); the row sums l go to shared memory for the epilogue.
//   warps 8..11: (bidirectional kernel) tile epilogue: wait for the tile's last PV, read O out of TMEM,
//                  o / l -> bf16 -> predicated row stores (rows >= L_b belong to the next sequence and are
//                  never written), so the softmax warps start the next tile right after its last P.  The
//                  causal kernel (256 threads; its softmax warps need 200 registers) keeps this epilogue in
//                  the softmax warps.  warps 2..3 complete warpgroup 0 (setmaxnreg works per warpgroup).
// Rows of a 128-row TMA box that lie past the sequence end are real rows of the next
// sequence (finite) or TMA zero-fill past T: their keys are masked and their queries discarded.
// Two CTAs per SM (112 KB smem, 256 TMEM columns each) overlap one CTA's softmax with the other's MMAs.
// Nothing of S or P goes through shared memory or HBM.  Short sequences may share a tile (packed window,
// block-diagonal mask, SURVEY f-4); causal attention (f-2) skips KV tiles above the diagonal.  The
// softmax warps prefetch the next tile's metadata into shared memory with cp.async.
#include <cuda_bf16.h>

#include <cstdint>
#include <type_traits>

#include "cora_internal.h"
#include "ptx.cuh"

CORA_KSPAN_DEFINE(attn)

namespace cora {
namespace {

constexpr int HD = 64;        // head dim (one SWIZZLE_128B row)
constexpr int TQ = 128;       // query rows per work tile
constexpr int TK = 128;       // keys per KV tile
constexpr int QSTAGES = 2;    // Q double buffer: the next tile's Q streams in under the current tile
constexpr int KSTAGES = 3;    // K ring depth
constexpr int VSTAGES = 2;    // V ring depth
// Work schedule ring: entries published by the producer thread, read in order by the V producer, the MMA
// thread (S and PV walks) and the 4 softmax warps -- 7 readers release each entry
constexpr int kRing = 8;
// The producer claims the next entry when it issues the current one's last K load, not when it starts it: the
// claim's latency still hides under the K ring (3 steps ahead of the MMA), and near the end of the list a CTA
// holds one claimed entry for less time (C4 84.5 -> 83.1 us, causal 73.9 -> 72.2, C3 23.0 -> 22.2)
#ifndef CORA_ATTN_LATE_CLAIM
#define CORA_ATTN_LATE_CLAIM 1
#endif
constexpr bool kLateClaim = CORA_ATTN_LATE_CLAIM != 0;
// Warp roles.  Bidirectional kernel (192 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2-5 softmax.  Causal kernel (256 threads): warps 0 / 1 the same, warps 2-3 idle (they complete
// warpgroup 0, whose registers go to the softmax warpgroup), warps 4-7 softmax.  Warp w of the softmax
// reads TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31.
// Bidirectional kernel (384 threads): warpgroup 2 (warps 8-11) is the tile epilogue -- it waits for the
// tile's last PV, reads O out of TMEM, normalises it by the row sums the softmax warps leave in shared memory
// and stores it -- so the softmax warps go straight on to the next tile's S_0.
template <bool CAUSAL>
constexpr bool kEpiWG = !CAUSAL;
template <bool CAUSAL>
constexpr int kThreadsOf = CAUSAL ? 256 : 384;
template <bool CAUSAL>
constexpr uint32_t kSoftmaxWarp0 = 4;
constexpr uint32_t kEpiWarp0 = 8;
// ring readers: V producer, two MMA walks, 4 softmax warps (+ 4 epilogue warps)
template <bool CAUSAL>
constexpr int kRingReadersOf = kEpiWG<CAUSAL> ? 11 : 7;
// causal: 2 CTAs x 256 threads x 128 registers at launch; setmaxnreg: 128 x 56 + 128 x 200 = 256 x 128 (the
// per-chunk liveness of the diagonal / tail tiles needs more than the 168 registers of 192 threads).
// bidirectional: 2 CTAs x 384 threads x 80 registers; 128 x (40 + 160 + 40) = 384 x 80.
#ifndef CORA_ATTN_REGS_SM
#define CORA_ATTN_REGS_SM 160
#endif
template <bool CAUSAL>
constexpr uint32_t kRegsSoftmax = CAUSAL ? 200 : CORA_ATTN_REGS_SM;
template <bool CAUSAL>
constexpr uint32_t kRegsOther = CAUSAL ? 56 : (240 - CORA_ATTN_REGS_SM) / 2;
constexpr uint32_t kRegsEpi = (240 - CORA_ATTN_REGS_SM) / 2;
constexpr int kTileBytes = TQ * HD * 2;  // 16 KB, also the K and V tile size
// Lazy rescaling (reading a3-r1): the running reference max m_ref of a row is only
// moved when a new score exceeds it by more than kRescaleLog2 (in log2 units), so P <= 2^8 and the
// O accumulator in TMEM is rescaled rarely.  O / l is unchanged mathematically.
constexpr float kRescaleLog2 = 8.0f;
// MUFU offload (experiment, off): of every 4 consecutive key pairs, kPolyPairs are exponentiated on the
// FMA pipe with a polynomial (exp2_poly) instead of MUFU.EX2.  Measured at C4: 0 -> 105 us, 1 -> 130 us,
// 2 -> 174 us, 3 -> 225 us: the softmax warps are issue/latency-bound, not MUFU-bound (XU 45 %), so
// the ~7 extra instructions per offloaded exponential cost more than the MUFU cycles they free.
#ifndef CORA_ATTN_POLY_PAIRS
#define CORA_ATTN_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = CORA_ATTN_POLY_PAIRS;
__device__ __forceinline__ constexpr bool poly_col(int c) { return ((c >> 1) & 3) < kPolyPairs; }

// 2^x on the FMA/ALU pipes, x >= -125 (callers clamp or select): x = j + f with j = rint(x) by the
// 1.5 * 2^23 magic-number add, f in [-1/2, 1/2]; 2^f by a degree-3 polynomial fitted for relative error
// (max 2.1e-4, below the bf16 rounding of P, 3.9e-3); 2^j added into the exponent field.  The integer
// part of t = x + 1.5 * 2^23 sits in its low mantissa bits, so (bits(t) << 23) == j << 23 (mod 2^32).
__device__ __forceinline__ float exp2_poly(float x) {
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  const float p = fmaf(fmaf(fmaf(0.053027520f, f, 0.24221394f), f, 0.69357257f), f, 0.99995904f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// 1 / x on the FMA pipe for normal x > 0 (the row sums l >= 2^-8): the bit-trick seed (relative error
// < 1/8) and three Newton steps r <- r (2 - x r) (error squares each step: < 6e-8).  Keeps the tile
// epilogue off MUFU, where a lone RCP queues behind the other CTA's exponentials.
__device__ __forceinline__ float rcp_fma(float x) {
  float r = __int_as_float(0x7EF311C3 - __float_as_int(x));
#pragma unroll
  for (int it = 0; it < 3; ++it) r = fmaf(r, fmaf(-x, r, 1.f), r);
  return r;
}

#ifdef CORA_ATTN_TRACE
// Phase trace (profiling builds only): softmax warp 0 lane 0 and the MMA thread of the first kTraceCtas
// CTAs record (clock64 << 8 | event) into a per-CTA, per-role buffer of kTraceLen entries.
constexpr int kTraceCtas = 296, kTraceLen = 2048;
__device__ uint64_t g_attn_trace[kTraceCtas][2][kTraceLen];
__device__ int g_attn_trace_n[kTraceCtas][2];
#define ATR(role, ev)                                                                              \
  do {                                                                                            \
    if (blockIdx.x < kTraceCtas && atr_n < kTraceLen)                                             \
      g_attn_trace[blockIdx.x][role][atr_n++] = (clock64() << 8) | (ev);                          \
  } while (0)
#define ATR_DONE(role) do { if (blockIdx.x < kTraceCtas) g_attn_trace_n[blockIdx.x][role] = atr_n; } while (0)
#define ATR_SM(ev) do { if (qd == 0 && lane == 0) ATR(0, ev); } while (0)
#define ATR_MMA(ev) ATR(1, ev)
#else
#define ATR_SM(ev) do {} while (0)
#define ATR_MMA(ev) do {} while (0)
#define ATR_DONE(role) do {} while (0)
#endif

struct AttnSmem {
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + QSTAGES * kTileBytes;
  static constexpr int kOffV = kOffK + KSTAGES * kTileBytes;
  static constexpr int kOffRing = kOffV + VSTAGES * kTileBytes;  // int4 [kRing] the CTA's work schedule
  static constexpr int kOffL = kOffRing + kRing * 16;            // float [TQ] row sums softmax -> epilogue
  static constexpr int kOffBar = kOffL + TQ * 4;
  // q_full/empty[QS], k_full/empty[KS], v_full/empty[VS], s_full, s_empty, p_full, pv_done, o_empty,
  // ring_full/empty[kRing], l_full, l_empty
  static constexpr int kNumBars = 2 * (QSTAGES + KSTAGES + VSTAGES) + 5 + 2 * kRing + 2;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  static constexpr int kAlloc = kBytes;
};
// TMEM columns: S (fp32, 128) | P (bf16 pairs, 64) | O (fp32, 64)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kTmemS = 0, kTmemP = 128, kTmemO = 192;

// One work tile: head h, q-tile qt of a sequence starting at packed row r0 with L tokens -- or, packed
// (SURVEY f-4, reading f4-r1), a window of L <= 128 consecutive tokens holding several short sequences,
// whose score tile is block-diagonal: row i attends to the keys of its own sequence only.
struct WorkTile {
  int h, qt, r0, L;
  bool packed;
};
// The walk of one CTA: bidirectional attention visits single q-tiles of the longest-first tile list;
// causal attention visits the UNIT list (same longest-first order, ceil(nq/2) units per (b, h)) and
// processes unit qp as the q-tile pair (nq-1-qp, qp), whose KV work (nq-qp) + (qp+1) = nq+1 is the
// same for every unit of a sequence (a lone middle tile when nq is odd).  The entries are handed out
// dynamically: CTA c starts with entry c, then each CTA's producer thread claims the next unclaimed
// entry from a global ticket counter when it starts a tile (longest-processing-time-first: the list is
// sorted by work, so the last entries handed out are the shortest), and publishes it to the CTA's roles
// through the schedule ring.
struct WorkUnit {
  int h, r0, L, qt0, qt1, count;
  bool packed;
  __device__ __forceinline__ WorkTile tile(int sub) const { return WorkTile{h, sub ? qt1 : qt0, r0, L, packed}; }
};
// A schedule entry: (idx, tile word, row_off[b], L_b) of a work-list entry, idx < 0 = end of the CTA's walk.
__device__ __forceinline__ int4 sched_entry(const int32_t* list, const int2* list_seq, int idx, int n) {
  if (idx >= n) return make_int4(-1, 0, 0, 0);
  const int32_t w = __ldg(list + idx);
  const int2 sq = __ldg(list_seq + idx);
  return make_int4(idx, w, sq.x, sq.y);
}
template <bool CAUSAL>
__device__ __forceinline__ WorkUnit decode_work(int4 e) {
  const WorkTile t{(e.y >> 16) & 0xFF, (e.y >> 24) & 0x7F, e.z, e.w, e.y < 0};
  if (!CAUSAL) return WorkUnit{t.h, t.r0, t.L, t.qt, t.qt, 1, t.packed};
  const int nq = (t.L + TQ - 1) / TQ, qp = t.qt;
  return WorkUnit{t.h, t.r0, t.L, nq - 1 - qp, qp, (nq - 1 - qp == qp) ? 1 : 2, t.packed};
}
// Reader of the schedule ring: entry k of the CTA's walk sits in slot k % kRing.  All lanes of a warp (or a
// single thread) wait for the slot, read it and release it with one arrive.
struct RingReader {
  uint32_t ring;  // shared address of the int4 entries
  uint64_t* full;
  uint64_t* empty;
  int k;
  __device__ __forceinline__ int4 next(bool warp_wide) {
    const int slot = k & (kRing - 1);
    mbar_wait<false>(&full[slot], (k / kRing) & 1);
    uint32_t a, b, c, d;
    ld_shared_v4(ring + slot * 16, a, b, c, d);
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane_id() == 0) mbar_arrive(&empty[slot]);
    ++k;
    return make_int4(static_cast<int>(a), static_cast<int>(b), static_cast<int>(c), static_cast<int>(d));
  }
};

// CAUSAL: masked MHA (App. D.3): query i attends to keys j <= i of its sequence, so
// q-tile qt needs only KV tiles j <= qt (the "lower triangular" ragged loop -- tiles above the diagonal
// are never loaded or computed) and the diagonal tile is masked per element.
template <bool CAUSAL>
__global__ void __launch_bounds__(kThreadsOf<CAUSAL>, 2)
    attention_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const int32_t* __restrict__ tiles,
                         const int2* __restrict__ tile_seq, int32_t* __restrict__ n_tiles_ptr,
                         const int32_t* __restrict__ seq_of_tok, const int32_t* __restrict__ pos_in_seq,
                         const int32_t* __restrict__ lengths, __nv_bfloat16* __restrict__ out, int32_t d_model,
                         float scale_log2) {
  // SWIZZLE_128B atoms need 1024-B alignment; the dynamic smem window is declared so aligned
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  KSPAN_ENTRY(attn, 1);
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AttnSmem::kOffBar);
  uint64_t* q_full = bars;
  uint64_t* q_empty = q_full + QSTAGES;
  uint64_t* k_full = q_empty + QSTAGES;
  uint64_t* k_empty = k_full + KSTAGES;
  uint64_t* v_full = k_empty + KSTAGES;
  uint64_t* v_empty = v_full + VSTAGES;
  uint64_t* s_full = v_empty + VSTAGES;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_empty + 1;
  uint64_t* pv_done = p_full + 1;
  uint64_t* o_empty = pv_done + 1;
  uint64_t* ring_full = o_empty + 1;
  uint64_t* ring_empty = ring_full + kRing;
  uint64_t* l_full = ring_empty + kRing;
  uint64_t* l_empty = l_full + 1;
  float* lbuf = reinterpret_cast<float*>(smem + AttnSmem::kOffL);
  const uint32_t ring_addr = smem_u32(smem + AttnSmem::kOffRing);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + AttnSmem::kNumBars);

  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    for (int s = 0; s < QSTAGES; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < KSTAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VSTAGES; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    mbar_init(o_empty, 4);
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&ring_full[r], 1);
      mbar_init(&ring_empty[r], kRingReadersOf<CAUSAL>);
    }
    mbar_init(l_full, 4);
    mbar_init(l_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_ptr);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // tmem_base: read by each role after its register reallocation (values live across setmaxnreg are spilled)
  uint32_t tmem_base = 0;
  pdl_wait();  // QKV (previous kernel) complete and visible
  KSPAN_WAITED(attn, 1);
  pdl_trigger();

  if (warp < kSoftmaxWarp0<CAUSAL>) {
    // warpgroup 0 (producer, MMA issuer, two idle warps) hands its registers to the softmax warpgroup
    setmaxnreg_dec<kRegsOther<CAUSAL>>();
    tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_ptr);
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    // lane 0 streams Q and K, lane 1 streams V: the two rings are refilled independently, so a V slot
    // still held by a pending PV never delays the next K load (and vice versa)
    if (lane == 0) {
      // the scheduler: publishes entry k of the walk to ring slot k % kRing once all readers released it
      const int n_tiles = *n_tiles_ptr;
      int n_pub = 0;
      auto publish = [&](int4 e) {
        const int slot = n_pub & (kRing - 1);
        if (n_pub >= kRing) mbar_wait<false>(&ring_empty[slot], ((n_pub / kRing) - 1) & 1);
        st_shared_v4(ring_addr + slot * 16, static_cast<uint32_t>(e.x), static_cast<uint32_t>(e.y),
                     static_cast<uint32_t>(e.z), static_cast<uint32_t>(e.w));
        mbar_arrive(&ring_full[slot]);  // release: the entry is visible to the readers that see the phase
        ++n_pub;
      };
      uint32_t q_ph = 0, k_ph = 0;
      int qs = 0, ks = 0;
      int4 e = sched_entry(tiles, tile_seq, blockIdx.x, n_tiles);
      publish(e);
      // the next entry is claimed when a tile starts; its ticket is read after the tile's loads are issued
      int ticket = (!kLateClaim && e.x >= 0) ? atomicAdd(n_tiles_ptr + 1, 1) : 0;
      while (e.x >= 0) {
        const WorkUnit wu = decode_work<CAUSAL>(e);
        for (int sub = 0; sub < wu.count; ++sub) {
          const WorkTile cur = wu.tile(sub);
          const int nkv = CAUSAL ? min((cur.L + TK - 1) / TK, cur.qt + 1) : (cur.L + TK - 1) / TK;
          mbar_wait<false>(&q_empty[qs], q_ph ^ 1);
          mbar_arrive_expect_tx(&q_full[qs], kTileBytes);
          tma_load_2d(smem + AttnSmem::kOffQ + qs * kTileBytes, &tm_qkv, &q_full[qs], cur.h * HD, cur.r0 + cur.qt * TQ);
          if (++qs == QSTAGES) qs = 0, q_ph ^= 1;
          for (int j = 0; j < nkv; ++j) {
            mbar_wait<false>(&k_empty[ks], k_ph ^ 1);
            mbar_arrive_expect_tx(&k_full[ks], kTileBytes);
            tma_load_2d(smem + AttnSmem::kOffK + ks * kTileBytes, &tm_qkv, &k_full[ks], d_model + cur.h * HD,
                        cur.r0 + j * TK);
            if (++ks == KSTAGES) ks = 0, k_ph ^= 1;
            if (kLateClaim && sub == wu.count - 1 && j == nkv - 1) ticket = atomicAdd(n_tiles_ptr + 1, 1);
          }
        }
        e = sched_entry(tiles, tile_seq, static_cast<int>(gridDim.x) + ticket, n_tiles);
        publish(e);
        if (!kLateClaim && e.x >= 0) ticket = atomicAdd(n_tiles_ptr + 1, 1);
      }
    } else if (lane == 1) {
      uint32_t v_ph = 0;
      int vs = 0;
      RingReader rr{ring_addr, ring_full, ring_empty, 0};
      for (int4 e = rr.next(false); e.x >= 0; e = rr.next(false)) {
        const WorkUnit wu = decode_work<CAUSAL>(e);
        for (int sub = 0; sub < wu.count; ++sub) {
          const WorkTile cur = wu.tile(sub);
          const int nkv = CAUSAL ? min((cur.L + TK - 1) / TK, cur.qt + 1) : (cur.L + TK - 1) / TK;
          for (int j = 0; j < nkv; ++j) {
            mbar_wait<false>(&v_empty[vs], v_ph ^ 1);
            mbar_arrive_expect_tx(&v_full[vs], kTileBytes);
            tma_load_2d(smem + AttnSmem::kOffV + vs * kTileBytes, &tm_qkv, &v_full[vs], 2 * d_model + cur.h * HD,
                        cur.r0 + j * TK);
            if (++vs == VSTAGES) vs = 0, v_ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
#ifdef CORA_ATTN_TRACE
      int atr_n = 0;
#endif
      constexpr uint32_t idesc_s = make_idesc_bf16(TQ, TK);
      constexpr uint32_t idesc_o = make_idesc_bf16(TQ, HD, /*b_mn_major=*/true);
      int ks = 0, vs = 0;
      uint32_t k_ph = 0, v_ph = 0, s_ph = 0, p_ph = 0, o_ph = 0;
      // The S iterator walks the flattened (tile, KV step) sequence one step ahead of the PV loop, across
      // tile boundaries: the next tile's S_0 is issued before this tile's last PV, so the softmax warps find
      // it ready when they finish the tile (their epilogue of the tile is deferred into the next one).
      int s_sub = 0, s_j = 0, s_nkv = 0, s_qs = 0;
      uint32_t s_qph = 0;
      auto tile_nkv = [](const WorkTile& t) {
        return CAUSAL ? min((t.L + TK - 1) / TK, t.qt + 1) : (t.L + TK - 1) / TK;
      };
      // two walks of the schedule: the S iterator (one KV step ahead) and the PV loop
      RingReader rs{ring_addr, ring_full, ring_empty, 0}, rp{ring_addr, ring_full, ring_empty, 0};
      int4 s_e = rs.next(false);
      WorkUnit s_wu{};
      if (s_e.x >= 0) {
        s_wu = decode_work<CAUSAL>(s_e);
        s_nkv = tile_nkv(s_wu.tile(0));
      }
      auto issue_next_s = [&]() {
        if (s_e.x < 0) return;
        ATR_MMA(20);
        if (s_j == 0) mbar_wait<false>(&q_full[s_qs], s_qph);
        mbar_wait<false>(&k_full[ks], k_ph);
        ATR_MMA(21);
        mbar_wait<false>(s_empty, s_ph ^ 1);  // the softmax has read the previous S
        ATR_MMA(22);
        s_ph ^= 1;
        tc_fence_after();
        const uint32_t q_addr = smem_u32(smem + AttnSmem::kOffQ + s_qs * kTileBytes);
        const uint32_t k_addr = smem_u32(smem + AttnSmem::kOffK + ks * kTileBytes);
  #pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ss(tmem_base + kTmemS, make_sdesc_sw128(q_addr + k * 32, 16, 1024),
                       make_sdesc_sw128(k_addr + k * 32, 16, 1024), idesc_s, k != 0);
        umma_commit(&k_empty[ks]);
        umma_commit(s_full);
        if (++ks == KSTAGES) ks = 0, k_ph ^= 1;
        if (++s_j == s_nkv) {  // the tile's last S: its Q slot is free once that MMA is done
          umma_commit(&q_empty[s_qs]);
          if (++s_qs == QSTAGES) s_qs = 0, s_qph ^= 1;
          s_j = 0;
          if (++s_sub == s_wu.count) {
            s_sub = 0;
            s_e = rs.next(false);
            if (s_e.x >= 0) s_wu = decode_work<CAUSAL>(s_e);
          }
          if (s_e.x >= 0) s_nkv = tile_nkv(s_wu.tile(s_sub));
        }
      };
      issue_next_s();
      for (int4 e = rp.next(false); e.x >= 0; e = rp.next(false)) {
        const WorkUnit wu = decode_work<CAUSAL>(e);
        for (int sub = 0; sub < wu.count; ++sub) {
          const int nkv = tile_nkv(wu.tile(sub));
          for (int j = 0; j < nkv; ++j) {
            issue_next_s();                        // S_{k+1} overlaps the softmax of S_k
            mbar_wait<false>(p_full, p_ph);        // P_j in TMEM (and O rescaled if needed)
            ATR_MMA(23);
            p_ph ^= 1;
            mbar_wait<false>(&v_full[vs], v_ph);
            ATR_MMA(24);
            if (j == 0) {  // the softmax warps have read the previous tile's O out of TMEM
              mbar_wait<false>(o_empty, o_ph ^ 1);
              o_ph ^= 1;
            }
            tc_fence_after();
            const uint32_t v_addr = smem_u32(smem + AttnSmem::kOffV + vs * kTileBytes);
  #pragma unroll
            for (int k = 0; k < TK / 16; ++k) {
              // A = P from TMEM (16 keys = 8 packed columns per step), B = V (MN-major, 16 key rows per step)
              const uint64_t vd = make_sdesc_sw128(v_addr + k * 16 * 128, kTileBytes, 1024);
              umma_bf16_ts(tmem_base + kTmemO, tmem_base + kTmemP + k * 8, vd, idesc_o, (j | k) != 0);
            }
            umma_commit(&v_empty[vs]);
            umma_commit(pv_done);
            ATR_MMA(25);
            if (++vs == VSTAGES) vs = 0, v_ph ^= 1;
          }
        }
      }
      ATR_DONE(1);
    }
  }
  } else if (!kEpiWG<CAUSAL> || warp < kEpiWarp0) {
    // ------------------------------------------------------------ softmax / correction (/ epilogue)
    setmaxnreg_inc<kRegsSoftmax<CAUSAL>>();
    tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_ptr);
    const uint32_t qd = warp & 3;  // TMEM lane quadrant
    const bool out_v8 = (reinterpret_cast<uintptr_t>(out) & 31u) == 0 && (d_model % 16) == 0 && (HD % 16) == 0;
    const int i = qd * 32 + lane;  // query row within the tile
    const uint32_t t_lane = (qd * 32) << 16;
    uint32_t s_ph = 0, pv_ph = 0;
#ifdef CORA_ATTN_TRACE
    int atr_n = 0;
#endif
    // epilogue warpgroup: the previous tile's last PV has not been waited for (its P columns are reused by
    // this tile's P_0); l_n: row sums handed over so far
    bool pv_pending = false;
    int l_n = 0;
    auto hand_l = [&](float lv) {
      if (l_n > 0) mbar_wait<false>(l_empty, (l_n - 1) & 1);  // the epilogue has read the previous tile's
      lbuf[i] = lv;
      __syncwarp();
      if (lane == 0) mbar_arrive(l_full);
      ++l_n;
    };
    // the walk's entries come from the schedule ring (published by the producer thread a tile ahead)
    RingReader rw{ring_addr, ring_full, ring_empty, 0};
    while (true) {
      ATR_SM(11);
      const int4 mt = rw.next(true);
      ATR_SM(12);
      if (mt.x < 0) break;
      const WorkUnit wu = decode_work<CAUSAL>(mt);
      for (int sub = 0; sub < wu.count; ++sub) {
        const WorkTile cur = wu.tile(sub);
        const int L = cur.L;
        const int nkv = CAUSAL ? min((L + TK - 1) / TK, cur.qt + 1) : (L + TK - 1) / TK;
        if (cur.qt * TQ + static_cast<int>(qd) * 32 >= L) {
          // none of this warp's 32 query rows belongs to the sequence: keep the barrier protocol,
          // skip the math (its P rows are stale, its O rows are never stored)
          for (int j = 0; j < nkv; ++j) {
            mbar_wait<false>(s_full, s_ph);
            s_ph ^= 1;
            tc_fence_after();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            if (j > 0 || pv_pending) {
              mbar_wait<false>(pv_done, pv_ph);
              pv_ph ^= 1;
              pv_pending = false;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
          }
          if constexpr (kEpiWG<CAUSAL>) {
            hand_l(0.f);  // keeps the handshake; the epilogue stores nothing for this warp
            pv_pending = true;
            continue;
          }
          mbar_wait<false>(pv_done, pv_ph);
          pv_ph ^= 1;
          tc_fence_after();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_empty);
          continue;
        }
        float m_ref = -INFINITY, l = 0.f;
        ATR_SM(9);
        for (int j = 0; j < nkv; ++j) {
          const int valid = L - j * TK;  // keys of this tile that belong to sequence b (>= 1)
          const bool diag = CAUSAL && j == cur.qt;
          // leading 32-key chunks holding a key visible to some row of this warp (warp-uniform): a tail tile
          // stops at the last valid key, a causal diagonal tile at this warp's last row; the chunks after
          // them are not exponentiated -- their P is 0
          // (causal kernel only: the bidirectional one keeps every chunk live -- within its 168 registers
          // per-chunk liveness spills -- and masks the tail tile element by element)
          int live = TK / 32;
          if constexpr (CAUSAL) {
            if (valid < TK) live = (valid + 31) >> 5;
            if (diag && live > static_cast<int>(qd) + 1) live = static_cast<int>(qd) + 1;
            if (cur.packed) live = TK / 32;
          }
          ATR_SM(1);
          mbar_wait<false>(s_full, s_ph);
          ATR_SM(2);
          s_ph ^= 1;
          tc_fence_after();
          uint32_t sr[TK];
  #pragma unroll
          for (int cb = 0; cb < TK / 32; ++cb) CORA_TMEM_LD_32X32B_X32(tmem_base + t_lane + kTmemS + cb * 32, (sr + cb * 32));
          tmem_ld_wait();
          ATR_SM(3);
          // S is in registers: hand the TMEM buffer back so S_{j+1} runs under this softmax
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty);
          float* sv = reinterpret_cast<float*>(sr);
          // keys >= L_b (tail tile) and, with CAUSAL, keys after the query (diagonal tile) get -inf before the
          // row max (reading c18); only the last live chunk can hold such keys
          const bool masked = diag || valid < TK || cur.packed;
          if (cur.packed) {  // block-diagonal (one KV tile: j == 0 == qt)
            // keys [lo, hi) of the window belong to this row's sequence (f_fo / f_fi maps of the prelude)
            int lo = 0, hi = 0;
            if (i < L) {
              const int t = cur.r0 + i;
              lo = i - __ldg(pos_in_seq + t);
              hi = lo + __ldg(lengths + __ldg(seq_of_tok + t));
            }
  #pragma unroll
            for (int c = 0; c < TK; ++c)
              if (c < lo || c >= hi || (CAUSAL && c > i)) sv[c] = -INFINITY;
          } else if (!CAUSAL && valid < TK) {
  #pragma unroll
            for (int c = 0; c < TK; ++c)
              if (c >= valid) sv[c] = -INFINITY;
          } else if (masked) {
            const int hi = diag ? min(valid, i + 1) : valid;
            auto mask_chunk = [&](auto cb_tag) {
              constexpr int cb = decltype(cb_tag)::value;
              if (cb == live - 1) {
  #pragma unroll
                for (int c = cb * 32; c < cb * 32 + 32; ++c)
                  if (c >= hi) sv[c] = -INFINITY;
              }
            };
            mask_chunk(std::integral_constant<int, 0>{});
            mask_chunk(std::integral_constant<int, 1>{});
            mask_chunk(std::integral_constant<int, 2>{});
            mask_chunk(std::integral_constant<int, 3>{});
          }
          float m8[8];
  #pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = -INFINITY;
          auto max_chunk = [&](auto cb_tag) {
            constexpr int cb = decltype(cb_tag)::value;
            if (cb < live) {
  #pragma unroll
              for (int c = cb * 32; c < cb * 32 + 32; ++c) m8[c & 7] = fmaxf(m8[c & 7], sv[c]);
            }
          };
          if constexpr (CAUSAL) {
            max_chunk(std::integral_constant<int, 0>{});
            max_chunk(std::integral_constant<int, 1>{});
            max_chunk(std::integral_constant<int, 2>{});
            max_chunk(std::integral_constant<int, 3>{});
          } else {
#ifdef CORA_ATTN_PROF_MAX_FIRST_ONLY  // profiling build only: the row max of the first KV tile alone
            if (j == 0)
#endif
  #pragma unroll
            for (int c = 0; c < TK; ++c) m8[c & 7] = fmaxf(m8[c & 7], sv[c]);
          }
          const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                 fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * scale_log2;
          ATR_SM(4);
          // lazy rescale: move the reference max only when it is exceeded by > kRescaleLog2
          const bool bump = mx > m_ref + kRescaleLog2;
          const float m_new = bump ? mx : m_ref;
          const float alpha = ex2_approx(m_ref - m_new);  // 1 when not bumped, 0 on the first tile
          m_ref = m_new;
          // p = exp2(s * scale_log2 - m_ref) (masked keys give exactly 0), fp32 row sum in 8 chains,
          // bf16 pairs packed right away (the A operand layout of the TS MMA: 2 keys per column)
          float r8[8];
  #pragma unroll
          for (int k = 0; k < 8; ++k) r8[k] = 0.f;
          uint32_t pk[TK / 2];
          auto exp_chunk = [&](auto cb_tag) {
            constexpr int cb = decltype(cb_tag)::value;
            if (cb < live) {
  #pragma unroll
              for (int c = cb * 32; c < cb * 32 + 32; c += 2) {
                const float x0 = fmaf(sv[c], scale_log2, -m_ref), x1 = fmaf(sv[c + 1], scale_log2, -m_ref);
                float p0, p1;
                if (poly_col(c)) {
                  // masked keys (-inf) must give exactly 0 like EX2; unmasked x is clamped into the poly's range
                  p0 = masked ? (x0 > -125.f ? exp2_poly(x0) : 0.f) : exp2_poly(fmaxf(x0, -125.f));
                  p1 = masked ? (x1 > -125.f ? exp2_poly(x1) : 0.f) : exp2_poly(fmaxf(x1, -125.f));
                } else {
                  p0 = ex2_approx(x0);
                  p1 = ex2_approx(x1);
                }
                r8[(c >> 1) & 7] += p0 + p1;
                pk[c / 2] = pack_bf16x2(p0, p1);
              }
            } else {
  #pragma unroll
              for (int c = cb * 32; c < cb * 32 + 32; c += 2) pk[c / 2] = 0u;
            }
          };
          if constexpr (CAUSAL) {
            exp_chunk(std::integral_constant<int, 0>{});
            exp_chunk(std::integral_constant<int, 1>{});
            exp_chunk(std::integral_constant<int, 2>{});
            exp_chunk(std::integral_constant<int, 3>{});
          } else {
  #pragma unroll
            for (int c = 0; c < TK; c += 2) {
              const float x0 = fmaf(sv[c], scale_log2, -m_ref), x1 = fmaf(sv[c + 1], scale_log2, -m_ref);
              float p0, p1;
              if (poly_col(c)) {
                // masked keys (-inf) must give exactly 0 like EX2; unmasked x is clamped into the poly's range
                p0 = masked ? (x0 > -125.f ? exp2_poly(x0) : 0.f) : exp2_poly(fmaxf(x0, -125.f));
                p1 = masked ? (x1 > -125.f ? exp2_poly(x1) : 0.f) : exp2_poly(fmaxf(x1, -125.f));
              } else {
                p0 = ex2_approx(x0);
                p1 = ex2_approx(x1);
              }
              r8[(c >> 1) & 7] += p0 + p1;
              pk[c / 2] = pack_bf16x2(p0, p1);
            }
          }
          ATR_SM(5);
          l = l * alpha + (((r8[0] + r8[1]) + (r8[2] + r8[3])) + ((r8[4] + r8[5]) + (r8[6] + r8[7])));
          if (j > 0 || pv_pending) {  // PV_{j-1} (or the previous tile's last PV) has consumed its P
            mbar_wait<false>(pv_done, pv_ph);
            pv_ph ^= 1;
            tc_fence_after();
            pv_pending = false;
          }
          ATR_SM(6);
          CORA_TMEM_ST_32X32B_X32(tmem_base + t_lane + kTmemP, pk);
          CORA_TMEM_ST_32X32B_X32(tmem_base + t_lane + kTmemP + 32, (pk + 32));
          // rescale the O accumulator in place when some row of this warp moved its reference max
          if (j > 0 && __any_sync(0xffffffffu, bump)) {
  #pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t orr[32];
              const uint32_t taddr = tmem_base + t_lane + kTmemO + half * 32;
              CORA_TMEM_LD_32X32B_X32(taddr, orr);
              tmem_ld_wait();
  #pragma unroll
              for (int c = 0; c < 32; ++c) orr[c] = __float_as_uint(__uint_as_float(orr[c]) * alpha);
              CORA_TMEM_ST_32X32B_X32(taddr, orr);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full);
          ATR_SM(7);
        }
        if constexpr (kEpiWG<CAUSAL>) {  // the epilogue warpgroup normalises and stores O
          hand_l(l);
          pv_pending = true;
          continue;
        }
        // epilogue: wait for the last PV, normalise, store the valid query rows of this tile
        mbar_wait<false>(pv_done, pv_ph);
        ATR_SM(8);
        pv_ph ^= 1;
        tc_fence_after();
        uint32_t orr[HD];
        CORA_TMEM_LD_32X32B_X32(tmem_base + t_lane + kTmemO, orr);
        CORA_TMEM_LD_32X32B_X32(tmem_base + t_lane + kTmemO + 32, (orr + 32));
        tmem_ld_wait();
        ATR_SM(13);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
        const int qrow = cur.qt * TQ + i;
#ifdef CORA_ATTN_PROF_NO_STORE  // profiling build only: O is not written
        if (qrow < L && l == 12345.f) {
#else
        if (qrow < L) {
#endif
          const float inv = rcp_fma(l);
          __nv_bfloat16* orow = out + static_cast<size_t>(cur.r0 + qrow) * d_model + cur.h * HD;
          if (out_v8) {  // 32-B stores: one full sector per lane
  #pragma unroll
            for (int g = 0; g < HD / 16; ++g) {
              const float* o = reinterpret_cast<const float*>(orr) + g * 16;
              uint32_t w[8];
  #pragma unroll
              for (int e = 0; e < 8; ++e) w[e] = pack_bf16x2(o[2 * e] * inv, o[2 * e + 1] * inv);
              st_global_v8(orow + g * 16, w);
            }
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow);
  #pragma unroll
            for (int g = 0; g < HD / 8; ++g) {
              const float* o = reinterpret_cast<const float*>(orr) + g * 8;
              dst[g] = make_uint4(pack_bf16x2(o[0] * inv, o[1] * inv), pack_bf16x2(o[2] * inv, o[3] * inv),
                                  pack_bf16x2(o[4] * inv, o[5] * inv), pack_bf16x2(o[6] * inv, o[7] * inv));
            }
          }
        }
        ATR_SM(10);
      }
    }
    if (qd == 0 && lane == 0) ATR_DONE(0);
  } else {
    // ------------------------------------------------------------ tile epilogue (bidirectional kernel)
    // Warp w reads TMEM lanes 32 (w % 4) ..: per tile, the row sum l of its row (shared memory, handed over
    // after the softmax warps stored the tile's last P -- by then every PV but the last has completed, so the
    // parity wait below is for that last PV), then O in four 16-column chunks; the O columns are released
    // to the MMA thread (the next tile's first PV) after the last chunk is read.
    if constexpr (kEpiWG<CAUSAL>) {
      setmaxnreg_dec<kRegsEpi>();
      tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_ptr);
      const uint32_t qd = warp & 3;
      const int i = qd * 32 + lane;
      const uint32_t t_lane = (qd * 32) << 16;
      const bool out_v8 = (reinterpret_cast<uintptr_t>(out) & 31u) == 0 && (d_model % 16) == 0;
      int pv_n = 0, l_n = 0;
      RingReader rw{ring_addr, ring_full, ring_empty, 0};
      for (int4 mt = rw.next(true); mt.x >= 0; mt = rw.next(true)) {
        const WorkUnit wu = decode_work<CAUSAL>(mt);
        for (int sub = 0; sub < wu.count; ++sub) {
          const WorkTile cur = wu.tile(sub);
          const int L = cur.L;
          pv_n += (L + TK - 1) / TK;
          mbar_wait<false>(l_full, l_n & 1);
          const float lv = lbuf[i];
          __syncwarp();
          if (lane == 0) mbar_arrive(l_empty);
          ++l_n;
          mbar_wait<false>(pv_done, (pv_n - 1) & 1);
          tc_fence_after();
          const int qrow = cur.qt * TQ + i;
          if (cur.qt * TQ + static_cast<int>(qd) * 32 < L) {
            const float inv = qrow < L ? rcp_fma(lv) : 0.f;
            __nv_bfloat16* orow = out + static_cast<size_t>(cur.r0 + qrow) * d_model + cur.h * HD;
  #pragma unroll
            for (int g = 0; g < HD / 16; ++g) {
              uint32_t r[16];
              CORA_TMEM_LD_32X32B_X16(tmem_base + t_lane + kTmemO + g * 16, r);
              tmem_ld_wait();
              if (g == HD / 16 - 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(o_empty);
              }
              if (qrow < L) {
                uint32_t w[8];
  #pragma unroll
                for (int e = 0; e < 8; ++e)
                  w[e] = pack_bf16x2(__uint_as_float(r[2 * e]) * inv, __uint_as_float(r[2 * e + 1]) * inv);
                if (out_v8) {
                  st_global_v8(orow + g * 16, w);
                } else {
                  uint4* dst = reinterpret_cast<uint4*>(orow + g * 16);
                  dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                  dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                }
              }
            }
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
  // the last CTA to finish resets the ticket counter for the next launch on this layout (every CTA has
  // claimed its last entry before it gets here; the next launch reads the counter after griddepcontrol.wait)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(n_tiles_ptr + 2, 1) == static_cast<int>(gridDim.x) - 1) {
      atomicExch(n_tiles_ptr + 1, 0);
      atomicExch(n_tiles_ptr + 2, 0);
    }
  }
  KSPAN_EXIT(attn, 1);
}

// ---------------------------------------------------------------- SIMT kernel for other head dims
// One warp per (token, head): online softmax over the keys of the token's own sequence, 32 keys
// at a time (lane = key), probabilities broadcast with shuffles, lane owns dims lane + 32k.
// Serves head_dim != 64 (e.g. the tiny C1 configuration, d_h = 8) where a 128x64 UMMA tile does
// not apply.
template <int DPL>  // dims per lane: head_dim <= 32 * DPL
__global__ void __launch_bounds__(256) attention_simt_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                             __nv_bfloat16* __restrict__ out,
                                                             const int32_t* __restrict__ lengths,
                                                             const int32_t* __restrict__ row_off,
                                                             const int32_t* __restrict__ seq_of_tok, int32_t T,
                                                             int32_t heads, int32_t hd, float scale, int causal) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wg >= static_cast<int64_t>(T) * heads) return;
  const int t = static_cast<int>(wg / heads), h = static_cast<int>(wg % heads);
  const int b = seq_of_tok[t];
  if (b < 0) return;
  const int r0 = row_off[b];
  const int L = causal ? (t - r0 + 1) : lengths[b];  // keys j < L of the sequence (j <= i when causal)
  const int d = heads * hd, ld = 3 * d;
  const __nv_bfloat16* q = qkv + static_cast<size_t>(t) * ld + h * hd;
  float m = -INFINITY, l = 0.f, o[DPL];
#pragma unroll
  for (int k = 0; k < DPL; ++k) o[k] = 0.f;
  for (int j0 = 0; j0 < L; j0 += 32) {
    const int j = j0 + lane;
    float s = -INFINITY;
    if (j < L) {
      const __nv_bfloat16* kr = qkv + static_cast<size_t>(r0 + j) * ld + d + h * hd;
      float acc = 0.f;
      for (int c = 0; c < hd; ++c) acc += __bfloat162float(q[c]) * __bfloat162float(kr[c]);
      s = acc * scale;
    }
    float mx = s;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float m_new = fmaxf(m, mx);
    const float alpha = __expf(m - m_new);
    const float p = j < L ? __expf(s - m_new) : 0.f;
    float ps = p;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l = l * alpha + ps;
    m = m_new;
#pragma unroll
    for (int k = 0; k < DPL; ++k) o[k] *= alpha;
    const int nk = min(32, L - j0);
    for (int jj = 0; jj < nk; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
      const __nv_bfloat16* vr = qkv + static_cast<size_t>(r0 + j0 + jj) * ld + 2 * d + h * hd;
#pragma unroll
      for (int k = 0; k < DPL; ++k) {
        const int c = lane + 32 * k;
        if (c < hd) o[k] += pj * __bfloat162float(vr[c]);
      }
    }
  }
  __nv_bfloat16* dst = out + static_cast<size_t>(t) * d + h * hd;
#pragma unroll
  for (int k = 0; k < DPL; ++k) {
    const int c = lane + 32 * k;
    if (c < hd) dst[c] = __float2bfloat16_rn(o[k] / l);
  }
}

}  // namespace

#ifdef CORA_ATTN_TRACE
extern "C" int cora_debug_attn_trace(void* dst, void* counts) {
  cudaMemcpyFromSymbol(dst, g_attn_trace, sizeof(g_attn_trace));
  cudaMemcpyFromSymbol(counts, g_attn_trace_n, sizeof(g_attn_trace_n));
  static int z[kTraceCtas][2] = {};
  return cudaMemcpyToSymbol(g_attn_trace_n, z, sizeof(z));
}
#endif

cudaError_t launch_attention(const cora_layout_t& L, const void* qkv, void* o, int32_t head_dim, float scale,
                             cudaStream_t stream, bool causal) {
  if (L.total_tokens == 0 || L.batch == 0) return cudaSuccess;
  const int32_t d = L.heads * head_dim;
  if (head_dim == HD) {
    CUtensorMap tm;
    if (!make_tmap_2d_bf16(&tm, qkv, 3ull * d, L.total_tokens, 3ull * d * 2, HD, TQ, true))
      return cudaErrorInvalidValue;
    static bool attr_set[kMaxDevices] = {};
    const int dev = current_device();
    if (!attr_set[dev]) {
      for (auto k : {attention_fwd_kernel<false>, attention_fwd_kernel<true>}) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem::kAlloc);
        if (e != cudaSuccess) return e;
      }

      attr_set[dev] = true;
    }
    const int max_grid = 2 * device_sm_count();
    const int grid = L.n_tiles_max < max_grid ? L.n_tiles_max : max_grid;
    if (grid == 0) return cudaSuccess;
    const float scale_log2 = scale * 1.4426950408889634f;
    if (causal) {
      const int ugrid = L.n_units_max < max_grid ? L.n_units_max : max_grid;
      return launch_pdl(attention_fwd_kernel<true>, dim3(ugrid > 0 ? ugrid : 1), dim3(kThreadsOf<true>), AttnSmem::kAlloc,
                        stream, 1, tm, L.units, reinterpret_cast<const int2*>(L.unit_seq), L.n_units,
                        L.seq_of_tok, L.pos_in_seq, L.lengths, static_cast<__nv_bfloat16*>(o), d, scale_log2);
    }
    return launch_pdl(attention_fwd_kernel<false>, dim3(grid), dim3(kThreadsOf<false>), AttnSmem::kAlloc, stream, 1, tm,
                      L.tiles, reinterpret_cast<const int2*>(L.tile_seq), L.n_tiles, L.seq_of_tok, L.pos_in_seq,
                      L.lengths, static_cast<__nv_bfloat16*>(o), d, scale_log2);
  }
  const int64_t warps = static_cast<int64_t>(L.total_tokens) * L.heads;
  const dim3 block(256), grid(static_cast<unsigned>((warps + 7) / 8));
  auto q = static_cast<const __nv_bfloat16*>(qkv);
  auto out = static_cast<__nv_bfloat16*>(o);
  if (head_dim <= 32)
    attention_simt_kernel<1><<<grid, block, 0, stream>>>(q, out, L.lengths, L.row_off, L.seq_of_tok,
                                                         L.total_tokens, L.heads, head_dim, scale, causal ? 1 : 0);
  else
    attention_simt_kernel<4><<<grid, block, 0, stream>>>(q, out, L.lengths, L.row_off, L.seq_of_tok,
                                                         L.total_tokens, L.heads, head_dim, scale, causal ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace cora
