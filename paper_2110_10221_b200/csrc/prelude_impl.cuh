// The prelude's device code (step a1), shared by the prelude kernels (prelude.cu) and the QKV GEMM, whose
// epilogue warps run it before their first unit in the one-call forward (cora_encoder_forward, batch <= 256).
// prelude.cu has the algorithm and its citations.
#pragma once
#include <cstdint>

#include "cora_internal.h"

namespace cora {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kMaxBuckets = 129;  // ceil(16383/128) + 1 distinct q-tile counts
constexpr int kPackMaxBatch = CORA_PACK_MAX_BATCH;  // short-sequence windows (merged prelude, batch <= this)

// A team of whole warps that runs the prelude: the CTA (CtaTeam) or some warps of a CTA synchronised by a
// named barrier (WarpTeam: the QKV GEMM's epilogue warps before their first unit).
struct CtaTeam {
  __device__ __forceinline__ int tid() const { return static_cast<int>(threadIdx.x); }
  __device__ __forceinline__ int size() const { return static_cast<int>(blockDim.x); }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct WarpTeam {
  int first;  // first thread of the team (a multiple of 32)
  int n;      // threads (a multiple of 32)
  int bar;    // named barrier id
  __device__ __forceinline__ int tid() const { return static_cast<int>(threadIdx.x) - first; }
  __device__ __forceinline__ int size() const { return n; }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(n) : "memory"); }
};

template <typename T, class Team>
__device__ T block_exclusive_scan(T v, T* warp_sums, T& total, const Team& team) {
  const int lane = team.tid() & 31, wid = team.tid() >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const int nwarps = team.size() >> 5;
  if (lane == 31) warp_sums[wid] = x;
  team.sync();
  if (wid == 0) {
    T s = lane < nwarps ? warp_sums[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s;  // inclusive over warps
  }
  team.sync();
  T warp_prefix = wid ? warp_sums[wid - 1] : T(0);
  total = warp_sums[31];
  team.sync();
  return warp_prefix + x - v;
}

// The scans, validation and longest-first lists of the whole batch, computed by one CTA.  With nparts > 1
// (merged prelude) every CTA of the grid runs it redundantly (the batch is small), CTA `part` writes
// the list entries of sequences b with b % nparts == part, and CTA 0 alone writes the per-batch arrays
// (row_off, attn_off, counts, status); s_off (shared, [batch + 1]) receives the exclusive prefix of the
// clamped lengths when non-NULL.  Returns the status word.
// Shared memory of one prelude team; CAP = the largest team size (per-thread arrays).
template <int CAP>
struct PreludeSmem {
  static constexpr int kPackCap = (kPackMaxBatch < CAP ? kPackMaxBatch : CAP) > 0 ? (kPackMaxBatch < CAP ? kPackMaxBatch : CAP) : 1;
  int64_t ws64[32];
  int32_t ws32[32];
  int32_t hist[kMaxBuckets];
  int32_t bucket_base[kMaxBuckets];
  int32_t unit_base[kMaxBuckets];
  int32_t running[kMaxBuckets];
  int32_t warp_cnt[CAP / 32][kMaxBuckets];
  int32_t s_bad;
  unsigned long long s_raw_sum;  // sum of the raw (unclamped) lengths, for the T check
  int32_t s_first[CAP], s_ufirst[CAP];  // per sequence of the current chunk
  int2 s_seq[CAP];
  // short-sequence windows (SURVEY f-4, reading f4-r1): (first sequence | packed << 31, tokens)
  int2 s_win[kPackCap];
  int32_t s_len[kPackCap];
  int32_t s_nwin, s_tot, s_utot;
};

template <int CAP, class Team>
__device__ __forceinline__ int32_t layout_scan_block(const Team& team, PreludeSmem<CAP>& sm,
                                                     const int32_t* __restrict__ lengths, int32_t batch,
                                                                   int32_t total_tokens, int32_t heads,
                                                                   int32_t max_len, int32_t* __restrict__ row_off,
                                                                   int64_t* __restrict__ attn_off,
                                                                   int32_t* __restrict__ tiles,
                                                                   int32_t* __restrict__ tile_seq,
                                                                   int32_t* __restrict__ n_tiles,
                                                                   int32_t* __restrict__ units,
                                                                   int32_t* __restrict__ unit_seq,
                                                                   int32_t* __restrict__ n_units,
                                                                   int32_t* __restrict__ status,
                                                                   int part, int nparts, int32_t* s_off) {
  auto& ws64 = sm.ws64;
  auto& ws32 = sm.ws32;
  auto& hist = sm.hist;
  auto& bucket_base = sm.bucket_base;
  auto& unit_base = sm.unit_base;
  auto& running = sm.running;
  auto& warp_cnt = sm.warp_cnt;
  auto& s_bad = sm.s_bad;
  auto& s_raw_sum = sm.s_raw_sum;
  auto& s_first = sm.s_first;
  auto& s_ufirst = sm.s_ufirst;
  auto& s_seq = sm.s_seq;
  auto& s_win = sm.s_win;
  auto& s_len = sm.s_len;
  auto& s_nwin = sm.s_nwin;
  auto& s_tot = sm.s_tot;
  auto& s_utot = sm.s_utot;
  const bool pack = s_off != nullptr && batch <= kPackMaxBatch && batch <= PreludeSmem<CAP>::kPackCap &&
                    batch <= team.size();

  const int tid = team.tid(), lane = tid & 31, wid = tid >> 5;
  const int nthreads = team.size(), nwarps = nthreads >> 5;
  for (int i = tid; i < kMaxBuckets; i += nthreads) {
    hist[i] = 0;
    running[i] = 0;
  }
  if (tid == 0) {
    s_bad = 0;
    s_raw_sum = 0ull;
  }
  team.sync();

  // ---- pass 1: prefix sums (A_1 arrays) + validation + bucket histogram
  int32_t carry32 = 0;
  int64_t carry64 = 0;
  for (int base = 0; base < batch; base += nthreads) {
    const int b = base + tid;
    int32_t L = 0;
    if (b < batch) {
      L = lengths[b];
      if (L < 0 || L > max_len) {
        s_bad = 1;  // benign race: every writer stores 1
        L = L < 0 ? 0 : max_len;
      }
    }
    // raw (unclamped) sum for the T check: warp reduction, one shared atomic per warp
    {
      int64_t raw = (b < batch) ? static_cast<int64_t>(lengths[b]) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) raw += __shfl_xor_sync(0xffffffffu, raw, o);
      if (lane == 0 && raw != 0) atomicAdd(&s_raw_sum, static_cast<unsigned long long>(raw));
    }
    int32_t tot32;
    int64_t tot64;
    const int32_t ex32 = block_exclusive_scan<int32_t>(L, ws32, tot32, team);
    const int64_t ex64 = block_exclusive_scan<int64_t>(static_cast<int64_t>(L) * L, ws64, tot64, team);
    if (b < batch && part == 0) {
      row_off[b] = carry32 + ex32;
      attn_off[b] = carry64 + ex64;
    }
    if (b < batch && s_off != nullptr) s_off[b] = carry32 + ex32;
    if (b < batch && pack) s_len[b] = L;
    {  // bucket histogram: one shared atomic per distinct bucket per warp
      const int32_t v = (b < batch) ? (L + CORA_TILE_ROWS - 1) / CORA_TILE_ROWS : -1;
      const uint32_t same = __match_any_sync(0xffffffffu, v);
      if (v >= 0 && (same & ((1u << lane) - 1u)) == 0) atomicAdd(&hist[v], __popc(same));
    }
    carry32 += tot32;
    carry64 += tot64;
  }
  team.sync();
  int32_t st = 0;
  if (s_bad) st |= CORA_STATUS_BAD_LENGTH;
  if (static_cast<int64_t>(s_raw_sum) != total_tokens) st |= CORA_STATUS_SUM_MISMATCH;
  if (wid == 0) {
    // bucket bases in descending tile-count order: exclusive scan of heads*v*hist[v] from v = 128
    // down to 0, 32 buckets per step
    // (units: the same with ceil(v / 2) pairs per (sequence, head))
    int32_t carry = 0, ucarry = 0;
    for (int base = 0; base < kMaxBuckets; base += 32) {
      const int v = kMaxBuckets - 1 - (base + lane);
      const int32_t x = v >= 0 ? heads * v * hist[v] : 0;
      const int32_t ux = v >= 0 ? heads * ((v + 1) / 2) * hist[v] : 0;
      int32_t incl = x, uincl = ux;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        const int32_t uy = __shfl_up_sync(0xffffffffu, uincl, o);
        if (lane >= o) incl += y, uincl += uy;
      }
      if (v >= 0) bucket_base[v] = carry + incl - x, unit_base[v] = ucarry + uincl - ux;
      carry += __shfl_sync(0xffffffffu, incl, 31);
      ucarry += __shfl_sync(0xffffffffu, uincl, 31);
    }
    if (lane == 0) s_tot = carry, s_utot = ucarry;
    if (lane == 0 && s_off != nullptr) s_off[batch] = carry32;
  }
  team.sync();
  if (pack) {
    // Greedy windows in batch order (oracle.short_windows), computed in parallel (one sequence per
    // thread, batch <= blockDim): a window opened by short sequence b (1 <= L <= 128) takes every
    // following sequence until the first one that overflows 128 tokens, end(b) (a long sequence always
    // does; zero-length ones never do) -- a binary search over the prefix sums.  The windows are the
    // short sequences on the chain 0 -> nxt -> nxt ... with nxt(b) = end(b) for a short b and b + 1
    // otherwise; the chain is marked by pointer doubling (ceil(log2 batch) rounds).
    int32_t* jmp = s_first;   // scratch: pass 2 reuses these arrays afterwards
    int32_t* on = s_ufirst;
    const int b = tid;
    int32_t Lb = 0, end = batch;
    if (b < batch) {
      Lb = s_len[b];
      if (Lb >= 1 && Lb <= CORA_TILE_ROWS) {
        int lo = b + 1, hi = batch;  // end = first j in [b+1, batch) with off[j+1] - off[b] > 128
        const int base_off = s_off[b];
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_off[mid + 1] - base_off > CORA_TILE_ROWS) hi = mid; else lo = mid + 1;
        }
        end = lo;
        jmp[b] = end;
      } else {
        jmp[b] = b + 1;
      }
      on[b] = b == 0;
    }
    team.sync();
    for (int span = 1; span < batch; span <<= 1) {
      const int nb = b < batch ? jmp[b] : batch;
      if (b < batch && on[b] && nb < batch) on[nb] = 1;
      const int nn = (b < batch && nb < batch) ? jmp[nb] : batch;
      team.sync();
      if (b < batch) jmp[b] = nn;
      team.sync();
    }
    const bool start = b < batch && on[b] && Lb >= 1 && Lb <= CORA_TILE_ROWS;
    int32_t n_win;
    const int32_t idx = block_exclusive_scan<int32_t>(start ? 1 : 0, ws32, n_win, team);
    if (start) {
      const int32_t W = s_off[end] - s_off[b];
      s_win[idx] = make_int2(b | (W > Lb ? static_cast<int>(0x80000000u) : 0), W);
    }
    if (tid == 0) s_nwin = n_win;
  }
  team.sync();
  if (tid == 0 && part == 0) {
    row_off[batch] = carry32;
    attn_off[batch] = carry64;
    *status = st;
    // packed: the one-tile sequences' heads * hist[1] entries become heads * (windows) entries
    *n_tiles = st ? 0 : (pack ? bucket_base[1] + heads * s_nwin : s_tot);
    *n_units = st ? 0 : (pack ? unit_base[1] + heads * s_nwin : s_utot);
    // the attention kernels' dynamic schedule words (ticket, finished CTAs) live after each count
    n_tiles[1] = n_tiles[2] = 0;
    n_units[1] = n_units[2] = 0;
  }
  if (st) return st;  // data error: empty work list, nothing else is read
  const int32_t* roff = s_off != nullptr ? s_off : row_off;  // this CTA's copy of the exclusive prefix

  // ---- pass 2: stable rank of each sequence inside its bucket -> tile list
  for (int base = 0; base < batch; base += nthreads) {
    const int b = base + tid;
    const bool valid = b < batch;
    const int32_t L = valid ? lengths[b] : 0;
    const int32_t v = valid ? (L + CORA_TILE_ROWS - 1) / CORA_TILE_ROWS : -1;
    for (int i = tid; i < nwarps * kMaxBuckets; i += nthreads) (&warp_cnt[0][0])[i] = 0;
    team.sync();
    const uint32_t same = __match_any_sync(0xffffffffu, v);
    const int rank_in_warp = __popc(same & ((1u << lane) - 1u));
    if (valid && rank_in_warp == 0) warp_cnt[wid][v] = __popc(same);
    team.sync();
    s_first[tid] = -1;
    if (valid && v > (pack ? 1 : 0)) {
      int32_t rank = running[v] + rank_in_warp;
      for (int w = 0; w < wid; ++w) rank += warp_cnt[w][v];
      s_first[tid] = bucket_base[v] + rank * heads * v;
      s_ufirst[tid] = unit_base[v] + rank * heads * ((v + 1) / 2);
      s_seq[tid] = make_int2(roff[b], L);
    }
    team.sync();
    // each warp writes whole sequences' entries (heads * v tiles, heads * ceil(v/2) units), lanes over
    // consecutive entries: coalesced stores instead of one thread streaming a sequence's entries alone
    // (this CTA's sequences: b % nparts == part, spread over the warps)
    const int j0 = (part - base % nparts + nparts) % nparts;
    for (int j = j0 + wid * nparts; j < nthreads && base + j < batch; j += nwarps * nparts) {
      const int32_t first = s_first[j];
      if (first < 0) continue;
      const int bj = base + j;
      const int2 seq = s_seq[j];
      const int32_t vj = (seq.y + CORA_TILE_ROWS - 1) / CORA_TILE_ROWS, np = (vj + 1) / 2;
      for (int k = lane; k < heads * vj; k += 32) {
        tiles[first + k] = bj | ((k / vj) << 16) | ((k % vj) << 24);
        reinterpret_cast<int2*>(tile_seq)[first + k] = seq;
      }
      const int32_t ufirst = s_ufirst[j];
      for (int k = lane; k < heads * np; k += 32) {
        units[ufirst + k] = bj | ((k / np) << 16) | ((k % np) << 24);
        reinterpret_cast<int2*>(unit_seq)[ufirst + k] = seq;
      }
    }
    team.sync();
    for (int u = tid; u < kMaxBuckets; u += nthreads) {
      int32_t s = 0;
      for (int w = 0; w < nwarps; ++w) s += warp_cnt[w][u];
      running[u] += s;
    }
    team.sync();
  }
  if (pack) {
    // window entries (this CTA's windows: w % nparts == part), one per (window, head), after the
    // multi-tile sequences' entries, ordered (first sequence, head) like every other bucket
    const int nw = s_nwin;
    for (int w = part + wid * nparts; w < nw; w += nwarps * nparts) {
      const int2 win = s_win[w];
      const int b0 = win.x & 0x7FFFFFFF;
      const int2 seq = make_int2(roff[b0], win.y);
      for (int k = lane; k < heads; k += 32) {
        const int32_t word = win.x | (k << 16);
        tiles[bucket_base[1] + w * heads + k] = word;
        reinterpret_cast<int2*>(tile_seq)[bucket_base[1] + w * heads + k] = seq;
        units[unit_base[1] + w * heads + k] = word;
        reinterpret_cast<int2*>(unit_seq)[unit_base[1] + w * heads + k] = seq;
      }
    }
  }
  return st;
}

// One part (of nparts) of the merged prelude: the (redundant) scans, this part's share of the tile / unit lists,
// and f_fo / f_fi for this part's sequences.  s_off: shared [batch + 1].
template <int CAP, class Team>
__device__ __forceinline__ void prelude_part(const Team& team, PreludeSmem<CAP>& sm, int32_t* s_off,
                                             const PreludeArgs& a, int part, int nparts) {
  const int32_t st = layout_scan_block<CAP>(team, sm, a.lengths, a.batch, a.total_tokens, a.heads, a.max_len,
                                            a.row_off, a.attn_off, a.tiles, a.tile_seq, a.n_tiles, a.units,
                                            a.unit_seq, a.n_units, a.status, part, nparts, s_off);
  const int tid = team.tid(), lane = tid & 31;
  if (st != 0) {  // data error: the maps say "no sequence" everywhere
    for (int t = part * team.size() + tid; t < a.total_tokens; t += nparts * team.size()) {
      a.seq_of_tok[t] = -1;
      a.pos_in_seq[t] = -1;
    }
    return;
  }
  // f_fo / f_fi by sequence: warp w of the grid fills sequences w, w + n_warps, ...; lanes write
  // consecutive tokens of a sequence (coalesced, no search)
  const int wpb = team.size() >> 5;
  const int n_warps = nparts * wpb;
  for (int b = part * wpb + (tid >> 5); b < a.batch; b += n_warps) {
    const int o = s_off[b], L = s_off[b + 1] - o;
    for (int i = lane; i < L; i += 32) {
      a.seq_of_tok[o + i] = b;
      a.pos_in_seq[o + i] = i;
    }
  }
}

}  // namespace
}  // namespace cora
