// Step a1: the "prelude" of CoRa as device kernels.
//
// CoRa builds its auxiliary arrays (A_d prefix sums, App. B.1, and the
// vloop-fusion maps f_fo / f_fi / f_oif, App. B.2) on the HOST and copies
// them to the GPU; that copy is "the major source of the overhead".
// Here the tables are computed on the device from the lengths, so only B lengths (or nothing,
// if they already live on the GPU) cross PCIe.
//
//   kernel 1 (one CTA, 1024 threads): block scans of L and L^2 -> row_off, attn_off;
//            validation -> status; longest-first attention tile list (PAPER.md:1747-1750,
//            reading c15: key (-ceil(L/128), b, h, qt)) by a stable counting sort.
//   kernel 2 (grid over T): f_fo / f_fi by binary search of row_off.
#include <cstdint>

#include "cora_internal.h"
#include "ptx.cuh"

CORA_KSPAN_DEFINE(prelude)

namespace cora {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kMaxBuckets = 129;  // ceil(16383/128) + 1 distinct q-tile counts
constexpr int kPackMaxBatch = CORA_PACK_MAX_BATCH;  // short-sequence windows (merged prelude, batch <= this)

template <typename T>
__device__ T block_exclusive_scan(T v, T* warp_sums, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const int nwarps = blockDim.x >> 5;
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nwarps ? warp_sums[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  T warp_prefix = wid ? warp_sums[wid - 1] : T(0);
  total = warp_sums[31];
  __syncthreads();
  return warp_prefix + x - v;
}

// The scans, validation and longest-first lists of the whole batch, computed by one CTA.  With nparts > 1
// (merged prelude) every CTA of the grid runs it redundantly (the batch is small), CTA `part` writes
// the list entries of sequences b with b % nparts == part, and CTA 0 alone writes the per-batch arrays
// (row_off, attn_off, counts, status); s_off (shared, [batch + 1]) receives the exclusive prefix of the
// clamped lengths when non-NULL.  Returns the status word.
__device__ __forceinline__ int32_t layout_scan_block(const int32_t* __restrict__ lengths, int32_t batch,
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
  __shared__ int64_t ws64[32];
  __shared__ int32_t ws32[32];
  __shared__ int32_t hist[kMaxBuckets];
  __shared__ int32_t bucket_base[kMaxBuckets];
  __shared__ int32_t unit_base[kMaxBuckets];
  __shared__ int32_t running[kMaxBuckets];
  __shared__ int32_t warp_cnt[32][kMaxBuckets];
  __shared__ int32_t s_bad;
  __shared__ unsigned long long s_raw_sum;  // sum of the raw (unclamped) lengths, for the T check
  __shared__ int32_t s_first[kScanThreads], s_ufirst[kScanThreads];  // per sequence of the current chunk
  __shared__ int2 s_seq[kScanThreads];
  // short-sequence windows (SURVEY f-4, reading f4-r1): (first sequence | packed << 31, tokens)
  __shared__ int2 s_win[kPackMaxBatch > 0 ? kPackMaxBatch : 1];
  __shared__ int32_t s_len[kPackMaxBatch > 0 ? kPackMaxBatch : 1];
  __shared__ int32_t s_nwin, s_tot, s_utot;
  const bool pack = s_off != nullptr && batch <= kPackMaxBatch && batch <= static_cast<int>(blockDim.x);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nthreads = blockDim.x, nwarps = nthreads >> 5;
  for (int i = tid; i < kMaxBuckets; i += nthreads) {
    hist[i] = 0;
    running[i] = 0;
  }
  if (tid == 0) {
    s_bad = 0;
    s_raw_sum = 0ull;
  }
  __syncthreads();

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
    const int32_t ex32 = block_exclusive_scan<int32_t>(L, ws32, tot32);
    const int64_t ex64 = block_exclusive_scan<int64_t>(static_cast<int64_t>(L) * L, ws64, tot64);
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
  __syncthreads();
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
  __syncthreads();
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
    __syncthreads();
    for (int span = 1; span < batch; span <<= 1) {
      const int nb = b < batch ? jmp[b] : batch;
      if (b < batch && on[b] && nb < batch) on[nb] = 1;
      const int nn = (b < batch && nb < batch) ? jmp[nb] : batch;
      __syncthreads();
      if (b < batch) jmp[b] = nn;
      __syncthreads();
    }
    const bool start = b < batch && on[b] && Lb >= 1 && Lb <= CORA_TILE_ROWS;
    int32_t n_win;
    const int32_t idx = block_exclusive_scan<int32_t>(start ? 1 : 0, ws32, n_win);
    if (start) {
      const int32_t W = s_off[end] - s_off[b];
      s_win[idx] = make_int2(b | (W > Lb ? static_cast<int>(0x80000000u) : 0), W);
    }
    if (tid == 0) s_nwin = n_win;
  }
  __syncthreads();
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
    __syncthreads();
    const uint32_t same = __match_any_sync(0xffffffffu, v);
    const int rank_in_warp = __popc(same & ((1u << lane) - 1u));
    if (valid && rank_in_warp == 0) warp_cnt[wid][v] = __popc(same);
    __syncthreads();
    s_first[tid] = -1;
    if (valid && v > (pack ? 1 : 0)) {
      int32_t rank = running[v] + rank_in_warp;
      for (int w = 0; w < wid; ++w) rank += warp_cnt[w][v];
      s_first[tid] = bucket_base[v] + rank * heads * v;
      s_ufirst[tid] = unit_base[v] + rank * heads * ((v + 1) / 2);
      s_seq[tid] = make_int2(roff[b], L);
    }
    __syncthreads();
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
    __syncthreads();
    for (int u = tid; u < kMaxBuckets; u += nthreads) {
      int32_t s = 0;
      for (int w = 0; w < nwarps; ++w) s += warp_cnt[w][u];
      running[u] += s;
    }
    __syncthreads();
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

__global__ void __launch_bounds__(kScanThreads) layout_scan_kernel(const int32_t* __restrict__ lengths, int32_t batch,
                                                                   int32_t total_tokens, int32_t heads,
                                                                   int32_t max_len, int32_t* __restrict__ row_off,
                                                                   int64_t* __restrict__ attn_off,
                                                                   int32_t* __restrict__ tiles,
                                                                   int32_t* __restrict__ tile_seq,
                                                                   int32_t* __restrict__ n_tiles,
                                                                   int32_t* __restrict__ units,
                                                                   int32_t* __restrict__ unit_seq,
                                                                   int32_t* __restrict__ n_units,
                                                                   int32_t* __restrict__ status) {
  layout_scan_block(lengths, batch, total_tokens, heads, max_len, row_off, attn_off, tiles, tile_seq, n_tiles, units,
                    unit_seq, n_units, status, 0, 1, nullptr);
}

constexpr int kMergedMaxBatch = 8192;   // merged single-launch prelude: row_off kept in smem per block
constexpr int kSeqPerBlock = 4;   // merged prelude: sequences per CTA (lists and maps)

// One launch for the whole prelude (batch <= kMergedMaxBatch): every CTA recomputes the (small) scans
// and bucket ranks of the whole batch in shared memory instead of waiting for one CTA to publish them,
// then writes its share of the tile / unit lists and of f_fo / f_fi (one CTA writing every list
// entry alone took ~15k cycles at bs 128: the store stream of a single SM, not the arithmetic, bound it).
__global__ void __launch_bounds__(kScanThreads) layout_merged_kernel(
    const int32_t* __restrict__ lengths, int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len,
    int32_t* __restrict__ row_off, int64_t* __restrict__ attn_off, int32_t* __restrict__ tiles,
    int32_t* __restrict__ tile_seq, int32_t* __restrict__ n_tiles, int32_t* __restrict__ units,
    int32_t* __restrict__ unit_seq, int32_t* __restrict__ n_units, int32_t* __restrict__ status,
    int32_t* __restrict__ seq_of_tok, int32_t* __restrict__ pos_in_seq) {
  KSPAN_ENTRY(prelude, 0);
  pdl_wait();  // the lengths may come from the previous kernel
  KSPAN_WAITED(prelude, 0);
  pdl_trigger();
  extern __shared__ int32_t s_off[];  // [batch + 1] exclusive prefix of the (clamped) lengths
  const int32_t st = layout_scan_block(lengths, batch, total_tokens, heads, max_len, row_off, attn_off, tiles,
                                       tile_seq, n_tiles, units, unit_seq, n_units, status, blockIdx.x, gridDim.x,
                                       s_off);
  const int tid = threadIdx.x, lane = tid & 31;
  if (st != 0) {  // data error: the maps say "no sequence" everywhere
    for (int t = blockIdx.x * blockDim.x + tid; t < total_tokens; t += gridDim.x * blockDim.x) {
      seq_of_tok[t] = -1;
      pos_in_seq[t] = -1;
    }
    return;
  }
  // f_fo / f_fi by sequence: warp w of the grid fills sequences w, w + n_warps, ...; lanes write
  // consecutive tokens of a sequence (coalesced, no search)
  const int wpb = static_cast<int>(blockDim.x) >> 5;
  const int n_warps = gridDim.x * wpb;
  for (int b = blockIdx.x * wpb + (tid >> 5); b < batch; b += n_warps) {
    const int o = s_off[b], L = s_off[b + 1] - o;
    for (int i = lane; i < L; i += 32) {
      seq_of_tok[o + i] = b;
      pos_in_seq[o + i] = i;
    }
  }
  KSPAN_EXIT(prelude, 0);
}

// f_fo / f_fi: for token t, b = max{b : row_off[b] <= t} (skips empty sequences), i = t - row_off[b].
__global__ void fusion_maps_kernel(const int32_t* __restrict__ row_off, const int32_t* __restrict__ status,
                                   int32_t batch, int32_t total_tokens, int32_t* __restrict__ seq_of_tok,
                                   int32_t* __restrict__ pos_in_seq) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total_tokens) return;
  if (*status != 0) {
    seq_of_tok[t] = -1;
    pos_in_seq[t] = -1;
    return;
  }
  int lo = 0, hi = batch;  // invariant: row_off[lo] <= t < row_off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (row_off[mid] <= t)
      lo = mid;
    else
      hi = mid;
  }
  seq_of_tok[t] = lo;
  pos_in_seq[t] = t - row_off[lo];
}

}  // namespace

cudaError_t launch_layout_build(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, const cora_layout_t& L, cudaStream_t stream) {
  // one CTA of the scan sized to the batch (>= 1 warp, <= 1024 threads; larger batches loop in chunks)
  int threads = ((batch + 31) / 32) * 32;
  threads = threads < 32 ? 32 : (threads > kScanThreads ? kScanThreads : threads);
  if (batch <= kMergedMaxBatch) {
    if (threads < 256) threads = 256;  // the map blocks share the block size
    int blocks = (batch + kSeqPerBlock - 1) / kSeqPerBlock;
    if (blocks > device_sm_count()) blocks = device_sm_count();
    if (blocks < 1) blocks = 1;
    static bool attr_set[kMaxDevices] = {};  // static (~36 KB) + dynamic (up to 32 KB) smem exceeds the 48 KB default
    const int dev = current_device();
    if (!attr_set[dev]) {
      const cudaError_t e = cudaFuncSetAttribute(layout_merged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 sizeof(int32_t) * (kMergedMaxBatch + 1));
      if (e != cudaSuccess) return e;
      attr_set[dev] = true;
    }
    return launch_pdl(layout_merged_kernel, dim3(blocks), dim3(threads), sizeof(int32_t) * (batch + 1), stream, 1,
               lengths, batch, total_tokens, heads, max_len, L.row_off, L.attn_off, L.tiles, L.tile_seq, L.n_tiles,
               L.units, L.unit_seq, L.n_units, L.status, L.seq_of_tok, L.pos_in_seq);
  }
  layout_scan_kernel<<<1, threads, 0, stream>>>(lengths, batch, total_tokens, heads, max_len, L.row_off, L.attn_off,
                                                L.tiles, L.tile_seq, L.n_tiles, L.units, L.unit_seq, L.n_units,
                                                L.status);
  if (total_tokens > 0) {
    const int mt = 256;
    fusion_maps_kernel<<<(total_tokens + mt - 1) / mt, mt, 0, stream>>>(L.row_off, L.status, batch, total_tokens,
                                                                         L.seq_of_tok, L.pos_in_seq);
  }
  return cudaGetLastError();
}

}  // namespace cora
