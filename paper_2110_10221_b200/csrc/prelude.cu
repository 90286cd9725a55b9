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
// Batches of <= 8192 sequences run ONE merged kernel instead (layout_merged_kernel: every CTA recomputes the
// scans, writes its share of the lists and maps).  The device code lives in prelude_impl.cuh, parameterised
// by the team of warps that runs it, so the one-call forward can run the same parts inside the QKV GEMM's
// epilogue warps (batches <= 256; gemm.cu, api.cu forward_impl).
#include <cstdint>

#include "cora_internal.h"
#include "prelude_impl.cuh"
#include "ptx.cuh"

CORA_KSPAN_DEFINE(prelude)

namespace cora {

namespace {

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
  __shared__ PreludeSmem<kScanThreads> sm;
  layout_scan_block<kScanThreads>(CtaTeam{}, sm, lengths, batch, total_tokens, heads, max_len, row_off, attn_off,
                                  tiles, tile_seq, n_tiles, units, unit_seq, n_units, status, 0, 1, nullptr);
}

constexpr int kMergedMaxBatch = 8192;   // merged single-launch prelude: row_off kept in smem per block
constexpr int kSeqPerBlock = 4;   // merged prelude: sequences per CTA (lists and maps)

// One launch for the whole prelude (batch <= kMergedMaxBatch): every CTA recomputes the (small) scans
// and bucket ranks of the whole batch in shared memory instead of waiting for one CTA to publish them,
// then writes its share of the tile / unit lists and of f_fo / f_fi (one CTA writing every list
// entry alone took ~15k cycles at bs 128: the store stream of a single SM, not the arithmetic, bound it).
__global__ void __launch_bounds__(kScanThreads) layout_merged_kernel(const PreludeArgs a) {
  KSPAN_ENTRY(prelude, 0);
  pdl_wait();  // the lengths may come from the previous kernel
  KSPAN_WAITED(prelude, 0);
  pdl_trigger();
  __shared__ PreludeSmem<kScanThreads> sm;
  extern __shared__ int32_t s_off[];  // [batch + 1] exclusive prefix of the (clamped) lengths
  prelude_part<kScanThreads>(CtaTeam{}, sm, s_off, a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
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
                      prelude_args(lengths, batch, total_tokens, heads, max_len, L));
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
