// Host logic of the sequence-sharded multi-GPU path: the FLOP-balanced
// contiguous shard plan and the split of every rank's range into the groups whose outputs are gathered
// while the next group computes.  No device code: callable without a GPU (tested on CPU).
//
// BASELINE.json north_star: "The batch is partitioned across the 8 GPUs of one box by sequence, balanced on
// sum(L_i d + L_i^2) FLOPs."  cost(L) = 2 L (4 d^2 + 2 d d_ff) + 4 d L^2 is the sequence's useful FLOPs.
// Readings s1 / s2: contiguous ranges, minimal max rank cost, canonical greedy-left; and cuts
// only where no short-sequence window (reading f4-r1; batches of <= CORA_PACK_MAX_BATCH sequences) spans,
// so every rank (and every group) rebuilds exactly the one-GPU windows of its sequences.
#include <cstdint>
#include <vector>

#include "cora_internal.h"

namespace {

// allowed[c], c in 0..B: may a boundary fall before sequence c?  The device prelude's windows (prelude.cu,
// oracle.short_windows): a sequence with 1 <= L <= 128 joins the open window while it stays <= 128 tokens,
// a longer one closes it, zero-length ones are transparent.  Forbidden: between a window's first and its
// last member.
std::vector<char> allowed_cuts(const int32_t* L, int32_t B) {
  std::vector<char> ok(static_cast<size_t>(B) + 1, 1);
  if (B > CORA_PACK_MAX_BATCH) return ok;
  int32_t first = -1, last = -1, tokens = 0;
  auto close = [&]() {
    for (int32_t c = first + 1; c <= last; ++c) ok[c] = 0;
    first = -1;
  };
  for (int32_t b = 0; b < B; ++b) {
    const int32_t l = L[b];
    if (l == 0) continue;
    if (l > CORA_TILE_ROWS) {
      if (first >= 0) close();
      continue;
    }
    if (first >= 0 && tokens + l <= CORA_TILE_ROWS) {
      tokens += l;
      last = b;
    } else {
      if (first >= 0) close();
      first = last = b;
      tokens = l;
    }
  }
  if (first >= 0) close();
  return ok;
}

// Greedy-left partition of [b0, b1) into parts of weight <= cap, cutting only where ok: returns the part
// count (a part that cannot be cut within cap takes the whole indivisible run).
int32_t greedy_parts(const std::vector<int64_t>& w, const std::vector<char>& ok, int32_t b0, int32_t b1, int64_t cap,
                     int32_t* cuts, int32_t max_cuts) {
  int32_t parts = 0, i = b0;
  while (i < b1) {
    int64_t run = 0;
    int32_t j = i, last = i;
    while (j < b1 && run + w[j] <= cap) {
      run += w[j++];
      if (ok[j]) last = j;
    }
    if (last == i) {  // the next indivisible run alone exceeds cap: take it whole
      j = i;
      do ++j;
      while (j < b1 && !ok[j]);
      last = j;
    }
    if (cuts != nullptr && parts < max_cuts) cuts[parts] = last;
    ++parts;
    i = last;
  }
  return parts;
}

}  // namespace

extern "C" {

cora_status_t cora_shard_plan(const int32_t* lengths_host, int32_t batch, int32_t d_model, int32_t d_ff,
                              int32_t n_ranks, int32_t* seq_begin_host, int32_t* row_begin_host) {
  if (n_ranks < 1 || batch < 0 || d_model <= 0 || d_ff <= 0 || seq_begin_host == nullptr ||
      (batch > 0 && lengths_host == nullptr))
    return CORA_ERR_INVALID;
  const int64_t per_tok = 2ll * (4ll * d_model * d_model + 2ll * d_model * d_ff);
  std::vector<int64_t> cost(batch);
  for (int32_t b = 0; b < batch; ++b) {
    const int64_t L = lengths_host[b];
    if (L < 0) return CORA_ERR_INVALID;
    cost[b] = L * per_tok + 4ll * d_model * L * L;
  }
  const std::vector<char> ok = allowed_cuts(lengths_host, batch);
  // smallest capacity C* for which the greedy partition over allowed cuts needs <= n_ranks parts (greedy
  // is optimal for a fixed capacity); bounds: the heaviest indivisible run .. the total
  int64_t total = 0, lo = 0, run = 0;
  for (int32_t b = 0; b < batch; ++b) {
    total += cost[b];
    run += cost[b];
    if (ok[b + 1]) {
      if (run > lo) lo = run;
      run = 0;
    }
  }
  int64_t hi = total > lo ? total : lo;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (greedy_parts(cost, ok, 0, batch, mid, nullptr, 0) <= n_ranks)
      hi = mid;
    else
      lo = mid + 1;
  }
  std::vector<int32_t> cuts(static_cast<size_t>(n_ranks) + 1, batch);
  const int32_t parts = batch > 0 ? greedy_parts(cost, ok, 0, batch, lo, cuts.data(), n_ranks) : 0;
  seq_begin_host[0] = 0;
  for (int32_t r = 0; r < n_ranks; ++r) seq_begin_host[r + 1] = r < parts ? cuts[r] : batch;
  seq_begin_host[n_ranks] = batch;
  if (row_begin_host != nullptr) {
    int64_t row = 0;
    int32_t b = 0;
    for (int32_t r = 0; r <= n_ranks; ++r) {
      while (b < seq_begin_host[r]) row += lengths_host[b++];
      if (row > INT32_MAX) return CORA_ERR_INVALID;
      row_begin_host[r] = static_cast<int32_t>(row);
    }
  }
  return CORA_OK;
}

cora_status_t cora_shard_groups(const int32_t* lengths_host, int32_t batch, const int32_t* seq_begin_host,
                                int32_t n_ranks, int32_t n_groups, int32_t* group_seq_host, int32_t* group_row_host) {
  if (batch < 0 || n_ranks < 1 || n_groups < 1 || seq_begin_host == nullptr || group_seq_host == nullptr ||
      (batch > 0 && lengths_host == nullptr))
    return CORA_ERR_INVALID;
  if (seq_begin_host[0] != 0 || seq_begin_host[n_ranks] != batch) return CORA_ERR_INVALID;
  for (int32_t r = 0; r < n_ranks; ++r)
    if (seq_begin_host[r] > seq_begin_host[r + 1]) return CORA_ERR_INVALID;
  std::vector<int64_t> tok(batch);
  for (int32_t b = 0; b < batch; ++b) {
    if (lengths_host[b] < 0) return CORA_ERR_INVALID;
    tok[b] = lengths_host[b];
  }
  const std::vector<char> ok = allowed_cuts(lengths_host, batch);
  std::vector<int64_t> row_off(static_cast<size_t>(batch) + 1, 0);
  for (int32_t b = 0; b < batch; ++b) row_off[b + 1] = row_off[b] + tok[b];
  const int32_t G = n_groups;
  for (int32_t r = 0; r < n_ranks; ++r) {
    const int32_t s0 = seq_begin_host[r], s1 = seq_begin_host[r + 1];
    int32_t* gs = group_seq_host + static_cast<size_t>(r) * (G + 1);
    // group g ends at the first allowed cut where the rank's token prefix reaches (g + 1) / G of its tokens
    const int64_t t0 = row_off[s0], tr = row_off[s1] - t0;
    gs[0] = s0;
    int32_t b = s0;
    for (int32_t g = 0; g < G - 1; ++g) {
      const int64_t target = (tr * (g + 1) + G - 1) / G;
      while (b < s1 && (row_off[b] - t0 < target || !ok[b])) ++b;
      gs[g + 1] = b;
    }
    gs[G] = s1;
    if (group_row_host != nullptr) {
      int32_t* gr = group_row_host + static_cast<size_t>(r) * (G + 1);
      for (int32_t g = 0; g <= G; ++g) {
        if (row_off[gs[g]] > INT32_MAX) return CORA_ERR_INVALID;
        gr[g] = static_cast<int32_t>(row_off[gs[g]]);
      }
    }
  }
  return CORA_OK;
}

}  // extern "C"
