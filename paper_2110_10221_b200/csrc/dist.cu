// the multi-GPU exchange of the sequence-sharded layer -- the final all-gather of
// the ragged outputs -- as C entry points over NCCL, and the sharded encoder stack whose gather overlaps
// the computation (cora_encoder_stack_sharded_fwd).
//
// Sequences are independent, so rank r runs the one-GPU layer on the contiguous sequence range
// [seq_begin[r], seq_begin[r+1]) chosen by cora_shard_plan and no collective runs inside the layer.  The
// gather is a variable-size all-gather whose data lands in place, in the original token order: one
// ncclBroadcast per rank (root r, rows [row_begin[r], row_begin[r+1]) of out) inside one ncclGroupStart /
// ncclGroupEnd, over NVLink / NVSwitch.  The sharded stack runs the paper's 6-layer model on ONE layout per
// group of the rank's sequences and gathers group g on a side stream while group g + 1
// computes, so the gather is amortised over the layers and overlapped with the compute.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch already loaded when called from
// Python), so the library has no link-time NCCL dependency and the single-GPU path never loads it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "cora_internal.h"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
  if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) return;
  g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.broadcast = reinterpret_cast<decltype(g_nccl.broadcast)>(dlsym(h, "ncclBroadcast"));
  g_nccl.group_start = reinterpret_cast<decltype(g_nccl.group_start)>(dlsym(h, "ncclGroupStart"));
  g_nccl.group_end = reinterpret_cast<decltype(g_nccl.group_end)>(dlsym(h, "ncclGroupEnd"));
  g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.comm_destroy && g_nccl.broadcast &&
              g_nccl.group_start && g_nccl.group_end;
}

bool nccl() {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.ok;
}

struct CoraComm {
  ncclComm_t comm;
  int n_ranks, rank;
};

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// One grouped set of in-place broadcasts: rank r's rows [ranges[r * stride], ranges[r * stride + 1]) from root r
// (stride 1: consecutive row_begin entries; stride 2: (begin, end) pairs).  Every rank issues the same set.
bool gather_rows(CoraComm* c, const int32_t* ranges, int stride, void* out, int32_t d, size_t elt, ncclDataType_t nt,
                 cudaStream_t stream) {
  if (g_nccl.group_start() != ncclSuccess) return false;
  ncclResult_t res = ncclSuccess;
  for (int r = 0; r < c->n_ranks && res == ncclSuccess; ++r) {
    const int64_t r0 = ranges[r * stride], r1 = ranges[r * stride + 1];
    if (r1 <= r0) continue;
    // in place: the root's rows are already in `out`; every other rank receives them at the same offset
    void* buf = static_cast<uint8_t*>(out) + static_cast<size_t>(r0) * d * elt;
    res = g_nccl.broadcast(buf, buf, static_cast<size_t>(r1 - r0) * d, nt, r, c->comm, stream);
  }
  const ncclResult_t end = g_nccl.group_end();
  return res == ncclSuccess && end == ncclSuccess;
}

// Side stream + events of the overlapped gather, created once per device.
constexpr int kMaxGroups = 16;
struct GatherPipe {
  cudaStream_t comm = nullptr;
  cudaEvent_t start = nullptr, done = nullptr, comp_ev[kMaxGroups] = {};
  bool ok = false;
};
GatherPipe g_gpipe[cora::kMaxDevices];
std::mutex g_gpipe_mu;

GatherPipe* gather_pipe() {
  const int dev = cora::current_device();
  std::lock_guard<std::mutex> lk(g_gpipe_mu);
  GatherPipe& gp = g_gpipe[dev];
  if (!gp.ok) {
    bool good = cudaStreamCreateWithFlags(&gp.comm, cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&gp.start, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&gp.done, cudaEventDisableTiming) == cudaSuccess;
    for (int g = 0; good && g < kMaxGroups; ++g)
      good = cudaEventCreateWithFlags(&gp.comp_ev[g], cudaEventDisableTiming) == cudaSuccess;
    if (!good) return nullptr;
    gp.ok = true;
  }
  return &gp;
}

}  // namespace

extern "C" {

int32_t cora_comm_unique_id_bytes(void) { return static_cast<int32_t>(sizeof(ncclUniqueId)); }

cora_status_t cora_comm_get_unique_id(void* id_out) {
  if (id_out == nullptr) return CORA_ERR_INVALID;
  if (!nccl()) return CORA_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.get_unique_id(&id) != ncclSuccess) return CORA_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return CORA_OK;
}

cora_status_t cora_comm_init(void** comm, const void* nccl_unique_id, int32_t n_ranks, int32_t rank) {
  if (comm == nullptr || nccl_unique_id == nullptr || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return CORA_ERR_INVALID;
  if (!nccl()) return CORA_ERR_NCCL;
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  CoraComm* c = new CoraComm{nullptr, n_ranks, rank};
  if (g_nccl.comm_init_rank(&c->comm, n_ranks, id, rank) != ncclSuccess) {
    delete c;
    return CORA_ERR_NCCL;
  }
  *comm = c;
  return CORA_OK;
}

cora_status_t cora_comm_destroy(void* comm) {
  if (comm == nullptr) return CORA_ERR_INVALID;
  CoraComm* c = static_cast<CoraComm*>(comm);
  const ncclResult_t r = nccl() ? g_nccl.comm_destroy(c->comm) : ncclSuccess;
  delete c;
  return r == ncclSuccess ? CORA_OK : CORA_ERR_NCCL;
}

cora_status_t cora_allgather_ragged(void* comm, const int32_t* row_begin_host, void* out, int32_t d, cora_dtype_t dt,
                                    void* stream) {
  if (comm == nullptr || row_begin_host == nullptr || d <= 0) return CORA_ERR_INVALID;
  if (dt != CORA_DT_BF16 && dt != CORA_DT_F32) return CORA_ERR_INVALID;
  CoraComm* c = static_cast<CoraComm*>(comm);
  for (int r = 0; r < c->n_ranks; ++r)
    if (row_begin_host[r] < 0 || row_begin_host[r] > row_begin_host[r + 1]) return CORA_ERR_INVALID;
  const int64_t total_rows = row_begin_host[c->n_ranks];
  if (total_rows > 0 && out == nullptr) return CORA_ERR_INVALID;
  if (total_rows == 0 || c->n_ranks == 1) return CORA_OK;
  if (!nccl()) return CORA_ERR_NCCL;
  return gather_rows(c, row_begin_host, 1, out, d, dt == CORA_DT_BF16 ? 2 : 4,
                     dt == CORA_DT_BF16 ? ncclBfloat16 : ncclFloat32, static_cast<cudaStream_t>(stream))
             ? CORA_OK
             : CORA_ERR_NCCL;
}

size_t cora_encoder_stack_sharded_workspace_bytes(const cora_encoder_params_t* layers, int32_t n_layers, int32_t batch,
                                                  int32_t total_tokens, int32_t max_len) {
  if (layers == nullptr || n_layers < 1) return 0;
  const size_t lay = cora_layout_workspace_bytes(batch, total_tokens, layers[0].heads, max_len);
  const size_t stack = cora_encoder_stack_workspace_bytes(layers, n_layers, total_tokens);
  if (lay == 0 || stack == 0) return 0;
  return align256(lay) + stack;
}

cora_status_t cora_encoder_stack_sharded_fwd(const cora_encoder_params_t* layers, int32_t n_layers,
                                             const int32_t* lengths, const int32_t* lengths_host, int32_t batch,
                                             int32_t total_tokens, int32_t max_len, void* comm, int32_t n_groups,
                                             const void* x, void* y, void* ws, size_t ws_bytes, void* stream) {
  if (layers == nullptr || n_layers < 1 || batch < 0 || total_tokens < 0 || n_groups < 1 || n_groups > kMaxGroups)
    return CORA_ERR_INVALID;
  if ((batch > 0 && (lengths == nullptr || lengths_host == nullptr)) || ws == nullptr) return CORA_ERR_INVALID;
  if (total_tokens > 0 && (x == nullptr || y == nullptr || x == y)) return CORA_ERR_INVALID;
  const size_t need = cora_encoder_stack_sharded_workspace_bytes(layers, n_layers, batch, total_tokens, max_len);
  if (need == 0 || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % 256) != 0) return CORA_ERR_INVALID;
  int64_t sum = 0;
  for (int32_t b = 0; b < batch; ++b) sum += lengths_host[b];
  if (sum != total_tokens) return CORA_ERR_INVALID;
  CoraComm* c = static_cast<CoraComm*>(comm);
  const int n_ranks = c != nullptr ? c->n_ranks : 1, rank = c != nullptr ? c->rank : 0;
  // the plan and the groups: computed identically on every rank from the host lengths
  std::vector<int32_t> seq_begin(n_ranks + 1), gseq(static_cast<size_t>(n_ranks) * (n_groups + 1)),
      grow(static_cast<size_t>(n_ranks) * (n_groups + 1));
  cora_status_t st = cora_shard_plan(lengths_host, batch, layers[0].d_model, layers[0].d_ff, n_ranks, seq_begin.data(),
                                     nullptr);
  if (st != CORA_OK) return st;
  st = cora_shard_groups(lengths_host, batch, seq_begin.data(), n_ranks, n_groups, gseq.data(), grow.data());
  if (st != CORA_OK) return st;
  const bool gather = n_ranks > 1;
  if (gather && !nccl()) return CORA_ERR_NCCL;
  GatherPipe* gp = gather ? gather_pipe() : nullptr;
  if (gather && gp == nullptr) return CORA_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t d = layers[0].d_model;
  const size_t row = 2ull * d;
  uint8_t* w = static_cast<uint8_t*>(ws);
  const size_t lay_bytes = cora_layout_workspace_bytes(batch, total_tokens, layers[0].heads, max_len);
  uint8_t* stack_ws = w + align256(lay_bytes);
  const size_t stack_bytes = ws_bytes - align256(lay_bytes);
  if (gather && (cudaEventRecord(gp->start, s) != cudaSuccess || cudaStreamWaitEvent(gp->comm, gp->start, 0) != cudaSuccess))
    return CORA_ERR_CUDA;
  const int32_t* my_seq = gseq.data() + static_cast<size_t>(rank) * (n_groups + 1);
  const int32_t* my_row = grow.data() + static_cast<size_t>(rank) * (n_groups + 1);
  std::vector<int32_t> rows_g(n_ranks + 1);
  for (int g = 0; g < n_groups; ++g) {
    const int32_t nb = my_seq[g + 1] - my_seq[g], nt = my_row[g + 1] - my_row[g];
    if (nt > 0) {
      cora_layout_t L;
      st = cora_layout_build(lengths + my_seq[g], nb, nt, layers[0].heads, max_len, w, lay_bytes, &L, stream);
      if (st != CORA_OK) return st;
      st = cora_encoder_stack_fwd(layers, n_layers, &L, static_cast<const uint8_t*>(x) + row * my_row[g],
                                  static_cast<uint8_t*>(y) + row * my_row[g], stack_ws, stack_bytes, stream);
      if (st != CORA_OK) return st;
    }
    if (!gather) continue;
    // group g of every rank leaves for every other rank on the side stream while group g + 1 computes
    if (cudaEventRecord(gp->comp_ev[g], s) != cudaSuccess || cudaStreamWaitEvent(gp->comm, gp->comp_ev[g], 0) != cudaSuccess)
      return CORA_ERR_CUDA;
    // rank r's group-g rows [grow[r][g], grow[r][g+1]) as a (begin, count) pair list for gather_rows
    std::vector<int32_t> pairs(2 * n_ranks);
    for (int r = 0; r < n_ranks; ++r) {
      const int32_t* gr = grow.data() + static_cast<size_t>(r) * (n_groups + 1);
      pairs[2 * r] = gr[g];
      pairs[2 * r + 1] = gr[g + 1];
    }
    if (!gather_rows(c, pairs.data(), 2, y, d, 2, ncclBfloat16, gp->comm)) return CORA_ERR_NCCL;
  }
  if (gather && (cudaEventRecord(gp->done, gp->comm) != cudaSuccess || cudaStreamWaitEvent(s, gp->done, 0) != cudaSuccess))
    return CORA_ERR_CUDA;
  return CORA_OK;
}

}  // extern "C"
