// the multi-GPU exchange of the sequence-sharded layer -- the final all-gather of
// the ragged outputs -- as C entry points over NCCL.
//
// Sequences are independent, so rank r runs the one-GPU layer on the contiguous sequence range
// [seq_begin[r], seq_begin[r+1]) chosen by cora_shard_plan and no collective runs inside the layer.  The
// gather is a variable-size all-gather whose data lands in place, in the original token order: one
// ncclBroadcast per rank (root r, rows [row_off[seq_begin[r]], row_off[seq_begin[r+1]]) of out) inside
// one ncclGroupStart / ncclGroupEnd, over NVLink / NVSwitch.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch already loaded when called from
// Python), so the library has no link-time NCCL dependency and the single-GPU path never loads it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>

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

cora_status_t cora_allgather_ragged(void* comm, const int32_t* row_off_host, const int32_t* seq_begin_host,
                                    void* out, int32_t d, cora_dtype_t dt, void* stream) {
  if (comm == nullptr || row_off_host == nullptr || seq_begin_host == nullptr || d <= 0) return CORA_ERR_INVALID;
  if (dt != CORA_DT_BF16 && dt != CORA_DT_F32) return CORA_ERR_INVALID;
  if (!nccl()) return CORA_ERR_NCCL;
  CoraComm* c = static_cast<CoraComm*>(comm);
  const size_t elt = dt == CORA_DT_BF16 ? 2 : 4;
  const ncclDataType_t nt = dt == CORA_DT_BF16 ? ncclBfloat16 : ncclFloat32;
  for (int r = 0; r < c->n_ranks; ++r)
    if (seq_begin_host[r] > seq_begin_host[r + 1]) return CORA_ERR_INVALID;
  const int64_t total_rows = row_off_host[seq_begin_host[c->n_ranks]];
  if (total_rows > 0 && out == nullptr) return CORA_ERR_INVALID;
  if (total_rows == 0) return CORA_OK;
  if (g_nccl.group_start() != ncclSuccess) return CORA_ERR_NCCL;
  ncclResult_t res = ncclSuccess;
  for (int r = 0; r < c->n_ranks && res == ncclSuccess; ++r) {
    const int64_t r0 = row_off_host[seq_begin_host[r]], r1 = row_off_host[seq_begin_host[r + 1]];
    if (r1 <= r0) continue;
    // in place: the root's rows are already in `out`; every other rank receives them at the same offset
    void* buf = static_cast<uint8_t*>(out) + static_cast<size_t>(r0) * d * elt;
    res = g_nccl.broadcast(buf, buf, static_cast<size_t>(r1 - r0) * d, nt, r, c->comm,
                           static_cast<cudaStream_t>(stream));
  }
  const ncclResult_t end = g_nccl.group_end();
  return (res == ncclSuccess && end == ncclSuccess) ? CORA_OK : CORA_ERR_NCCL;
}

}  // extern "C"
