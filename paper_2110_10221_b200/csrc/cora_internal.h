// Internal launcher declarations shared by the kernel translation units and api.cu.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "../../include/cora.h"

// Kernel spans (profiling builds only, -DCORA_KSPAN): per kernel slot, %globaltimer of the first CTA entry,
// the last CTA exit and the first / last return from griddepcontrol.wait, the sum (low 40 bits) and count of the CTA
// exits (mean exit: the kernel's tail), collected with 64-bit atomics.
// Slots: 0 prelude, 1 attention, 2 QKV, 3 out-proj + LN1, 4 FF1, 5 FF2 + LN2.  Each translation unit owns
// its array (no relocatable device code) and exports cora_debug_kspan_<tu>(host[8][6], reset).
#ifdef CORA_KSPAN
__device__ __forceinline__ unsigned long long kspan_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CORA_KSPAN_DEFINE(tu)                                                                            \
  __device__ unsigned long long g_kspan_##tu[8][6];                                                      \
  extern "C" int cora_debug_kspan_##tu(unsigned long long* host, int reset) {                           \
    if (reset) {                                                                                         \
      unsigned long long init[8][6];                                                                     \
      for (int i = 0; i < 8; ++i)                                                                        \
        init[i][0] = init[i][3] = ~0ull, init[i][1] = init[i][2] = init[i][4] = init[i][5] = 0ull;      \
      return cudaMemcpyToSymbol(g_kspan_##tu, init, sizeof(init)) == cudaSuccess ? 0 : 1;               \
    }                                                                                                    \
    return cudaMemcpyFromSymbol(host, g_kspan_##tu, sizeof(g_kspan_##tu)) == cudaSuccess ? 0 : 1;       \
  }
#define KSPAN_ENTRY(tu, slot) do { if (threadIdx.x == 0) atomicMin(&g_kspan_##tu[slot][0], kspan_now()); } while (0)
#define KSPAN_EXIT(tu, slot)                                                                             \
  do {                                                                                                   \
    if (threadIdx.x == 0) {                                                                              \
      const unsigned long long t_ = kspan_now();                                                         \
      atomicMax(&g_kspan_##tu[slot][1], t_);                                                             \
      atomicAdd(&g_kspan_##tu[slot][4], t_ & ((1ull << 40) - 1));                                                        \
      atomicAdd(&g_kspan_##tu[slot][5], 1ull);                                                           \
    }                                                                                                    \
  } while (0)
#define KSPAN_WAITED(tu, slot)                                                                           \
  do {                                                                                                   \
    if (threadIdx.x == 0) {                                                                              \
      const unsigned long long t_ = kspan_now();                                                         \
      atomicMax(&g_kspan_##tu[slot][2], t_);                                                             \
      atomicMin(&g_kspan_##tu[slot][3], t_);                                                             \
    }                                                                                                    \
  } while (0)
#else
#define CORA_KSPAN_DEFINE(tu)
#define KSPAN_ENTRY(tu, slot) ((void)0)
#define KSPAN_EXIT(tu, slot) ((void)0)
#define KSPAN_WAITED(tu, slot) ((void)0)
#endif

namespace cora {

constexpr int kAttnHeadDim = 64;  // head_dim of the tcgen05 attention kernel

// Short-sequence windows (reading f4-r1) are built by the prelude for batches of at most this many sequences.
#ifndef CORA_PACK_MAX_BATCH
#define CORA_PACK_MAX_BATCH 1024
#endif

// The prelude's inputs and outputs (the layout tables), for the prelude kernels and the QKV GEMM that runs the
// prelude in its epilogue warps (GemmArgs::prelude)
struct PreludeArgs {
  const int32_t* lengths;
  int32_t batch, total_tokens, heads, max_len;
  int32_t* row_off;
  int64_t* attn_off;
  int32_t *tiles, *tile_seq, *n_tiles, *units, *unit_seq, *n_units, *status, *seq_of_tok, *pos_in_seq;
  int32_t nparts;  // prelude parts (GEMM: run by CTAs c, c + gridDim, ...); 0 = no prelude
};
inline PreludeArgs prelude_args(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, const cora_layout_t& L) {
  return PreludeArgs{lengths, batch, total_tokens, heads, max_len, L.row_off, L.attn_off, L.tiles, L.tile_seq,
                     L.n_tiles, L.units, L.unit_seq, L.n_units, L.status, L.seq_of_tok, L.pos_in_seq, 0};
}
cudaError_t launch_layout_build(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, const cora_layout_t& L, cudaStream_t stream);

// GEMM: C[m,n] = act(A[m,k] B[n,k]^T + bias) + residual.  Tensor maps are built by the caller.
struct GemmArgs {
  const void* a;
  const void* b;
  const void* bias;
  const void* residual;
  void* c;
  int32_t m, n, k;
  int32_t act;
  const float* ln_gamma = nullptr;  // launch_gemm_ln: c = LN(act(a b^T + bias) + residual; gamma, beta, eps)
  const float* ln_beta = nullptr;
  float ln_eps = 0.f;
  bool late_wait = false;  // a / residual complete before the previous launch: wait for it only at the end
  // plain GEMM only: the epilogue warps run the prelude (parts c, c + gridDim, ... of prelude.nparts) before
  // their first unit -- the one-call forward's QKV GEMM (cora_encoder_forward, batch <= kPreludeInGemmMaxBatch)
  PreludeArgs prelude{};
};
constexpr int kPreludeInGemmMaxBatch = 256;
cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream);
bool gemm_ln_supported(const GemmArgs& g);
cudaError_t launch_gemm_ln(const GemmArgs& g, cudaStream_t stream);

// vgemm / trmm (vgemm.cu, SURVEY f-3)
size_t vgemm_plan_bytes(int32_t batch, const int32_t* dims_host);
void vgemm_plan(int32_t batch, const int32_t* dims_host, void* plan_host);
bool vgemm_plan_valid(const void* plan_host, size_t ws_bytes);
cudaError_t launch_vgemm(const void* plan_host, const void* a, const void* b, void* c, int32_t m_max, int32_t n_max,
                         int32_t k_max, void* ws, cudaStream_t stream);
cudaError_t launch_trmm(const void* l, const void* b, void* c, int32_t n, int32_t n_cols, cudaStream_t stream);

cudaError_t launch_attention(const cora_layout_t& L, const void* qkv, void* o, int32_t head_dim, float scale,
                             cudaStream_t stream, bool causal = false);

cudaError_t launch_layernorm(const void* x, const void* residual, const float* gamma, const float* beta, void* y,
                             int32_t rows, int32_t cols, float eps, cora_dtype_t dt, cudaStream_t stream);

cudaError_t launch_ragged_softmax(const cora_layout_t& L, const void* x, void* y, cora_dtype_t dt,
                                  cudaStream_t stream);

// Tensor-map creation through the driver entry point (no -lcuda link dependency).
bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                       uint32_t box_inner, uint32_t box_outer, bool swizzle128);

int device_sm_count();

// Function attributes (max dynamic smem) and occupancy answers are per device: one-time setup state is
// kept per device ordinal so one process may drive several GPUs.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

// Launch with programmatic dependent launch (PDL) enabled, and an optional cluster dimension.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int cluster,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace cora
