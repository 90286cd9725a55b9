// C ABI of libcora_b200.so (include/cora.h): argument validation, workspace carving, tensor-map
// creation and the orchestration of the encoder layer.  All arithmetic of the method runs in the
// kernels of prelude.cu, gemm.cu, attention.cu and elementwise.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "cora_internal.h"

namespace cora {

// ---------------------------------------------------------------- driver entry point for TMA maps
namespace {
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_t g_encode = nullptr;
std::once_flag g_encode_once;

void load_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_encodeTiled_t>(fn);
}

int g_sm_count[64] = {0};
}  // namespace

bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                       uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  std::call_once(g_encode_once, load_encode);
  if (g_encode == nullptr) return false;
  if (inner == 0 || outer == 0) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (g_sm_count[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sm_count[dev] = n > 0 ? n : 148;
  }
  return g_sm_count[dev];
}

}  // namespace cora

using namespace cora;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
inline cora_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return CORA_OK;
  if (e == cudaErrorInvalidValue) return CORA_ERR_UNSUPPORTED;
  return CORA_ERR_CUDA;
}

int64_t tiles_bound(int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len) {
  // sum_b ceil(L_b/128) <= min((T + 127 B) / 128, B * ceil(max_len / 128))
  const int64_t a = (static_cast<int64_t>(total_tokens) + 127ll * batch) / CORA_TILE_ROWS;
  const int64_t b = static_cast<int64_t>(batch) * ((max_len + CORA_TILE_ROWS - 1) / CORA_TILE_ROWS);
  return heads * (a < b ? a : b);
}

int64_t units_bound(int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len) {
  // sum_b ceil(nq_b / 2) <= (sum_b nq_b + B) / 2
  return heads * ((tiles_bound(batch, total_tokens, 1, max_len) + batch) / 2);
}

struct LayoutCarve {
  size_t row_off, attn_off, seq_of_tok, pos_in_seq, tiles, tile_seq, n_tiles, status, units, unit_seq, n_units,
      total;
};
LayoutCarve carve_layout(int32_t batch, int32_t total_tokens, int64_t n_tiles_max, int64_t n_units_max) {
  LayoutCarve c;
  size_t o = 0;
  c.attn_off = o;
  o = align_up(o + sizeof(int64_t) * (batch + 1));
  c.row_off = o;
  o = align_up(o + sizeof(int32_t) * (batch + 1));
  c.seq_of_tok = o;
  o = align_up(o + sizeof(int32_t) * static_cast<size_t>(total_tokens));
  c.pos_in_seq = o;
  o = align_up(o + sizeof(int32_t) * static_cast<size_t>(total_tokens));
  c.tiles = o;
  o = align_up(o + sizeof(int32_t) * static_cast<size_t>(n_tiles_max));
  c.tile_seq = o;
  o = align_up(o + 2 * sizeof(int32_t) * static_cast<size_t>(n_tiles_max));
  c.n_tiles = o;
  o = align_up(o + sizeof(int32_t));
  c.status = o;
  o = align_up(o + sizeof(int32_t));
  c.units = o;
  o = align_up(o + sizeof(int32_t) * static_cast<size_t>(n_units_max));
  c.unit_seq = o;
  o = align_up(o + 2 * sizeof(int32_t) * static_cast<size_t>(n_units_max));
  c.n_units = o;
  o = align_up(o + sizeof(int32_t));
  c.total = o;
  return c;
}

bool layout_args_ok(int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len) {
  return batch >= 0 && batch <= 65536 && total_tokens >= 0 && heads >= 1 && heads <= 255 && max_len >= 0 &&
         max_len <= 16383;
}

struct EncoderCarve {
  size_t qkv, o, y1, h1, f, y2, total;
};
EncoderCarve carve_encoder(const cora_encoder_params_t* p, int32_t T) {
  EncoderCarve c;
  const size_t t = static_cast<size_t>(T), d = p->d_model, ff = p->d_ff;
  size_t o = 0;
  c.qkv = o;
  o = align_up(o + 2 * t * 3 * d);
  c.o = o;
  o = align_up(o + 2 * t * d);
  c.y1 = o;
  o = align_up(o + 2 * t * d);
  c.h1 = o;
  o = align_up(o + 2 * t * d);
  c.f = o;
  o = align_up(o + 2 * t * ff);
  c.y2 = o;
  o = align_up(o + 2 * t * d);
  c.total = o;
  return c;
}

}  // namespace

extern "C" {

size_t cora_layout_workspace_bytes(int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len) {
  if (!layout_args_ok(batch, total_tokens, heads, max_len)) return 0;
  return carve_layout(batch, total_tokens, tiles_bound(batch, total_tokens, heads, max_len),
                      units_bound(batch, total_tokens, heads, max_len))
      .total;
}

}  // extern "C"
namespace {
// cora_layout_build without (launch = false) or with the prelude launch: the layout's tables carved from ws
cora_status_t layout_build_impl(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, void* ws, size_t ws_bytes, cora_layout_t* out, void* stream,
                                bool launch) {
  if (out == nullptr || !layout_args_ok(batch, total_tokens, heads, max_len)) return CORA_ERR_INVALID;
  if (batch > 0 && lengths == nullptr) return CORA_ERR_INVALID;
  const int64_t ntm = tiles_bound(batch, total_tokens, heads, max_len);
  const int64_t num = units_bound(batch, total_tokens, heads, max_len);
  if (ntm > INT32_MAX) return CORA_ERR_INVALID;
  const LayoutCarve c = carve_layout(batch, total_tokens, ntm, num);
  if (ws == nullptr || ws_bytes < c.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0)
    return CORA_ERR_INVALID;
  uint8_t* w = static_cast<uint8_t*>(ws);
  cora_layout_t L;
  std::memset(&L, 0, sizeof(L));
  L.batch = batch;
  L.heads = heads;
  L.max_len = max_len;
  L.total_tokens = total_tokens;
  L.n_tiles_max = static_cast<int32_t>(ntm);
  L.total_attn = -1;  // known on the host after cora_layout_status
  L.lengths = lengths;
  L.row_off = reinterpret_cast<int32_t*>(w + c.row_off);
  L.attn_off = reinterpret_cast<int64_t*>(w + c.attn_off);
  L.seq_of_tok = reinterpret_cast<int32_t*>(w + c.seq_of_tok);
  L.pos_in_seq = reinterpret_cast<int32_t*>(w + c.pos_in_seq);
  L.tiles = reinterpret_cast<int32_t*>(w + c.tiles);
  L.tile_seq = reinterpret_cast<int32_t*>(w + c.tile_seq);
  L.n_tiles = reinterpret_cast<int32_t*>(w + c.n_tiles);
  L.status = reinterpret_cast<int32_t*>(w + c.status);
  L.n_units_max = static_cast<int32_t>(num);
  L.units = reinterpret_cast<int32_t*>(w + c.units);
  L.unit_seq = reinterpret_cast<int32_t*>(w + c.unit_seq);
  L.n_units = reinterpret_cast<int32_t*>(w + c.n_units);
  const cudaError_t e =
      launch ? launch_layout_build(lengths, batch, total_tokens, heads, max_len, L, as_stream(stream)) : cudaSuccess;
  *out = L;
  return e == cudaSuccess ? CORA_OK : CORA_ERR_CUDA;
}
}  // namespace
extern "C" {

cora_status_t cora_layout_build(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, void* ws, size_t ws_bytes, cora_layout_t* out, void* stream) {
  return layout_build_impl(lengths, batch, total_tokens, heads, max_len, ws, ws_bytes, out, stream, true);
}

cora_status_t cora_layout_status(cora_layout_t* layout, void* stream) {
  if (layout == nullptr || layout->status == nullptr || layout->attn_off == nullptr) return CORA_ERR_INVALID;
  int32_t st = 0;
  int64_t s2 = 0;
  cudaError_t e = cudaMemcpyAsync(&st, layout->status, sizeof(st), cudaMemcpyDeviceToHost, as_stream(stream));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&s2, layout->attn_off + layout->batch, sizeof(s2), cudaMemcpyDeviceToHost, as_stream(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(as_stream(stream));
  if (e != cudaSuccess) return CORA_ERR_CUDA;
  layout->total_attn = st == 0 ? s2 : -1;
  return st == 0 ? CORA_OK : CORA_ERR_DATA;
}

size_t cora_encoder_workspace_bytes(const cora_encoder_params_t* p, int32_t total_tokens) {
  if (p == nullptr || total_tokens < 0) return 0;
  return carve_encoder(p, total_tokens).total;
}

cora_status_t cora_linear_fwd(const void* a, const void* w, const void* bias, const void* residual, void* c,
                              int32_t m, int32_t n, int32_t k, cora_act_t act, void* stream) {
  if (m < 0 || n <= 0 || k <= 0 || (n % 8) != 0 || (k % 8) != 0) return CORA_ERR_INVALID;
  if (act < CORA_ACT_NONE || act > CORA_ACT_GELU_ERF) return CORA_ERR_INVALID;
  if (m == 0) return CORA_OK;
  if (a == nullptr || w == nullptr || c == nullptr || !aligned16(a) || !aligned16(w) || !aligned16(c))
    return CORA_ERR_INVALID;
  if ((bias != nullptr && !aligned16(bias)) || (residual != nullptr && !aligned16(residual))) return CORA_ERR_INVALID;
  GemmArgs g{a, w, bias, residual, c, m, n, k, act};
  return cuda_status(launch_gemm(g, as_stream(stream)));
}

cora_status_t cora_linear_residual_layernorm_fwd(const void* a, const void* w, const void* bias, const void* residual,
                                                 const float* gamma, const float* beta, float eps, void* c, int32_t m,
                                                 int32_t n, int32_t k, cora_act_t act, void* stream) {
  if (m < 0 || n <= 0 || k <= 0 || (k % 8) != 0 || act < CORA_ACT_NONE || act > CORA_ACT_GELU_ERF)
    return CORA_ERR_INVALID;
  if (m == 0) return CORA_OK;
  if (a == nullptr || w == nullptr || c == nullptr || residual == nullptr || gamma == nullptr || beta == nullptr ||
      !aligned16(a) || !aligned16(w) || !aligned16(c) || !aligned16(residual) || (bias != nullptr && !aligned16(bias)))
    return CORA_ERR_INVALID;
  GemmArgs g{a, w, bias, residual, c, m, n, k, act};
  g.ln_gamma = gamma;
  g.ln_beta = beta;
  g.ln_eps = eps;
  if (gemm_ln_supported(g)) return cuda_status(launch_gemm_ln(g, as_stream(stream)));
  if ((n % 8) != 0) return CORA_ERR_UNSUPPORTED;
  // not fusable (an activation, or N != 512): act(a w^T + bias) + residual is written to c itself, then
  // LayerNorm'd in place (each row is read completely before it is written) -- no temporary is allocated
  cudaStream_t s = as_stream(stream);
  cudaError_t e = launch_gemm(g, s);
  if (e == cudaSuccess) e = launch_layernorm(c, nullptr, gamma, beta, c, m, n, eps, CORA_DT_BF16, s);
  return cuda_status(e);
}

size_t cora_vgemm_plan_bytes(int32_t batch, const int32_t* dims_host) {
  if (batch < 0 || (batch > 0 && dims_host == nullptr)) return 0;
  for (int i = 0; i < batch; ++i)
    if (dims_host[3 * i] < 0 || dims_host[3 * i + 1] < 0 || dims_host[3 * i + 2] < 0) return 0;
  return vgemm_plan_bytes(batch, dims_host);
}

size_t cora_vgemm_workspace_bytes(int32_t batch, const int32_t* dims_host) {
  return cora_vgemm_plan_bytes(batch, dims_host);
}

cora_status_t cora_vgemm_plan(int32_t batch, const int32_t* dims_host, int32_t m_max, int32_t n_max, int32_t k_max,
                              void* plan_host, size_t plan_bytes) {
  if (batch < 0 || m_max < 0 || n_max < 0 || k_max < 0 || plan_host == nullptr) return CORA_ERR_INVALID;
  if (batch > 0 && dims_host == nullptr) return CORA_ERR_INVALID;
  if ((n_max % 8) != 0 || (k_max % 8) != 0) return CORA_ERR_INVALID;
  for (int i = 0; i < batch; ++i) {
    const int32_t m = dims_host[3 * i], n = dims_host[3 * i + 1], k = dims_host[3 * i + 2];
    if (m < 0 || n < 0 || k < 0 || m > m_max || n > n_max || k > k_max) return CORA_ERR_INVALID;
    // a partial last k-block would read the padding of A and B unless it is the tensor's own tail
    if ((k % 64) != 0 && k != k_max) return CORA_ERR_UNSUPPORTED;
  }
  if (plan_bytes < vgemm_plan_bytes(batch, dims_host)) return CORA_ERR_INVALID;
  vgemm_plan(batch, dims_host, plan_host);
  return CORA_OK;
}

cora_status_t cora_vgemm_fwd(const void* plan_host, const void* a, const void* b, void* c, int32_t m_max, int32_t n_max,
                             int32_t k_max, void* ws, size_t ws_bytes, void* stream) {
  if (plan_host == nullptr || m_max < 0 || n_max < 0 || k_max < 0) return CORA_ERR_INVALID;
  const int32_t* h = static_cast<const int32_t*>(plan_host);
  if (h[1] == 0 || h[2] == 0 || m_max == 0 || n_max == 0) return CORA_OK;  // nothing to compute
  if (a == nullptr || b == nullptr || c == nullptr || ws == nullptr) return CORA_ERR_INVALID;
  if (!aligned16(a) || !aligned16(b) || !aligned16(c) || !aligned16(ws) || (n_max % 8) != 0 || (k_max % 8) != 0 ||
      k_max == 0)
    return CORA_ERR_INVALID;
  if (!vgemm_plan_valid(plan_host, ws_bytes)) return CORA_ERR_INVALID;
  return cuda_status(launch_vgemm(plan_host, a, b, c, m_max, n_max, k_max, ws, as_stream(stream)));
}

cora_status_t cora_trmm_fwd(const void* l, const void* b, void* c, int32_t n, int32_t n_cols, void* stream) {
  if (n < 0 || n_cols < 0) return CORA_ERR_INVALID;
  if (n == 0 || n_cols == 0) return CORA_OK;
  if (l == nullptr || b == nullptr || c == nullptr || !aligned16(l) || !aligned16(b) || !aligned16(c) ||
      (n % 8) != 0 || (n_cols % 8) != 0)
    return CORA_ERR_INVALID;
  return cuda_status(launch_trmm(l, b, c, n, n_cols, as_stream(stream)));
}

cora_status_t cora_ragged_attention_fwd(const cora_layout_t* layout, const void* qkv, void* o, int32_t head_dim,
                                        float scale, void* stream) {
  if (layout == nullptr || head_dim <= 0 || head_dim > 128 || (head_dim % 2) != 0) return CORA_ERR_INVALID;
  if (layout->total_tokens == 0 || layout->batch == 0) return CORA_OK;
  if (qkv == nullptr || o == nullptr || !aligned16(qkv) || !aligned16(o)) return CORA_ERR_INVALID;
  if (((layout->heads * head_dim) % 8) != 0) return CORA_ERR_INVALID;
  return cuda_status(launch_attention(*layout, qkv, o, head_dim, scale, as_stream(stream)));
}

cora_status_t cora_ragged_masked_attention_fwd(const cora_layout_t* layout, const void* qkv, void* o,
                                               int32_t head_dim, float scale, void* stream) {
  if (layout == nullptr || head_dim <= 0 || head_dim > 128 || (head_dim % 2) != 0) return CORA_ERR_INVALID;
  if (layout->total_tokens == 0 || layout->batch == 0) return CORA_OK;
  if (qkv == nullptr || o == nullptr || !aligned16(qkv) || !aligned16(o)) return CORA_ERR_INVALID;
  if (((layout->heads * head_dim) % 8) != 0) return CORA_ERR_INVALID;
  return cuda_status(launch_attention(*layout, qkv, o, head_dim, scale, as_stream(stream), /*causal=*/true));
}

cora_status_t cora_ragged_softmax_fwd(const cora_layout_t* layout, const void* x, void* y, cora_dtype_t dt,
                                      void* stream) {
  if (layout == nullptr || (dt != CORA_DT_BF16 && dt != CORA_DT_F32)) return CORA_ERR_INVALID;
  if (layout->total_tokens == 0 || layout->batch == 0) return CORA_OK;
  if (x == nullptr || y == nullptr) return CORA_ERR_INVALID;
  return cuda_status(launch_ragged_softmax(*layout, x, y, dt, as_stream(stream)));
}

cora_status_t cora_layernorm_fwd(const void* x, const void* residual, const float* gamma, const float* beta, void* y,
                                 int32_t rows, int32_t cols, float eps, cora_dtype_t dt, void* stream) {
  if (rows < 0 || cols <= 0 || (cols % 8) != 0 || (dt != CORA_DT_BF16 && dt != CORA_DT_F32)) return CORA_ERR_INVALID;
  if (rows == 0) return CORA_OK;
  if (x == nullptr || y == nullptr || gamma == nullptr || beta == nullptr || !aligned16(x) || !aligned16(y) ||
      (residual != nullptr && !aligned16(residual)))
    return CORA_ERR_INVALID;
  return cuda_status(launch_layernorm(x, residual, gamma, beta, y, rows, cols, eps, dt, as_stream(stream)));
}

namespace {
// qkv_late_wait: x was complete before the previous launch on the stream (the prelude of
// cora_encoder_forward), so the QKV GEMM need not wait for that launch before reading x -- it runs under
// the prelude and waits for it only before completing
cora_status_t encoder_layer_impl(const cora_encoder_params_t* p, const cora_layout_t* layout, const void* x, void* y,
                                 void* ws, size_t ws_bytes, void* stream, void* const* events, bool qkv_late_wait,
                                 const PreludeArgs* prelude = nullptr) {
  if (p == nullptr || layout == nullptr) return CORA_ERR_INVALID;
  const int32_t d = p->d_model, H = p->heads, ff = p->d_ff, T = layout->total_tokens;
  if (d <= 0 || H <= 0 || ff <= 0 || (d % H) != 0 || (d % 8) != 0 || (ff % 8) != 0 || H != layout->heads)
    return CORA_ERR_INVALID;
  const int32_t hd = d / H;
  if (hd > 128 || (hd % 2) != 0) return CORA_ERR_UNSUPPORTED;
  if (p->act < CORA_ACT_NONE || p->act > CORA_ACT_GELU_ERF) return CORA_ERR_INVALID;
  if (T == 0 || layout->batch == 0) return CORA_OK;
  const void* ptrs[] = {p->w_qkv, p->b_qkv, p->w_o, p->b_o, p->ln1_g, p->ln1_b, p->w1, p->b1, p->w2, p->b2,
                        p->ln2_g, p->ln2_b, x, y, ws};
  for (const void* q : ptrs)
    if (q == nullptr || !aligned16(q)) return CORA_ERR_INVALID;
  if (x == y) return CORA_ERR_INVALID;
  const EncoderCarve c = carve_encoder(p, T);
  if (ws_bytes < c.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return CORA_ERR_INVALID;
  uint8_t* w = static_cast<uint8_t*>(ws);
  void* qkv = w + c.qkv;
  void* o = w + c.o;
  void* y1 = w + c.y1;
  void* h1 = w + c.h1;
  void* f = w + c.f;
  void* y2 = w + c.y2;
  cudaStream_t s = as_stream(stream);
  auto mark = [&](int k) {
    if (events == nullptr) return;
    // inside stream capture an external record becomes an event-record node of the graph
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive)
      cudaEventRecordWithFlags(static_cast<cudaEvent_t>(events[k]), s, cudaEventRecordExternal);
    else
      cudaEventRecord(static_cast<cudaEvent_t>(events[k]), s);
  };
  cudaError_t e;
  // a2: QKV = x W_qkv^T + b_qkv
  mark(0);
  GemmArgs g2{x, p->w_qkv, p->b_qkv, nullptr, qkv, T, 3 * d, d, CORA_ACT_NONE};
  g2.late_wait = qkv_late_wait && events == nullptr;
  if (prelude != nullptr) {  // the QKV GEMM's epilogue warps build the layout (no prelude kernel to wait for)
    g2.prelude = *prelude;
    g2.late_wait = false;
  }
  if ((e = launch_gemm(g2, s)) != cudaSuccess) return cuda_status(e);
  // a3: fused ragged attention
  mark(1);
  if ((e = launch_attention(*layout, qkv, o, hd, 1.0f / sqrtf(static_cast<float>(hd)), s)) != cudaSuccess)
    return cuda_status(e);
  // a4 + a5: H1 = LN1(O W_o^T + b_o + x)   (fused when d_model == 512; Y1 never reaches HBM)
  mark(2);
  GemmArgs g4{o, p->w_o, p->b_o, x, y1, T, d, d, CORA_ACT_NONE};
  g4.ln_gamma = static_cast<const float*>(p->ln1_g);
  g4.ln_beta = static_cast<const float*>(p->ln1_b);
  g4.ln_eps = p->ln_eps;
  const bool fuse = gemm_ln_supported(g4);
  if (fuse) {
    g4.c = h1;
    if ((e = launch_gemm_ln(g4, s)) != cudaSuccess) return cuda_status(e);
    mark(3);
  } else {
    if ((e = launch_gemm(GemmArgs{o, p->w_o, p->b_o, x, y1, T, d, d, CORA_ACT_NONE}, s)) != cudaSuccess)
      return cuda_status(e);
    mark(3);
    if ((e = launch_layernorm(y1, nullptr, static_cast<const float*>(p->ln1_g), static_cast<const float*>(p->ln1_b),
                              h1, T, d, p->ln_eps, CORA_DT_BF16, s)) != cudaSuccess)
      return cuda_status(e);
  }
  // a6: F = act(H1 W1^T + b1)
  mark(4);
  if ((e = launch_gemm(GemmArgs{h1, p->w1, p->b1, nullptr, f, T, ff, d, p->act}, s)) != cudaSuccess)
    return cuda_status(e);
  // a7 + a8: y = LN2(F W2^T + b2 + H1)   (fused when d_model == 512; Y2 never reaches HBM)
  mark(5);
  if (fuse) {
    GemmArgs g7{f, p->w2, p->b2, h1, y, T, d, ff, CORA_ACT_NONE};
    g7.ln_gamma = static_cast<const float*>(p->ln2_g);
    g7.ln_beta = static_cast<const float*>(p->ln2_b);
    g7.ln_eps = p->ln_eps;
    if ((e = launch_gemm_ln(g7, s)) != cudaSuccess) return cuda_status(e);
    mark(6);
  } else {
    if ((e = launch_gemm(GemmArgs{f, p->w2, p->b2, h1, y2, T, d, ff, CORA_ACT_NONE}, s)) != cudaSuccess)
      return cuda_status(e);
    mark(6);
    if ((e = launch_layernorm(y2, nullptr, static_cast<const float*>(p->ln2_g), static_cast<const float*>(p->ln2_b), y,
                              T, d, p->ln_eps, CORA_DT_BF16, s)) != cudaSuccess)
      return cuda_status(e);
  }
  mark(7);
  return CORA_OK;
}
}  // namespace

cora_status_t cora_encoder_layer_fwd_ex(const cora_encoder_params_t* p, const cora_layout_t* layout, const void* x,
                                        void* y, void* ws, size_t ws_bytes, void* stream, void* const* events) {
  return encoder_layer_impl(p, layout, x, y, ws, ws_bytes, stream, events, false);
}

}  // extern "C"
namespace {
// Prelude + layer on one layout.  Batches of at most kPreludeInGemmMaxBatch sequences: the QKV GEMM's epilogue
// warps build the layout while its first units run (no prelude kernel; CORA_QKV_PRELUDE=0 disables), else the
// prelude kernel runs beside a late-waiting QKV GEMM.
cora_status_t forward_impl(const cora_encoder_params_t* p, const int32_t* lengths, int32_t batch, int32_t T,
                           int32_t max_len, void* lay_ws, size_t lay_bytes, const void* x, void* y, void* ws,
                           size_t ws_bytes, cora_layout_t* L, cora_layout_t* layout_out, void* stream) {
  const char* pv = getenv("CORA_QKV_PRELUDE");
  const bool in_gemm = (pv == nullptr || atoi(pv) != 0) && batch >= 1 && batch <= kPreludeInGemmMaxBatch && T > 0;
  cora_status_t st = layout_build_impl(lengths, batch, T, p->heads, max_len, lay_ws, lay_bytes, L, stream, !in_gemm);
  if (st != CORA_OK) return st;
  if (layout_out != nullptr) *layout_out = *L;
  if (!in_gemm) return encoder_layer_impl(p, L, x, y, ws, ws_bytes, stream, nullptr, true);
  PreludeArgs pre = prelude_args(lengths, batch, T, p->heads, max_len, *L);
  const char* spv = getenv("CORA_PRELUDE_SPB");  // experiments: sequences per part
  const int spb = spv != nullptr && atoi(spv) > 0 ? atoi(spv) : 8;
  pre.nparts = (batch + spb - 1) / spb;  // 8 sequences per part (4 / 16: +1 / -0.2 us at C4)
  return encoder_layer_impl(p, L, x, y, ws, ws_bytes, stream, nullptr, false, &pre);
}
}  // namespace
extern "C" {

size_t cora_encoder_forward_workspace_bytes(const cora_encoder_params_t* p, int32_t batch, int32_t total_tokens,
                                            int32_t max_len) {
  if (p == nullptr || !layout_args_ok(batch, total_tokens, p->heads, max_len)) return 0;
  return align_up(cora_layout_workspace_bytes(batch, total_tokens, p->heads, max_len)) +
         carve_encoder(p, total_tokens).total;
}

cora_status_t cora_encoder_forward(const cora_encoder_params_t* p, const int32_t* lengths, int32_t batch,
                                   int32_t total_tokens, int32_t max_len, const void* x, void* y, void* ws,
                                   size_t ws_bytes, cora_layout_t* layout_out, void* stream) {
  if (p == nullptr || ws == nullptr || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return CORA_ERR_INVALID;
  const size_t need = cora_encoder_forward_workspace_bytes(p, batch, total_tokens, max_len);
  if (need == 0 || ws_bytes < need) return CORA_ERR_INVALID;
  const size_t lay_bytes = cora_layout_workspace_bytes(batch, total_tokens, p->heads, max_len);
  uint8_t* w = static_cast<uint8_t*>(ws);
  cora_layout_t L;
  const size_t off = align_up(lay_bytes);
  return forward_impl(p, lengths, batch, total_tokens, max_len, w, lay_bytes, x, y, w + off, ws_bytes - off, &L,
                      layout_out, stream);
}

int32_t cora_encoder_layer_launches(const cora_encoder_params_t* p, int32_t total_tokens) {
  if (p == nullptr || total_tokens < 0) return -1;
  if (total_tokens == 0) return 0;
  GemmArgs g{nullptr, p->w_o, p->b_o, p->w_o, nullptr, total_tokens, p->d_model, p->d_model, CORA_ACT_NONE};
  g.ln_gamma = static_cast<const float*>(p->ln1_g);
  g.ln_beta = static_cast<const float*>(p->ln1_b);
  return gemm_ln_supported(g) ? 5 : 7;
}

cora_status_t cora_encoder_layer_fwd(const cora_encoder_params_t* p, const cora_layout_t* layout, const void* x,
                                     void* y, void* ws, size_t ws_bytes, void* stream) {
  return cora_encoder_layer_fwd_ex(p, layout, x, y, ws, ws_bytes, stream, nullptr);
}

size_t cora_encoder_stack_workspace_bytes(const cora_encoder_params_t* layers, int32_t n_layers, int32_t total_tokens) {
  if (layers == nullptr || n_layers < 1 || total_tokens < 0) return 0;
  size_t layer_ws = 0;
  for (int i = 0; i < n_layers; ++i) {
    const size_t b = carve_encoder(&layers[i], total_tokens).total;
    if (b > layer_ws) layer_ws = b;
  }
  // + one [T, d] activation buffer: the layers ping-pong between it and y
  return layer_ws + (n_layers > 1 ? align_up(2ull * static_cast<size_t>(total_tokens) * layers[0].d_model) : 0);
}

cora_status_t cora_encoder_stack_fwd(const cora_encoder_params_t* layers, int32_t n_layers, const cora_layout_t* layout,
                                     const void* x, void* y, void* ws, size_t ws_bytes, void* stream) {
  if (layers == nullptr || layout == nullptr || n_layers < 1) return CORA_ERR_INVALID;
  for (int i = 1; i < n_layers; ++i)
    if (layers[i].d_model != layers[0].d_model || layers[i].heads != layers[0].heads) return CORA_ERR_INVALID;
  const int32_t T = layout->total_tokens;
  const size_t need = cora_encoder_stack_workspace_bytes(layers, n_layers, T);
  if (need == 0 || ws == nullptr || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0)
    return CORA_ERR_INVALID;
  if (T == 0 || layout->batch == 0) return CORA_OK;
  uint8_t* w = static_cast<uint8_t*>(ws);
  void* tmp = nullptr;
  if (n_layers > 1) {
    tmp = w;
    w += align_up(2ull * static_cast<size_t>(T) * layers[0].d_model);
  }
  const size_t layer_ws = ws_bytes - static_cast<size_t>(w - static_cast<uint8_t*>(ws));
  // layer i writes y when (n_layers - 1 - i) is even, else tmp, so the last layer lands in y and no layer
  // reads and writes the same buffer
  const void* in = x;
  for (int i = 0; i < n_layers; ++i) {
    void* out = ((n_layers - 1 - i) % 2 == 0) ? y : tmp;
    const cora_status_t st = cora_encoder_layer_fwd_ex(&layers[i], layout, in, out, w, layer_ws, stream, nullptr);
    if (st != CORA_OK) return st;
    in = out;
  }
  return CORA_OK;
}

size_t cora_forward_host_workspace_bytes(const cora_encoder_params_t* p, int32_t batch, int32_t total_tokens,
                                         int32_t max_len) {
  if (p == nullptr || !layout_args_ok(batch, total_tokens, p->heads, max_len)) return 0;
  const size_t xy = align_up(2ull * static_cast<size_t>(total_tokens) * p->d_model);
  // lengths + x + y + the whole batch's layout (layout_out) + one chunk layout + the layer workspace
  return align_up(sizeof(int32_t) * (batch + 1)) + 2 * xy +
         2 * cora_layout_workspace_bytes(batch, total_tokens, p->heads, max_len) + carve_encoder(p, total_tokens).total;
}

namespace {
// Side streams and events of the pipelined host forward, created once per device (never on the hot path
// after the first call).
constexpr int kMaxChunks = 16;
// The host pipeline of one device: two side streams + fork/join events, a capture stream, and the CUDA
// graph of the last call (re-used while the call's arguments are the same: its enqueue cost -- ~100 kernel
// launches and copies at 16 chunks, ~0.8 ms of host time -- would otherwise bound the call).
struct HostGraph {
  uint64_t key = 0;  // hash of every argument that shapes the enqueued work (0: none cached)
  cudaGraphExec_t exec = nullptr;
  cora_layout_t layout{};
  bool has_layout = false;
};
struct HostPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr, cap = nullptr;
  cudaEvent_t start = nullptr, done = nullptr, h2d_ev[kMaxChunks] = {}, comp_ev[kMaxChunks] = {};
  HostGraph graph;
  bool ok = false;
};
HostPipe g_pipe[64];
std::mutex g_pipe_mu;

HostPipe* host_pipe() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe& hp = g_pipe[dev];
  if (!hp.ok) {
    bool good = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&hp.cap, cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming) == cudaSuccess;
    for (int c = 0; good && c < kMaxChunks; ++c)
      good = cudaEventCreateWithFlags(&hp.h2d_ev[c], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&hp.comp_ev[c], cudaEventDisableTiming) == cudaSuccess;
    if (!good) return nullptr;
    hp.ok = true;
  }
  return &hp;
}
#ifdef CORA_HOST_TRACE
// Pipeline timeline (profiling builds only, with CORA_HOST_NO_GRAPH set): timing events after each chunk's
// H2D, layer and D2H, read back by cora_debug_host_trace.
struct HostTrace {
  bool on = false, made = false;
  int K = 0;
  cudaEvent_t t0 = nullptr, h2d[kMaxChunks] = {}, comp[kMaxChunks] = {}, d2h[kMaxChunks] = {};
};
HostTrace g_htrace;
void htrace_rec(cudaEvent_t* e, cudaStream_t st) {
  if (!g_htrace.on) return;
  if (*e == nullptr) cudaEventCreate(e);
  cudaEventRecord(*e, st);
}
#define HTRACE(e, st) htrace_rec(&g_htrace.e, st)
#else
#define HTRACE(e, st) \
  do {                \
  } while (0)
#endif

// FNV-1a over raw bytes (the graph-cache key)
uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// Number of pipeline chunks for a batch (1 = one shot): the lengths are on the host, so the batch is cut
// there; invalid lengths disable the chunking (the device status word reports them).
int host_chunks(const int32_t* lengths_host, int32_t batch, int32_t total_tokens, int32_t max_len) {
  int64_t sum = 0;
  bool bad = false;
  for (int b = 0; b < batch; ++b) {
    sum += lengths_host[b];
    bad |= lengths_host[b] < 0 || lengths_host[b] > max_len;
  }
  int K = (bad || sum != total_tokens) ? 1
          : total_tokens >= 32768 ? 16
          : total_tokens >= 16384 ? 8
          : total_tokens >= 8192  ? 4
                                  : 1;
  if (const char* e = getenv("CORA_HOST_CHUNKS")) {  // experiments: force the chunk count (1..16)
    const int k = atoi(e);
    if (k >= 1 && k <= kMaxChunks && !bad && sum == total_tokens) K = k;
  }
  if (K > batch) K = batch > 0 ? batch : 1;
  return K;
}

// Enqueue the whole host-buffer forward on stream `s` (the caller's, or the capture stream).
cora_status_t host_forward_enqueue(const cora_encoder_params_t* p, const int32_t* lengths_host, int32_t batch,
                                   int32_t total_tokens, int32_t max_len, const void* x_host, void* y_host, void* ws,
                                   size_t ws_bytes, cora_layout_t* layout_out, cudaStream_t s, int K, HostPipe* hp) {
  void* stream = s;
  const int32_t d = p->d_model;
  const size_t xbytes = 2ull * static_cast<size_t>(total_tokens) * d;
  const size_t xy = align_up(xbytes);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int32_t* d_len = reinterpret_cast<int32_t*>(w);
  w += align_up(sizeof(int32_t) * (batch + 1));
  uint8_t* d_x = w;
  w += xy;
  uint8_t* d_y = w;
  w += xy;
  const size_t lay_bytes = cora_layout_workspace_bytes(batch, total_tokens, p->heads, max_len);
  void* lay_ws = w;  // the whole batch's layout (layout_out)
  w += lay_bytes;
  void* chunk_lay_ws = w;  // the current chunk's layout
  w += lay_bytes;
  const size_t layer_ws = ws_bytes - static_cast<size_t>(w - static_cast<uint8_t*>(ws));

  // K contiguous sequence ranges of ~T/K tokens each are copied in, computed and copied out as a pipeline
  // over three streams (H2D of chunk c+1 and D2H of chunk c-1 overlap the layer on chunk c; PCIe is full
  // duplex): sequences are independent, so a chunk is a ragged batch of its own (its layout rebased to its
  // first token).
  int32_t seq_begin[kMaxChunks + 1], tok_begin[kMaxChunks + 1];
  seq_begin[0] = 0, tok_begin[0] = 0;
  {
    int b = 0;
    int64_t acc = 0;
    for (int c = 1; c < K; ++c) {
      const int64_t target = static_cast<int64_t>(total_tokens) * c / K;
      while (b < batch && acc + lengths_host[b] <= target) acc += lengths_host[b++];
      seq_begin[c] = b, tok_begin[c] = static_cast<int32_t>(acc);
    }
    seq_begin[K] = batch, tok_begin[K] = total_tokens;
  }
  if (hp == nullptr) K = 1, seq_begin[1] = batch, tok_begin[1] = total_tokens;

  if (batch > 0 && cudaMemcpyAsync(d_len, lengths_host, sizeof(int32_t) * batch, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return CORA_ERR_CUDA;
  if (layout_out != nullptr || K == 1) {
    // the whole batch's layout: the status word checks sum L == T and 0 <= L <= max_len on the device
    cora_layout_t L;
    const cora_status_t st = cora_layout_build(d_len, batch, total_tokens, p->heads, max_len, lay_ws, lay_bytes, &L, stream);
    if (st != CORA_OK) return st;
    if (layout_out != nullptr) *layout_out = L;
    if (K == 1) {
      if (xbytes > 0 && cudaMemcpyAsync(d_x, x_host, xbytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return CORA_ERR_CUDA;
      const cora_status_t st2 = encoder_layer_impl(p, &L, d_x, d_y, w, layer_ws, stream, nullptr, true);
      if (st2 != CORA_OK) return st2;
      if (xbytes > 0 && cudaMemcpyAsync(y_host, d_y, xbytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return CORA_ERR_CUDA;
      return CORA_OK;
    }
  }
  // pipelined: fork the side streams off the caller's stream, join them back at the end
#ifdef CORA_HOST_TRACE
  g_htrace.on = true;
  g_htrace.K = K;
#endif
  HTRACE(t0, s);
  if (cudaEventRecord(hp->start, s) != cudaSuccess || cudaStreamWaitEvent(hp->h2d, hp->start, 0) != cudaSuccess ||
      cudaStreamWaitEvent(hp->d2h, hp->start, 0) != cudaSuccess)
    return CORA_ERR_CUDA;
  const size_t row = 2ull * d;
  for (int c = 0; c < K; ++c) {
    const size_t off = row * tok_begin[c], bytes = row * (tok_begin[c + 1] - tok_begin[c]);
    if (bytes > 0 && cudaMemcpyAsync(d_x + off, static_cast<const uint8_t*>(x_host) + off, bytes,
                                     cudaMemcpyHostToDevice, hp->h2d) != cudaSuccess)
      return CORA_ERR_CUDA;
    if (cudaEventRecord(hp->h2d_ev[c], hp->h2d) != cudaSuccess) return CORA_ERR_CUDA;
    HTRACE(h2d[c], hp->h2d);
  }
  for (int c = 0; c < K; ++c) {
    const int32_t nb = seq_begin[c + 1] - seq_begin[c], nt = tok_begin[c + 1] - tok_begin[c];
    if (cudaStreamWaitEvent(s, hp->h2d_ev[c], 0) != cudaSuccess) return CORA_ERR_CUDA;
    if (nt > 0) {
      cora_layout_t Lc;
      const cora_status_t st = forward_impl(p, d_len + seq_begin[c], nb, nt, max_len, chunk_lay_ws, lay_bytes,
                                            d_x + row * tok_begin[c], d_y + row * tok_begin[c], w, layer_ws, &Lc,
                                            nullptr, stream);
      if (st != CORA_OK) return st;
    }
    if (cudaEventRecord(hp->comp_ev[c], s) != cudaSuccess) return CORA_ERR_CUDA;
    HTRACE(comp[c], s);
    if (cudaStreamWaitEvent(hp->d2h, hp->comp_ev[c], 0) != cudaSuccess) return CORA_ERR_CUDA;
    const size_t off = row * tok_begin[c], bytes = row * nt;
    if (bytes > 0 && cudaMemcpyAsync(static_cast<uint8_t*>(y_host) + off, d_y + off, bytes, cudaMemcpyDeviceToHost,
                                     hp->d2h) != cudaSuccess)
      return CORA_ERR_CUDA;
    HTRACE(d2h[c], hp->d2h);
  }
  if (cudaEventRecord(hp->done, hp->d2h) != cudaSuccess || cudaStreamWaitEvent(s, hp->done, 0) != cudaSuccess)
    return CORA_ERR_CUDA;
  return CORA_OK;
}
}  // namespace

#ifdef CORA_HOST_TRACE
// profiling: ms from the pipeline start to each chunk's H2D / layer / D2H completion (3 x K values)
extern "C" int cora_debug_host_trace(float* out, int max_chunks) {
  if (!g_htrace.on || g_htrace.t0 == nullptr) return 0;
  const int K = g_htrace.K < max_chunks ? g_htrace.K : max_chunks;
  cudaDeviceSynchronize();
  for (int c = 0; c < K; ++c) {
    cudaEventElapsedTime(&out[c], g_htrace.t0, g_htrace.h2d[c]);
    cudaEventElapsedTime(&out[K + c], g_htrace.t0, g_htrace.comp[c]);
    cudaEventElapsedTime(&out[2 * K + c], g_htrace.t0, g_htrace.d2h[c]);
  }
  return K;
}
#endif

cora_status_t cora_encoder_forward_host(const cora_encoder_params_t* p, const int32_t* lengths_host, int32_t batch,
                                        int32_t total_tokens, int32_t max_len, const void* x_host, void* y_host,
                                        void* ws, size_t ws_bytes, cora_layout_t* layout_out, void* stream) {
  if (p == nullptr || !layout_args_ok(batch, total_tokens, p->heads, max_len)) return CORA_ERR_INVALID;
  if ((batch > 0 && lengths_host == nullptr) || ws == nullptr || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0)
    return CORA_ERR_INVALID;
  if (total_tokens > 0 && (x_host == nullptr || y_host == nullptr)) return CORA_ERR_INVALID;
  const size_t need = cora_forward_host_workspace_bytes(p, batch, total_tokens, max_len);
  if (need == 0 || ws_bytes < need) return CORA_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  int K = host_chunks(lengths_host, batch, total_tokens, max_len);
  HostPipe* hp = K > 1 ? host_pipe() : nullptr;
  if (hp == nullptr) K = 1;
  if (K == 1 || getenv("CORA_HOST_NO_GRAPH") != nullptr)
    return host_forward_enqueue(p, lengths_host, batch, total_tokens, max_len, x_host, y_host, ws, ws_bytes,
                                layout_out, s, K, hp);
  // Pipelined calls replay a CUDA graph of the enqueued work, captured on the library's capture stream
  // (the caller's stream may be the legacy default stream, which cannot be captured) and launched on the
  // caller's stream.  The key covers every argument the enqueue depends on: the parameter struct (weight
  // pointers, dims, activation, eps), the lengths, the sizes, the host and workspace pointers, the chunk
  // count and whether a whole-batch layout is wanted.
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t key = 1469598103934665603ull;
  key = fnv1a(key, p, sizeof(*p));
  key = fnv1a(key, lengths_host, sizeof(int32_t) * static_cast<size_t>(batch));
  const int64_t scal[5] = {batch, total_tokens, max_len, K, layout_out != nullptr};
  const void* ptrs[3] = {x_host, y_host, ws};
  key = fnv1a(key, scal, sizeof(scal));
  key = fnv1a(key, ptrs, sizeof(ptrs));
  key = fnv1a(key, &ws_bytes, sizeof(ws_bytes));
  key = fnv1a(key, &dev, sizeof(dev));
  key |= 1;  // 0 means "nothing cached"
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostGraph& g = hp->graph;
  if (g.key != key) {
    if (g.exec != nullptr) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr, g.key = 0;
    cora_layout_t lay{};
    if (cudaStreamBeginCapture(hp->cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return CORA_ERR_CUDA;
    const cora_status_t st = host_forward_enqueue(p, lengths_host, batch, total_tokens, max_len, x_host, y_host, ws,
                                                  ws_bytes, layout_out != nullptr ? &lay : nullptr, hp->cap, K, hp);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(hp->cap, &graph);
    if (st != CORA_OK || ce != cudaSuccess || graph == nullptr) {
      if (graph != nullptr) cudaGraphDestroy(graph);
      cudaGetLastError();
      // not capturable here (e.g. pageable host buffers): enqueue directly
      return st != CORA_OK ? st
                           : host_forward_enqueue(p, lengths_host, batch, total_tokens, max_len, x_host, y_host, ws,
                                                  ws_bytes, layout_out, s, K, hp);
    }
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      g.exec = nullptr;
      return CORA_ERR_CUDA;
    }
    g.key = key, g.layout = lay, g.has_layout = layout_out != nullptr;
  }
  if (cudaGraphLaunch(g.exec, s) != cudaSuccess) return CORA_ERR_CUDA;
  if (layout_out != nullptr && g.has_layout) *layout_out = g.layout;
  return CORA_OK;
}

const char* cora_status_string(cora_status_t s) {
  switch (s) {
    case CORA_OK:
      return "ok";
    case CORA_ERR_INVALID:
      return "invalid argument";
    case CORA_ERR_DATA:
      return "data error (bad lengths or sum(L) != T)";
    case CORA_ERR_CUDA:
      return "CUDA error";
    case CORA_ERR_UNSUPPORTED:
      return "unsupported shape";
    case CORA_ERR_NCCL:
      return "NCCL error";
    default:
      return "unknown status";
  }
}

int32_t cora_device_sm_count(void) { return device_sm_count(); }

const char* cora_build_info(void) { return "libcora_b200 sm_100a tcgen05/TMA; CUDA " CORA_CUDA_VERSION_STR; }

}  // extern "C"
