/*
 * cora.h -- C ABI of libcora_b200.so: the forward pass of one post-LN transformer
 * encoder layer over a RAGGED mini-batch on NVIDIA B200 (sm_100a), after
 * "The CoRa Tensor Compiler: Compilation for Ragged Tensors with Minimal
 * Padding" (Fegade et al., MLSys 2022, arXiv 2110.10221).
 *
 * Problem statement: a ragged tensor is
 * a dense buffer plus per-sequence lengths/offsets; a ragged operator takes
 * ragged tensors in and produces a ragged tensor out.  The raggedness (the
 * lengths) is known before the computation and is shared by every layer
 * (PAPER.md:333-349, 955-958), so it is turned into offset tables once
 * (cora_layout_build, the "prelude" of PAPER.md:364-380) and reused.
 *
 * Conventions for every entry point
 *  - Pointers are DEVICE pointers unless the name ends in `_host`.
 *  - Streams are `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 *    All device work is enqueued asynchronously on that stream; nothing
 *    synchronises the host except cora_layout_status.
 *  - Ownership: the caller owns every buffer (inputs, weights, outputs,
 *    workspaces) and the stream; the library never allocates device memory
 *    and never frees caller memory ("expects users to
 *    correctly allocate memory").
 *  - Packed token layout: sequence b occupies rows [row_off[b], row_off[b]+L_b)
 *    of a row-major [T, C] matrix, T = sum_b L_b, no padding rows.
 *    (loop + dimension fusion; fused bound F = sum_o s(o)).
 *  - bf16 matrices are row-major with 16-byte aligned base pointers and rows.
 *  - Errors: synchronous argument validation returns CORA_ERR_INVALID (1);
 *    data errors detected on the device (a negative length, L_b > max_len,
 *    sum L_b != T) are recorded in the layout's status word and reported by
 *    cora_layout_status as CORA_ERR_DATA (2) -- in that case the attention
 *    work list is empty and no kernel reads or writes out of range.  CUDA
 *    launch errors map to CORA_ERR_CUDA (3), unsupported shapes to
 *    CORA_ERR_UNSUPPORTED (4).  Mirrors SPEC.md:643 (0 ok, 1 validation,
 *    2 runtime data error).
 *  - Zero-length sequences are legal; batch == 0 or T == 0
 *    is a no-op returning CORA_OK.
 *  - Determinism: identical inputs give bitwise-identical outputs (no atomics
 *    in floating-point reductions, no split-K).
 */
#ifndef CORA_B200_H_
#define CORA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t cora_status_t;
enum {
  CORA_OK = 0,
  CORA_ERR_INVALID = 1,
  CORA_ERR_DATA = 2,
  CORA_ERR_CUDA = 3,
  CORA_ERR_UNSUPPORTED = 4,
  CORA_ERR_NCCL = 5
};

typedef int32_t cora_dtype_t;
enum { CORA_DT_BF16 = 0, CORA_DT_F32 = 1 };

typedef int32_t cora_act_t;
enum { CORA_ACT_NONE = 0, CORA_ACT_RELU = 1, CORA_ACT_GELU_ERF = 2 };

/* Device status word bits (cora_layout_t.status). */
enum { CORA_STATUS_BAD_LENGTH = 1, CORA_STATUS_SUM_MISMATCH = 2 };

/* Attention work-tile word: bits [0,16) = sequence b, [16,24) = head h,
 * [24,31) = q-tile qt (rows [128 qt, 128 qt + 128) of sequence b). */
#define CORA_TILE_ROWS 128
#define CORA_TILE_B(w) ((w) & 0xFFFF)
#define CORA_TILE_H(w) (((w) >> 16) & 0xFF)
#define CORA_TILE_QT(w) (((w) >> 24) & 0x7F)

/*
 * Offset tables of the ragged storage ("prelude"; A_d arrays
 * of App. B.1; fusion maps of App. B.2).
 * Filled by cora_layout_build; device tables live inside the caller's workspace.
 * Immutable after build; one layout serves every layer of the batch.
 */
typedef struct cora_layout {
  int32_t batch;        /* B */
  int32_t heads;        /* H */
  int32_t max_len;      /* upper bound on every L_b (validated on device) */
  int32_t total_tokens; /* T = sum_b L_b (host-known: the caller packed X) */
  int32_t n_tiles_max;  /* host bound on the attention work list length */
  int32_t _pad;
  int64_t total_attn;   /* host-visible S2 = sum_b L_b^2 (the ragged score tensor's size per head, A_1 of
                           X[b,i,h,j]): -1 after cora_layout_build (the lengths live on the device), filled
                           by cora_layout_status, which synchronises anyway */
  const int32_t* lengths; /* [B]   L_b (caller-owned) */
  int32_t* row_off;       /* [B+1] row_off[b] = sum_{j<b} L_j   (A_1 of [b,i,c], exclusive) */
  int64_t* attn_off;      /* [B+1] attn_off[b] = sum_{j<b} L_j^2 (A_1 of X[b,i,h,j]) */
  int32_t* seq_of_tok;    /* [T]   f_fo: fused token index -> sequence b */
  int32_t* pos_in_seq;    /* [T]   f_fi: fused token index -> position i (f_oif(b,i) = row_off[b]+i) */
  int32_t* tiles;         /* [n_tiles_max] attention work list, longest first */
  int32_t* tile_seq;      /* [2*n_tiles_max] (row_off[b], L_b) of each work tile (one 8-byte load) */
  int32_t* n_tiles;       /* [3]   n_tiles[0]: number of valid entries of `tiles` (0 if status != 0);
                             [1], [2]: the attention kernel's dynamic schedule (ticket counter, finished
                             CTAs), zeroed by cora_layout_build and reset by every attention launch --
                             attention launches on one layout must therefore not run concurrently */
  int32_t* status;        /* [1]   CORA_STATUS_* bits, 0 = ok */
  /* Attention work UNITS: pairs of consecutive q-tiles (2 qp, 2 qp + 1) of one (b, h) that share
   * their K/V tiles; same longest-first order.  Word layout as `tiles` with qt replaced by qp. */
  int32_t n_units_max;    /* host bound on the unit list length */
  int32_t _pad2;
  int32_t* units;         /* [n_units_max] */
  int32_t* unit_seq;      /* [2*n_units_max] (row_off[b], L_b) of each unit */
  int32_t* n_units;       /* [3]   n_units[0]: number of valid entries of `units` (0 if status != 0);
                             [1], [2]: the causal attention kernel's schedule words (as n_tiles) */
} cora_layout_t;

/* Encoder layer parameters (nn.Linear convention W[out, in], bf16; LayerNorm fp32).
 * w_qkv = [W_q; W_k; W_v] as [3d, d]; head h uses rows [h*d_h, (h+1)*d_h) of each block.
 * Hyper-parameters of the paper: d_model 512, 8 heads x 64, d_ff 2048. */
typedef struct cora_encoder_params {
  int32_t d_model, heads, d_ff;
  float ln_eps;   /* LayerNorm epsilon (reading c3: 1e-5) */
  cora_act_t act; /* FF1 activation (reading c1: ReLU) */
  int32_t _pad;
  const void *w_qkv, *b_qkv; /* [3d, d] bf16, [3d] bf16 */
  const void *w_o, *b_o;     /* [d, d], [d] */
  const void *ln1_g, *ln1_b; /* [d] fp32 */
  const void *w1, *b1;       /* [d_ff, d], [d_ff] */
  const void *w2, *b2;       /* [d, d_ff], [d] */
  const void *ln2_g, *ln2_b; /* [d] fp32 */
} cora_encoder_params_t;

/* ---------------------------------------------------------------- layout (step a1) */

/* Bytes of workspace cora_layout_build needs for this batch. */
size_t cora_layout_workspace_bytes(int32_t batch, int32_t total_tokens, int32_t heads, int32_t max_len);

/* Build the offset tables on the device (two kernels, no host synchronisation).
 * lengths: device int32 [batch].  ws: device workspace (>= cora_layout_workspace_bytes,
 * 256-byte aligned).  out: host struct filled with pointers into ws.
 * Computes row_off/attn_off (exclusive prefix sums, reading c7), seq_of_tok/pos_in_seq,
 * the attention tile list ordered by (-ceil(L_b/128), b, h, qt) (reading c15) and the
 * status word.  Returns CORA_ERR_INVALID on bad arguments (batch < 0, heads < 1 or > 255,
 * max_len < 0 or > 16383, batch > 65536, null pointers, small workspace). */
cora_status_t cora_layout_build(const int32_t* lengths, int32_t batch, int32_t total_tokens, int32_t heads,
                                int32_t max_len, void* ws, size_t ws_bytes, cora_layout_t* out, void* stream);

/* Synchronise `stream`, read the device status word (CORA_OK or CORA_ERR_DATA) and fill layout->total_attn. */
cora_status_t cora_layout_status(cora_layout_t* layout, void* stream);

/* ---------------------------------------------------------------- whole layer */

/* Workspace for cora_encoder_layer_fwd: QKV[T,3d] + O[T,d] + Y1[T,d] + H1[T,d] + F[T,d_ff] + Y2[T,d], bf16. */
size_t cora_encoder_workspace_bytes(const cora_encoder_params_t* p, int32_t total_tokens);

/* y[T, d] = EncoderLayer(x[T, d]) over the ragged batch described by `layout` (bf16 in/out).
 * When d_model == 512 and T > 128 the two "GEMM + bias + residual, LayerNorm" pairs run as single
 * fused kernels (cora_linear_residual_layernorm_fwd); otherwise as GEMM then LayerNorm kernels.
 * Steps (Table ap_op_times):
 *   QKV = x W_qkv^T + b_qkv                     (tcgen05 GEMM)
 *   O   = ragged MHA(QKV)                       (fused tcgen05 attention, longest-first tiles)
 *   Y1  = O W_o^T + b_o + x                     (GEMM + bias + residual)
 *   H1  = LN(Y1; ln1)                           (warp-per-row LayerNorm)
 *   F   = act(H1 W1^T + b1)                     (GEMM + bias + activation)
 *   Y2  = F W2^T + b2 + H1                      (GEMM + bias + residual)
 *   y   = LN(Y2; ln2)
 * x and y must not alias. */
cora_status_t cora_encoder_layer_fwd(const cora_encoder_params_t* p, const cora_layout_t* layout, const void* x,
                                     void* y, void* ws, size_t ws_bytes, void* stream);

/* Kernel launches cora_encoder_layer_fwd makes for this configuration (prelude excluded): 5 when the
 * two "GEMM + bias + residual, LayerNorm" pairs are fused (d_model == 512, total_tokens > 128 and
 * non-NULL LayerNorm parameters), else 7; 0 when total_tokens == 0; -1 on a NULL p or negative T. */
int32_t cora_encoder_layer_launches(const cora_encoder_params_t* p, int32_t total_tokens);

/* Number of events cora_encoder_layer_fwd_ex records (one before each of the 7 kernels + one after). */
#define CORA_LAYER_EVENTS 8

/* Same as cora_encoder_layer_fwd; when `events` is non-NULL it points to CORA_LAYER_EVENTS
 * cudaEvent_t handles (caller-created) and event k is recorded on `stream` right before step k
 * (0 QKV GEMM, 1 attention, 2 out-proj GEMM, 3 LN1, 4 FF1 GEMM, 5 FF2 GEMM, 6 LN2) and event 7
 * after the last one, so the caller can time every kernel of the layer on the launching stream.
 * With the fused GEMM + LayerNorm kernels, steps 3 and 6 are empty (events 3 / 4 and 6 / 7 coincide). */
cora_status_t cora_encoder_layer_fwd_ex(const cora_encoder_params_t* p, const cora_layout_t* layout, const void* x,
                                        void* y, void* ws, size_t ws_bytes, void* stream, void* const* events);

/* Workspace for cora_encoder_forward: the layout tables + the layer workspace. */
size_t cora_encoder_forward_workspace_bytes(const cora_encoder_params_t* p, int32_t batch, int32_t total_tokens,
                                            int32_t max_len);

/* One ragged batch through one layer from its lengths: cora_layout_build (step a1) + the layer (a2..a8)
 * in one call, with the tables in `ws` (bitwise the tables cora_layout_build writes).  Batches of at most
 * 256 sequences: the QKV GEMM's epilogue warps build the tables while its first units' mainloops run (no
 * prelude kernel).  Larger batches: the prelude kernel runs and, because x must be complete before this
 * call, the QKV GEMM does not wait for it (it does not read the tables) and only waits before completing.
 * Either way the prelude is off the critical path.  lengths: device int32 [batch]; x, y as for
 * cora_encoder_layer_fwd; layout_out (may be NULL) receives the layout (for cora_layout_status).
 * Errors as cora_layout_build and cora_encoder_layer_fwd. */
cora_status_t cora_encoder_forward(const cora_encoder_params_t* p, const int32_t* lengths, int32_t batch,
                                   int32_t total_tokens, int32_t max_len, const void* x, void* y, void* ws,
                                   size_t ws_bytes, cora_layout_t* layout_out, void* stream);

/* Workspace for cora_encoder_stack_fwd: the largest layer workspace + one [T, d_model] bf16 buffer
 * (n_layers > 1); 0 on invalid arguments. */
size_t cora_encoder_stack_workspace_bytes(const cora_encoder_params_t* layers, int32_t n_layers, int32_t total_tokens);

/* y = layer_{n-1}( ... layer_0(x)) over one ragged batch: a stack of encoder layers (the paper's 6-layer
 * model) sharing ONE layout -- the prelude runs once per batch, not per layer, as the
 * raggedness is the same for every layer (SURVEY f-4).  layers: n_layers parameter
 * structs (same d_model and heads); activations ping-pong between y and a workspace buffer (x is only
 * read; x and y must not alias).  Same validation and errors as cora_encoder_layer_fwd. */
cora_status_t cora_encoder_stack_fwd(const cora_encoder_params_t* layers, int32_t n_layers, const cora_layout_t* layout,
                                     const void* x, void* y, void* ws, size_t ws_bytes, void* stream);

/* Workspace for cora_encoder_forward_host (device lengths + X + Y + layout tables + layer workspace). */
size_t cora_forward_host_workspace_bytes(const cora_encoder_params_t* p, int32_t batch, int32_t total_tokens,
                                         int32_t max_len);

/* End-to-end call with HOST buffers: copies lengths_host[batch] (int32) and x_host[T, d] (bf16)
 * host->device, builds the layout (step a1), runs the layer (a2..a8) and copies y_host[T, d] back,
 * all ordered after prior work on `stream` and before later work on it (asynchronous when the host
 * buffers are pinned; the caller synchronises the stream before reading y_host).  For T >= 8192 the
 * batch is cut (on the host, from lengths_host) into 4 (T >= 16384: 8; T >= 32768: 16) contiguous
 * sequence ranges that
 * are copied in, computed and copied out as a pipeline over the caller's stream and two library-owned
 * side streams (H2D of chunk c+1 and D2H of chunk c-1 overlap the layer on chunk c); each chunk is a
 * ragged batch of its own, so every row is computed as in the one-shot path (bitwise, except that
 * sequences of < 128 tokens may be packed into different attention windows).  The pipelined work is
 * captured once into a CUDA graph (on a library-owned stream) and replayed while every argument that
 * shapes it is unchanged -- the parameter struct, the lengths' contents, the sizes, the host / workspace
 * pointers and whether layout_out is given (a 64-bit hash of them); the contents of x_host are read at
 * replay time.  A call with other arguments re-captures; a capture failure (e.g. pageable host memory)
 * falls back to enqueueing directly; CORA_HOST_NO_GRAPH (environment) disables the graph.  The side
 * streams, events and graph are kept once per device; concurrent calls from several host threads on one
 * device are not supported.  The device status word is not read (no hidden sync): call cora_layout_status on
 * *layout_out (the whole batch's layout, built on `stream`) after synchronising to detect data errors
 * (invalid lengths also disable the chunking).  layout_out may be NULL (then no whole-batch layout is
 * built when chunking).  T = total_tokens must equal sum(lengths_host). */
cora_status_t cora_encoder_forward_host(const cora_encoder_params_t* p, const int32_t* lengths_host, int32_t batch,
                                        int32_t total_tokens, int32_t max_len, const void* x_host, void* y_host,
                                        void* ws, size_t ws_bytes, cora_layout_t* layout_out, void* stream);

/* ---------------------------------------------------------------- op-level entry points */

/* c[m, n] = act(a[m, k] w[n, k]^T + bias[n]) + residual[m, n]  (bf16, fp32 accumulate in TMEM).
 * bias and residual may be NULL.  Packed "vloop-fused" linear op over T = m tokens
 * (PAPER.md:598-604, 929-935).  Requires k % 8 == 0, n % 8 == 0, 16-byte aligned pointers. */
cora_status_t cora_linear_fwd(const void* a, const void* w, const void* bias, const void* residual, void* c,
                              int32_t m, int32_t n, int32_t k, cora_act_t act, void* stream);

/* c[m, n] = LN(act(a w^T + bias) + residual; gamma, beta, eps) with the LayerNorm (post-LN, biased
 * variance, fp32 statistics of the bf16-rounded pre-LN values, readings
 * c2/c3) fused into the GEMM epilogue: a 4-CTA cluster (two CTA pairs) owns full rows and exchanges the
 * row statistics (mean, M2 pairs merged with Chan's formula: no E[v^2] - mean^2 cancellation) through
 * distributed shared memory.  The fused kernel needs n == 512, m > 128 and act == CORA_ACT_NONE; other
 * shapes with n % 8 == 0 (an activation, another n) run the GEMM with its epilogue into c and then the
 * LayerNorm kernel in place on c (no temporary, no allocation).  n % 8 != 0: CORA_ERR_UNSUPPORTED;
 * residual, gamma, beta non-NULL; bias may be NULL. */
cora_status_t cora_linear_residual_layernorm_fwd(const void* a, const void* w, const void* bias, const void* residual,
                                                 const float* gamma, const float* beta, float eps, void* c, int32_t m,
                                                 int32_t n, int32_t k, cora_act_t act, void* stream);

/* o[T, H*d_h] = per sequence, per head softmax(Q_h K_h^T * scale) V_h on qkv[T, 3*H*d_h] (bf16).
 * Only keys j < L_b of the query's own sequence are attended (no padded rows or columns).
 * PAPER.md:296-300, 625-633, 2256-2259.  head_dim 64 runs the tcgen05 kernel; other head
 * dims (<= 128, even) run a SIMT kernel.  Uses layout->tiles / n_tiles / row_off / lengths. */
cora_status_t cora_ragged_attention_fwd(const cora_layout_t* layout, const void* qkv, void* o, int32_t head_dim,
                                        float scale, void* stream);

/* Masked (causal) variant: query i of sequence b attends to keys j <= i of b only -- the decoder's
 * masked MHA as a batch of lower-triangular ragged matrices (App. D.3
 * PAPER.md:1752-1806).  KV tiles above the diagonal are neither loaded nor computed. */
cora_status_t cora_ragged_masked_attention_fwd(const cora_layout_t* layout, const void* qkv, void* o,
                                               int32_t head_dim, float scale, void* stream);

/* Row softmax of the ragged attention matrix X[b, i, h, 0:L_b] stored flat at offset
 * H*attn_off[b] + (i*H + h)*L_b (App. B.1 lowering); x and y have
 * H * sum_b L_b^2 elements of dtype dt.  Warp-wide reductions. */
cora_status_t cora_ragged_softmax_fwd(const cora_layout_t* layout, const void* x, void* y, cora_dtype_t dt,
                                      void* stream);

/* y[r, :] = LN(x[r, :] (+ residual[r, :]); gamma, beta, eps), biased variance, fp32 math.
 * x, residual, y of dtype dt; gamma/beta fp32.  residual may be NULL.  cols % 8 == 0. */
cora_status_t cora_layernorm_fwd(const void* x, const void* residual, const float* gamma, const float* beta, void* y,
                                 int32_t rows, int32_t cols, float eps, cora_dtype_t dt, void* stream);

/* ---------------------------------------------------------------- vgemm / trmm (SURVEY f-3)
 * The paper's matrix-multiplication workloads (Sec. "Matrix Multiplication"), bf16
 * inputs, fp32 accumulation in TMEM, bf16 outputs, one persistent tcgen05 kernel (128 x 256 tiles). */

/* Bytes of the serialised vgemm work list ("plan") of these problems (0 on invalid arguments); also the
 * device workspace cora_vgemm_fwd needs.  dims_host: [batch][3] = (M_i, N_i, K_i). */
size_t cora_vgemm_plan_bytes(int32_t batch, const int32_t* dims_host);
size_t cora_vgemm_workspace_bytes(int32_t batch, const int32_t* dims_host);

/* Build the work list of cora_vgemm_fwd on the host into caller memory plan_host (>= cora_vgemm_plan_bytes):
 * every 128 x 256 output tile of every problem, scheduled longest reduction first (stable).  Validation:
 * M_i <= m_max, N_i <= n_max, K_i <= k_max, n_max % 8 == 0, k_max % 8 == 0 (CORA_ERR_INVALID); K_i % 64 == 0
 * unless K_i == k_max (a partial last k-block would read A/B padding: CORA_ERR_UNSUPPORTED). */
cora_status_t cora_vgemm_plan(int32_t batch, const int32_t* dims_host, int32_t m_max, int32_t n_max, int32_t k_max,
                              void* plan_host, size_t plan_bytes);

/* Variable-sized batched GEMM: C_i = A_i B_i for every problem of the plan, each with its
 * own (M_i, N_i, K_i).  Fully padded storage as in the paper's evaluation: a = A
 * [batch, m_max, k_max], b = B [batch, k_max, n_max], c = C [batch, m_max, n_max], row-major bf16 device
 * buffers (caller-owned).  Only C_i[:M_i, :N_i] is written (the padding of c is left untouched; K_i == 0
 * gives C_i = 0) and only K_i of each reduction is visited.  The plan (cora_vgemm_plan) is copied into ws
 * (>= cora_vgemm_workspace_bytes) with one cudaMemcpyAsync on `stream`: from PINNED host memory the call is
 * stream-capturable (a memcpy node that re-reads plan_host at every replay; keep it alive and unchanged).
 * 16-B aligned pointers.  An empty plan is a no-op.  CORA_ERR_INVALID on bad arguments / small ws. */
cora_status_t cora_vgemm_fwd(const void* plan_host, const void* a, const void* b, void* c, int32_t m_max, int32_t n_max,
                             int32_t k_max, void* ws, size_t ws_bytes, void* stream);

/* Triangular matrix multiplication: c[n, n_cols] = tril(l) b, l [n, n] and
 * b [n, n_cols] row-major bf16.  Only the lower triangle of l (diagonal included) is read (BLAS trmm
 * semantics; the upper triangle may hold anything).  Row tile r reduces over k < 128 (r + 1) only; the
 * blocks straddling the diagonal are masked in shared memory; row tiles run longest first.
 * Requires n % 8 == 0, n_cols % 8 == 0, 16-B aligned pointers.  No workspace. */
cora_status_t cora_trmm_fwd(const void* l, const void* b, void* c, int32_t n, int32_t n_cols, void* stream);

/* ---------------------------------------------------------------- multi-GPU (host logic) */

/* Short-sequence windows (reading f4-r1) are built by the prelude for batches of at most this many sequences. */
#define CORA_PACK_MAX_BATCH 1024

/* Contiguous sequence partition over n_ranks minimising the max per-rank cost,
 * cost(L) = 2L(4d^2 + 2 d d_ff) + 4 d L^2 (the sequence's useful FLOPs; BASELINE.json
 * north_star "balanced on sum(L_i d + L_i^2) FLOPs"); canonical greedy-left among optimal
 * plans (reading s1).  A boundary never splits a short-sequence window of the batch (reading s2:
 * batches of <= CORA_PACK_MAX_BATCH sequences), so every rank rebuilds the one-GPU windows of its
 * sequences and the sharded result equals the one-GPU result row for row.  Host-only (no GPU needed).
 * seq_begin_host[0..n_ranks]: rank r owns sequences [begin[r], begin[r+1]); row_begin_host[0..n_ranks]
 * (may be NULL): the same ranges as packed token rows (the exclusive prefix of the lengths at begin[r]).
 * CORA_ERR_INVALID on bad arguments (n_ranks < 1, batch < 0, a negative length, NULL pointers). */
cora_status_t cora_shard_plan(const int32_t* lengths_host, int32_t batch, int32_t d_model, int32_t d_ff,
                              int32_t n_ranks, int32_t* seq_begin_host, int32_t* row_begin_host);

/* Split every rank's range of a plan into n_groups contiguous groups of about equal token counts, cutting
 * only where cora_shard_plan may cut (groups may be empty).  group_seq_host / group_row_host:
 * [n_ranks][n_groups + 1] (row-major; group_row_host may be NULL): group g of rank r is sequences
 * [gs[r][g], gs[r][g+1]) = rows [gr[r][g], gr[r][g+1]).  Deterministic: every rank derives the same groups
 * (the schedule of cora_encoder_stack_sharded_fwd's overlapped gather).  Host-only. */
cora_status_t cora_shard_groups(const int32_t* lengths_host, int32_t batch, const int32_t* seq_begin_host,
                                int32_t n_ranks, int32_t n_groups, int32_t* group_seq_host, int32_t* group_row_host);

/* The final all-gather of the sequence-sharded layer's ragged outputs over NCCL, resolved
 * at run time (dlopen of libnccl.so.2: the copy torch loaded when called from Python).  Bootstrap: rank 0
 * calls cora_comm_get_unique_id, the caller distributes the cora_comm_unique_id_bytes() bytes (e.g. with
 * torch.distributed), every rank calls cora_comm_init (collective: all ranks, on their own GPU).
 * CORA_ERR_NCCL if NCCL cannot be loaded or fails; CORA_ERR_INVALID on bad arguments. */
int32_t cora_comm_unique_id_bytes(void);
cora_status_t cora_comm_get_unique_id(void* id_out_host);
cora_status_t cora_comm_init(void** comm, const void* nccl_unique_id_host, int32_t n_ranks, int32_t rank);
cora_status_t cora_comm_destroy(void* comm);

/* In-place variable-size all-gather of out[T, d] (dt = bf16 or fp32, device): rank r owns rows
 * [row_begin_host[r], row_begin_host[r+1]) (cora_shard_plan's row_begin_host, [n_ranks + 1] of the
 * communicator); after the call every rank holds all T rows in the original order.  ncclGroupStart; one
 * ncclBroadcast per rank with a non-empty range (root r); ncclGroupEnd -- enqueued on `stream`.  A
 * one-rank communicator is a no-op.  Collective: every rank of the communicator calls it with the same table. */
cora_status_t cora_allgather_ragged(void* comm, const int32_t* row_begin_host, void* out, int32_t d, cora_dtype_t dt,
                                    void* stream);

/* Workspace for cora_encoder_stack_sharded_fwd: one layout (batch bound) + cora_encoder_stack_workspace_bytes. */
size_t cora_encoder_stack_sharded_workspace_bytes(const cora_encoder_params_t* layers, int32_t n_layers, int32_t batch,
                                                  int32_t total_tokens, int32_t max_len);

/* The sequence-sharded encoder stack with its gather: every rank computes the layers
 * of its sequences (cora_shard_plan from lengths_host, identical on every rank) and, at the end, holds all
 * T output rows.  The rank's range is cut into n_groups window-aligned groups (cora_shard_groups); each
 * group is ONE ragged batch through all n_layers layers on ONE layout (the prelude once per group, not per
 * layer: PAPER.md:955-959), and as soon as group g is done its rows leave for every rank (one grouped set of
 * in-place ncclBroadcasts per group, on a library-owned side stream) while group g + 1 computes -- the
 * gather is amortised over the layers and overlapped with the compute.  lengths: device int32 [batch];
 * lengths_host: the same on the host (sum must equal total_tokens); x, y: [T, d_model] bf16 device buffers
 * indexed by packed row (only the rank's own rows of x are read; all of y is written), x != y.
 * comm: a communicator (cora_comm_init) or NULL for one rank (no collective).  n_groups in [1, 16].
 * The caller's stream waits for the side stream before the call returns its work (the call is asynchronous).
 * Collective when comm has > 1 rank: every rank calls it with the same lengths_host / n_groups. */
cora_status_t cora_encoder_stack_sharded_fwd(const cora_encoder_params_t* layers, int32_t n_layers,
                                             const int32_t* lengths, const int32_t* lengths_host, int32_t batch,
                                             int32_t total_tokens, int32_t max_len, void* comm, int32_t n_groups,
                                             const void* x, void* y, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- misc */
const char* cora_status_string(cora_status_t s);
/* Number of SMs of the current device (for callers sizing their own grids); -1 on error. */
int32_t cora_device_sm_count(void);
/* Library build string (arch, version). */
const char* cora_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* CORA_B200_H_ */
