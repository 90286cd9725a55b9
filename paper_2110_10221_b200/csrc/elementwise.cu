// Steps a5/a8 (LayerNorm) and a3' (standalone ragged softmax): HBM-bound warp-per-row kernels.
//
// Both use warp-wide shuffle reductions instead of block-wide ones, the schedule CoRa found
// faster than FasterTransformer's block reductions (App. D.6): no
// __syncthreads, and the reduction never touches padding because rows are read at their
// exact ragged extent.
#include <cuda_bf16.h>

#include <cstdint>

#include "cora_internal.h"
#include "ptx.cuh"

namespace cora {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
struct Vec;  // 16-byte vectors
template <>
struct Vec<float> {
  static constexpr int E = 4;
  __device__ static void load(const float* p, float* v) {
    float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
  }
  __device__ static void store(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int E = 8;
  __device__ static void load(const __nv_bfloat16* p, float* v) {
    uint4 q = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// LayerNorm kernels may run in place (y == x): every row is read completely by the warp that writes it.
//
// Persistent warps; NV 16-byte vectors per lane held in registers (cols <= 32 * NV * E).  gamma and
// beta are staged once per block in shared memory; each warp streams RPW rows per iteration with
// all loads issued before the reductions (memory-level parallelism for an HBM-bound kernel).
template <typename T, int NV, int RPW>
__global__ void __launch_bounds__(256, 4) layernorm_kernel(const T* x, const T* __restrict__ res,
                                                           const float* __restrict__ gamma,
                                                           const float* __restrict__ beta, T* y,
                                                           int32_t rows, int32_t cols, float eps) {
  constexpr int E = Vec<T>::E;
  // gamma/beta staged lane-major: element e of lane l's j-th vector at [(j*E + e)*32 + l], so a
  // warp reading "its" parameter for (j, e) touches 32 consecutive words (no bank conflicts).
  extern __shared__ float4 gb_smem[];
  const int nvec = cols / E;
  const int slots = ((nvec + 31) / 32) * 32 * E;
  float* sg = reinterpret_cast<float*>(gb_smem);
  float* sb = sg + slots;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const int vi = c / E, e = c % E;
    const int idx = ((vi >> 5) * E + e) * 32 + (vi & 31);
    sg[idx] = __ldg(gamma + c);
    sb[idx] = __ldg(beta + c);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const float inv_cols = 1.0f / cols;
  for (int row0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW; row0 < rows;
       row0 += warps_total * RPW) {
    float v[RPW][NV][E];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int row = row0 + r;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int vi = lane + 32 * j;
        if (row < rows && vi < nvec) {
          const size_t off = static_cast<size_t>(row) * cols + vi * E;
          Vec<T>::load(x + off, v[r][j]);
          if (res != nullptr) {
            float rr[E];
            Vec<T>::load(res + off, rr);
#pragma unroll
            for (int e = 0; e < E; ++e) v[r][j][e] += rr[e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) v[r][j][e] = 0.f;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int row = row0 + r;
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int e = 0; e < E; ++e) s += v[r][j][e];
      const float mean = warp_sum(s) * inv_cols;
      float q = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (lane + 32 * j < nvec) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const float dlt = v[r][j][e] - mean;
            q += dlt * dlt;
          }
        }
      }
      const float rstd = rsqrtf(warp_sum(q) * inv_cols + eps);
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const int vi = lane + 32 * j;
          if (vi < nvec) {
            float o[E];
#pragma unroll
            for (int e = 0; e < E; ++e)
              o[e] = (v[r][j][e] - mean) * rstd * sg[(j * E + e) * 32 + lane] + sb[(j * E + e) * 32 + lane];
            Vec<T>::store(y + static_cast<size_t>(row) * cols + vi * E, o);
          }
        }
      }
    }
  }
}

// Residual-free LayerNorm with bulk-copy staging: a producer warp streams chunks of RC contiguous rows
// (<= 32 KB) into a 3-stage shared-memory ring with cp.async.bulk (the bytes in flight per SM no longer
// depend on registers: 2 CTAs x 3 stages x 32 KB); 8 consumer warps normalise the rows straight out of
// shared memory and write 16-B vectors to global memory.  Lane l owns columns {(l + 32 j) E + e}, so
// gamma / beta live in registers for the whole kernel.
constexpr int kLnStages = 3;
constexpr int kLnChunkBytes = 32 * 1024;
constexpr int kLnConsumers = 8;

template <typename T, int NV, int RPW>
__global__ void __launch_bounds__(32 * (kLnConsumers + 1), 2)
    layernorm_bulk_kernel(const T* x, const float* __restrict__ gamma, const float* __restrict__ beta,
                          T* y, int32_t rows, int32_t cols, int32_t rc, float eps) {
  constexpr int E = Vec<T>::E;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ln_smem + kLnStages * kLnChunkBytes);
  uint64_t* empty = full + kLnStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_chunks = (rows + rc - 1) / rc;
  const size_t row_bytes = static_cast<size_t>(cols) * sizeof(T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kLnConsumers);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // the input rows (previous kernel) are complete and visible
  pdl_trigger();
  if (warp == kLnConsumers) {
    // ---- producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int r0 = c * rc, nr = min(rc, rows - r0);
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t bytes = static_cast<uint32_t>(nr * row_bytes);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_load(ln_smem + stage * kLnChunkBytes, reinterpret_cast<const uint8_t*>(x) + r0 * row_bytes, bytes,
                  &full[stage]);
        if (++stage == kLnStages) stage = 0, phase ^= 1;
      }
    }
    return;
  }
  // ---- consumers
  const int nvec = cols / E;
  const float inv_cols = 1.0f / cols;
  float g[NV][E], bt[NV][E];
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = (lane + 32 * j) * E + e;
      g[j][e] = c < cols ? __ldg(gamma + c) : 0.f;
      bt[j][e] = c < cols ? __ldg(beta + c) : 0.f;
    }
  int stage = 0;
  uint32_t phase = 0;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int r0 = c * rc, nr = min(rc, rows - r0);
    mbar_wait(&full[stage], phase);
    const T* xs = reinterpret_cast<const T*>(ln_smem + stage * kLnChunkBytes);
    // RPW rows per warp at a time, interleaved so their shuffle reductions overlap
    for (int rb = warp * RPW; rb < nr; rb += kLnConsumers * RPW) {
      float v[RPW][NV][E];
      float s[RPW];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        s[r] = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const int vi = lane + 32 * j;
          if (rb + r < nr && vi < nvec) {
            Vec<T>::load(xs + static_cast<size_t>(rb + r) * cols + vi * E, v[r][j]);
#pragma unroll
            for (int e = 0; e < E; ++e) s[r] += v[r][j][e];
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[r][j][e] = 0.f;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < RPW; ++r) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o);
      float q[RPW];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        s[r] *= inv_cols;  // mean
        q[r] = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (lane + 32 * j < nvec) {
#pragma unroll
            for (int e = 0; e < E; ++e) q[r] += (v[r][j][e] - s[r]) * (v[r][j][e] - s[r]);
          }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < RPW; ++r) q[r] += __shfl_xor_sync(0xffffffffu, q[r], o);
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        if (rb + r >= nr) break;
        const float rstd = rsqrtf(q[r] * inv_cols + eps);
        T* yr = y + static_cast<size_t>(r0 + rb + r) * cols;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const int vi = lane + 32 * j;
          if (vi < nvec) {
            float o[E];
#pragma unroll
            for (int e = 0; e < E; ++e) o[e] = (v[r][j][e] - s[r]) * rstd * g[j][e] + bt[j][e];
            Vec<T>::store(yr + vi * E, o);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kLnStages) stage = 0, phase ^= 1;
  }
}

// Rows wider than the register budget: three passes over global memory (L1/L2 hits after the first).
template <typename T>
__global__ void __launch_bounds__(256) layernorm_wide_kernel(const T* x, const T* __restrict__ res,
                                                             const float* __restrict__ gamma,
                                                             const float* __restrict__ beta, T* y,
                                                             int32_t rows, int32_t cols, float eps) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nvec = cols / E;
  const size_t rbase = static_cast<size_t>(row) * cols;
  auto load = [&](int vi, float* v) {
    Vec<T>::load(x + rbase + vi * E, v);
    if (res != nullptr) {
      float r[E];
      Vec<T>::load(res + rbase + vi * E, r);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] += r[e];
    }
  };
  float s = 0.f;
  for (int vi = lane; vi < nvec; vi += 32) {
    float v[E];
    load(vi, v);
#pragma unroll
    for (int e = 0; e < E; ++e) s += v[e];
  }
  const float mean = warp_sum(s) / cols;
  float q = 0.f;
  for (int vi = lane; vi < nvec; vi += 32) {
    float v[E];
    load(vi, v);
#pragma unroll
    for (int e = 0; e < E; ++e) q += (v[e] - mean) * (v[e] - mean);
  }
  const float rstd = rsqrtf(warp_sum(q) / cols + eps);
  for (int vi = lane; vi < nvec; vi += 32) {
    float v[E], o[E];
    load(vi, v);
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = (v[e] - mean) * rstd * gamma[vi * E + e] + beta[vi * E + e];
    Vec<T>::store(y + rbase + vi * E, o);
  }
}

template <typename T, int NV, int RPW = (NV == 1 ? 4 : 2)>
cudaError_t launch_layernorm_bulk(const T* x, const float* g, const float* b, T* y, int32_t rows, int32_t cols,
                                  float eps, cudaStream_t s) {
  const int row_bytes = cols * static_cast<int>(sizeof(T));
  int rc = kLnChunkBytes / row_bytes;  // rows per chunk
  if (rc > 64) rc = 64;
  const size_t smem = kLnStages * kLnChunkBytes + 2 * kLnStages * sizeof(uint64_t);
  static bool attr_set[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(layernorm_bulk_kernel<T, NV, RPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  const int chunks = (rows + rc - 1) / rc;
  const int cap = 2 * device_sm_count();
  return launch_pdl(layernorm_bulk_kernel<T, NV, RPW>, dim3(chunks < cap ? chunks : cap), dim3(32 * (kLnConsumers + 1)),
                    smem, s, 1, x, g, b, y, rows, cols, rc, eps);
}

template <typename T>
cudaError_t dispatch_layernorm(const void* x, const void* res, const float* g, const float* b, void* y, int32_t rows,
                               int32_t cols, float eps, cudaStream_t s) {
  constexpr int E = Vec<T>::E;
  const int per_lane = (cols / E + 31) / 32;
  const int row_bytes = cols * static_cast<int>(sizeof(T));
  if (res == nullptr && row_bytes % 16 == 0 && row_bytes <= kLnChunkBytes && per_lane <= 2) {
    if (per_lane <= 1)
      return launch_layernorm_bulk<T, 1>(static_cast<const T*>(x), g, b, static_cast<T*>(y), rows, cols, eps, s);
    return launch_layernorm_bulk<T, 2>(static_cast<const T*>(x), g, b, static_cast<T*>(y), rows, cols, eps, s);
  }
  const dim3 block(256);
  auto X = static_cast<const T*>(x);
  auto R = static_cast<const T*>(res);
  auto Y = static_cast<T*>(y);
  constexpr int RPW = 2;
  // persistent grid: 4 resident 256-thread blocks per SM, never more warps than row groups
  const int want = (rows + 8 * RPW - 1) / (8 * RPW);
  const int cap = device_sm_count() * 4;
  const dim3 grid(want < cap ? want : cap);
  const size_t smem = 2 * sizeof(float) * (((cols / E + 31) / 32) * 32 * E);
  if (per_lane <= 1)
    layernorm_kernel<T, 1, RPW><<<grid, block, smem, s>>>(X, R, g, b, Y, rows, cols, eps);
  else if (per_lane <= 2)
    layernorm_kernel<T, 2, RPW><<<grid, block, smem, s>>>(X, R, g, b, Y, rows, cols, eps);
  else if (per_lane <= 4)
    layernorm_kernel<T, 4, 1><<<grid, block, smem, s>>>(X, R, g, b, Y, rows, cols, eps);
  else
    layernorm_wide_kernel<T><<<dim3((rows + 7) / 8), block, 0, s>>>(X, R, g, b, Y, rows, cols, eps);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- ragged softmax (a3')
template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, float v);
template <>
__device__ __forceinline__ void st_f<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void st_f<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// One warp per row (b, i, h) of X[b, i, h, 0:L_b].  Row r = t*H + h with t the fused token index,
// b = f_fo(t), i = f_fi(t) (App. B.2 maps); the row starts at H*attn_off[b] + (i*H + h)*L_b
// (App. B.1 lowering).  Consecutive rows are contiguous, so a block streams a contiguous range.
template <typename T, int MAXE>
__global__ void __launch_bounds__(256) ragged_softmax_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                             const int32_t* __restrict__ lengths,
                                                             const int64_t* __restrict__ attn_off,
                                                             const int32_t* __restrict__ seq_of_tok,
                                                             const int32_t* __restrict__ pos_in_seq, int32_t heads,
                                                             int64_t n_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const int32_t t = static_cast<int32_t>(r / heads), h = static_cast<int32_t>(r % heads);
  const int32_t b = seq_of_tok[t];
  if (b < 0) return;  // layout status != 0
  const int32_t i = pos_in_seq[t];
  const int32_t L = lengths[b];
  const int64_t base = heads * attn_off[b] + static_cast<int64_t>(i * heads + h) * L;
  const T* xr = x + base;
  T* yr = y + base;
  if (L <= 32 * MAXE) {
    float v[MAXE];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int j = lane + 32 * k;
      v[k] = j < L ? ld_f(xr + j) : -INFINITY;
      m = fmaxf(m, v[k]);
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int j = lane + 32 * k;
      v[k] = j < L ? expf(v[k] - m) : 0.f;
      s += v[k];
    }
    const float inv = 1.0f / warp_sum(s);
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int j = lane + 32 * k;
      if (j < L) st_f(yr + j, v[k] * inv);
    }
  } else {
    float m = -INFINITY;
    for (int j = lane; j < L; j += 32) m = fmaxf(m, ld_f(xr + j));
    m = warp_max(m);
    float s = 0.f;
    for (int j = lane; j < L; j += 32) s += expf(ld_f(xr + j) - m);
    const float inv = 1.0f / warp_sum(s);
    for (int j = lane; j < L; j += 32) st_f(yr + j, expf(ld_f(xr + j) - m) * inv);
  }
}

// bf16 rows (L <= 512), vectorised: the row's 16-B-aligned interior is read and written as 8-element
// vectors (<= 2 per lane), the unaligned head and tail (<= 7 elements each) by single lanes -- rows start
// at arbitrary element offsets H*attn_off[b] + (i*H + h)*L_b.  exp2 with log2(e) folded into one FFMA.
__global__ void __launch_bounds__(256) ragged_softmax_bf16_vec_kernel(
    const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ lengths,
    const int64_t* __restrict__ attn_off, const int32_t* __restrict__ seq_of_tok,
    const int32_t* __restrict__ pos_in_seq, int32_t heads, int64_t n_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const int32_t t = static_cast<int32_t>(r / heads), h = static_cast<int32_t>(r % heads);
  const int32_t b = seq_of_tok[t];
  if (b < 0) return;  // layout status != 0
  const int32_t i = pos_in_seq[t];
  const int32_t L = lengths[b];
  const int64_t base = heads * attn_off[b] + static_cast<int64_t>(i * heads + h) * L;
  const int64_t a0 = (base + 7) & ~static_cast<int64_t>(7), a1 = (base + L) & ~static_cast<int64_t>(7);
  const int nvec = a1 > a0 ? static_cast<int>((a1 - a0) >> 3) : 0;
  const int head = nvec > 0 ? static_cast<int>(a0 - base) : L;  // scalar elements before the interior
  const int tail = nvec > 0 ? static_cast<int>(base + L - a1) : 0;
  constexpr float kLog2e = 1.4426950408889634f;
  float v[2][8];
  float sc = -INFINITY;  // this lane's scalar element (head: lanes 0..head-1, tail: lanes 8..8+tail-1;
                         // short rows without an interior: lanes 0..L-1, L < 32 + 8)
  int64_t sidx = -1;
  if (nvec == 0) {
    if (lane < L) sidx = base + lane;
  } else if (lane < head) {
    sidx = base + lane;
  } else if (lane >= 8 && lane < 8 + tail) {
    sidx = a1 + (lane - 8);
  }
  if (sidx >= 0) sc = __bfloat162float(x[sidx]);
  float m = sc;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nvec) {
      Vec<__nv_bfloat16>::load(x + a0 + 8 * vi, v[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, v[k][e]);
    }
  }
  m = warp_max(m) * kLog2e;
  float s = 0.f;
  if (sidx >= 0) {
    sc = exp2f(fmaf(sc, kLog2e, -m));
    s = sc;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k)
    if (lane + 32 * k < nvec) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[k][e] = exp2f(fmaf(v[k][e], kLog2e, -m));
        s += v[k][e];
      }
    }
  const float inv = 1.0f / warp_sum(s);
  if (sidx >= 0) y[sidx] = __float2bfloat16_rn(sc * inv);
#pragma unroll
  for (int k = 0; k < 2; ++k)
    if (lane + 32 * k < nvec) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[k][e] *= inv;
      Vec<__nv_bfloat16>::store(y + a0 + 8 * (lane + 32 * k), v[k]);
    }
}

// One warp per TOKEN: the H rows (i, h = 0..H-1) of token t share the layout lookups (seq_of_tok ->
// pos_in_seq / lengths / attn_off, a chain of dependent loads) and are contiguous in memory; the next
// row's loads are issued before the current row is reduced, so each warp keeps two rows in flight.
struct SmRow {
  int64_t a0, sidx;
  int nvec;
};
__device__ __forceinline__ SmRow sm_plan_row(int64_t base, int L, int lane) {
  SmRow p;
  p.a0 = (base + 7) & ~static_cast<int64_t>(7);
  const int64_t a1 = (base + L) & ~static_cast<int64_t>(7);
  p.nvec = a1 > p.a0 ? static_cast<int>((a1 - p.a0) >> 3) : 0;
  const int head = p.nvec > 0 ? static_cast<int>(p.a0 - base) : L;
  const int tail = p.nvec > 0 ? static_cast<int>(base + L - a1) : 0;
  p.sidx = -1;
  if (p.nvec == 0) {
    if (lane < L) p.sidx = base + lane;
  } else if (lane < head) {
    p.sidx = base + lane;
  } else if (lane >= 8 && lane < 8 + tail) {
    p.sidx = a1 + (lane - 8);
  }
  return p;
}
__device__ __forceinline__ void sm_load_row(const __nv_bfloat16* __restrict__ x, const SmRow& p, int lane, uint4 (&raw)[2],
                                            uint16_t& sraw) {
#pragma unroll
  for (int k = 0; k < 2; ++k)
    raw[k] = lane + 32 * k < p.nvec ? __ldg(reinterpret_cast<const uint4*>(x + p.a0) + lane + 32 * k)
                                    : make_uint4(0u, 0u, 0u, 0u);
  sraw = p.sidx >= 0 ? __ldg(reinterpret_cast<const unsigned short*>(x) + p.sidx) : static_cast<uint16_t>(0);
}

__global__ void __launch_bounds__(256) ragged_softmax_bf16_token_kernel(
    const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ lengths,
    const int64_t* __restrict__ attn_off, const int32_t* __restrict__ seq_of_tok,
    const int32_t* __restrict__ pos_in_seq, int32_t heads, int32_t n_tok) {
  const int lane = threadIdx.x & 31;
  const int32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= n_tok) return;
  const int32_t b = seq_of_tok[t];
  if (b < 0) return;  // layout status != 0
  const int32_t i = pos_in_seq[t];
  const int32_t L = lengths[b];
  const int64_t base0 = heads * attn_off[b] + static_cast<int64_t>(i) * heads * L;
  constexpr float kLog2e = 1.4426950408889634f;
  SmRow p = sm_plan_row(base0, L, lane);
  uint4 raw[2];
  uint16_t sraw;
  sm_load_row(x, p, lane, raw, sraw);
  for (int h = 0; h < heads; ++h) {
    SmRow pn = p;
    uint4 rawn[2] = {make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)};
    uint16_t srawn = 0;
    if (h + 1 < heads) {  // the next row's loads go out before this row is reduced
      pn = sm_plan_row(base0 + static_cast<int64_t>(h + 1) * L, L, lane);
      sm_load_row(x, pn, lane, rawn, srawn);
    }
    float v[2][8];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t w[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) v[k][2 * e] = __uint_as_float(w[e] << 16), v[k][2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
    float sc = p.sidx >= 0 ? __uint_as_float(static_cast<uint32_t>(sraw) << 16) : -INFINITY;
    float m = sc;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (lane + 32 * k < p.nvec) {
#pragma unroll
        for (int e = 0; e < 8; ++e) m = fmaxf(m, v[k][e]);
      }
    m = warp_max(m) * kLog2e;
    float s = 0.f;
    if (p.sidx >= 0) {
      sc = exp2f(fmaf(sc, kLog2e, -m));
      s = sc;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (lane + 32 * k < p.nvec) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          v[k][e] = exp2f(fmaf(v[k][e], kLog2e, -m));
          s += v[k][e];
        }
      }
    const float inv = 1.0f / warp_sum(s);
    if (p.sidx >= 0) y[p.sidx] = __float2bfloat16_rn(sc * inv);
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (lane + 32 * k < p.nvec) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] *= inv;
        Vec<__nv_bfloat16>::store(y + p.a0 + 8 * (lane + 32 * k), v[k]);
      }
    p = pn;
    raw[0] = rawn[0], raw[1] = rawn[1];
    sraw = srawn;
  }
}

}  // namespace

cudaError_t launch_layernorm(const void* x, const void* residual, const float* gamma, const float* beta, void* y,
                             int32_t rows, int32_t cols, float eps, cora_dtype_t dt, cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  if (dt == CORA_DT_BF16)
    return dispatch_layernorm<__nv_bfloat16>(x, residual, gamma, beta, y, rows, cols, eps, stream);
  return dispatch_layernorm<float>(x, residual, gamma, beta, y, rows, cols, eps, stream);
}

cudaError_t launch_ragged_softmax(const cora_layout_t& L, const void* x, void* y, cora_dtype_t dt,
                                  cudaStream_t stream) {
  const int64_t n_rows = static_cast<int64_t>(L.total_tokens) * L.heads;
  if (n_rows == 0) return cudaSuccess;
  const dim3 block(256), grid(static_cast<unsigned>((n_rows + 7) / 8));
  // vectorised bf16 path: rows of <= 512 keys (two 8-element vectors per lane + head / tail scalars);
  // x and y 16-B aligned so the interior vectors are aligned
  if (dt == CORA_DT_BF16 && L.max_len <= 512 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
    // a warp per token (its H rows pipelined) once there are enough tokens to fill the SMs with warps
    // (C4: 198 -> 158 us); a warp per row below that (C2-mnli: 12 vs 16 us)
    if (L.total_tokens >= 4096) {
      const dim3 tgrid(static_cast<unsigned>((L.total_tokens + 7) / 8));
      ragged_softmax_bf16_token_kernel<<<tgrid, block, 0, stream>>>(
          static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), L.lengths, L.attn_off,
          L.seq_of_tok, L.pos_in_seq, L.heads, L.total_tokens);
    } else {
      ragged_softmax_bf16_vec_kernel<<<grid, block, 0, stream>>>(
          static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), L.lengths, L.attn_off,
          L.seq_of_tok, L.pos_in_seq, L.heads, n_rows);
    }
    return cudaGetLastError();
  }
  if (dt == CORA_DT_BF16)
    ragged_softmax_kernel<__nv_bfloat16, 16><<<grid, block, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), L.lengths, L.attn_off, L.seq_of_tok,
        L.pos_in_seq, L.heads, n_rows);
  else
    ragged_softmax_kernel<float, 16><<<grid, block, 0, stream>>>(static_cast<const float*>(x),
                                                                 static_cast<float*>(y), L.lengths, L.attn_off,
                                                                 L.seq_of_tok, L.pos_in_seq, L.heads, n_rows);
  return cudaGetLastError();
}

}  // namespace cora
