// the paper's second workload family -- variable-sized batched GEMM (vgemm) and
// triangular matrix multiplication (trmm) -- on the tcgen05 tensor cores.
//
//   vgemm: C_i = A_i B_i for a batch of problems with different (M_i, N_i, K_i) ("a batch of gemm
//          operations, each with different dimensions").  Storage is fully padded, as
//          in the paper's evaluation ("the CoRa implementations of these operators use fully padded
//          storage for all tensors"): A [batch, M_max, K_max], B [batch, K_max, N_max],
//          C [batch, M_max, N_max], row-major bf16; only the valid M_i x N_i block of each C_i is
//          computed and written, and only K_i of the reduction is visited (the raggedness saving).
//   trmm:  C = tril(L) B with L square [N, N] (only its lower triangle is referenced, BLAS semantics)
//          and B dense [N, N_c].  The reduction loop of row tile r is a vloop of length 128 (r + 1)
//          ("In trmm, the reduction loop is a vloop"): k-blocks above the diagonal
//          are never loaded, and the two k-blocks that straddle it have their upper triangle zeroed in
//          shared memory before the MMA (CoRa's operation splitting of the last iterations, PAPER.md:
//          827-831, is this peeled, masked block).  Work is ordered longest-first ("thread remapping
//          ... to schedule thread blocks with the most amount of work first").
//
// sm_100a design: one persistent kernel for both; one CTA per SM computes 128 x 256 tiles (cta_group::1,
// M128 N256 K16 tcgen05.mma, fp32 accumulators double-buffered in TMEM: 2 x 256 of the 512 columns).
//   warp 0     : TMA producer: A box 128 rows x 64 k (K-major, SWIZZLE_128B) + B as four 64 k x 64 n boxes
//                (MN-major, SWIZZLE_128B), 48 KB per stage, 4 stages
//   warp 1     : MMA issuer (lane 0) + diagonal masking of straddling A blocks (whole warp, trmm)
//   warps 2..5 : epilogue, one TMEM lane quadrant each: tcgen05.ld -> bf16 -> predicated 16-B global
//                stores (rows < M_i, columns < N_i: the padded tails of C are never written)
// The work list (problem, m0, n0, k-blocks), sorted by k-blocks descending, is built on the host and
// staged in the caller's workspace (vgemm); trmm's list is implicit (row tile r = R - 1 - u / NT).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "cora_internal.h"
#include "ptx.cuh"

namespace cora {
namespace {

constexpr int VM = 128;   // tile rows
constexpr int VN = 256;   // tile columns
constexpr int VK = 64;    // k per stage (one 128-B swizzle row of A)
constexpr int VSTAGES = 4;
constexpr int kVThreads = 192;
constexpr int kABytes = VM * VK * 2;        // 16 KB
constexpr int kBBoxBytes = VK * 64 * 2;     // 8 KB: 64 k-rows x 64 n-columns
constexpr int kBBytes = 4 * kBBoxBytes;     // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kOffBar = VSTAGES * kStageBytes;
constexpr int kNumBars = 2 * VSTAGES + 4;   // full, empty, tmem_full[2], tmem_empty[2]
constexpr int kSmemBytes = kOffBar + kNumBars * 8 + 16;

struct VUnit {
  int32_t p, m0, n0, kb;  // problem, first row, first column, k-blocks to visit
};

struct ProblemDims {
  int32_t m, n;  // valid rows / columns of this problem's C
};

// Zero the elements of the staged A block (rows m0.., k columns kb*64..) that lie above the diagonal
// (column > row): the SWIZZLE_128B layout puts 16-B chunk c of row i at chunk position c ^ (i & 7).
__device__ __forceinline__ void mask_upper_triangle(uint8_t* a_tile, int m0, int k0, uint32_t lane) {
  for (int i = static_cast<int>(lane); i < VM; i += 32) {
    const int row = m0 + i;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col0 = k0 + c * 8;
      if (col0 + 7 <= row) continue;  // chunk entirely on / below the diagonal
      uint4* chunk = reinterpret_cast<uint4*>(a_tile + i * 128 + ((c ^ (i & 7)) << 4));
      if (col0 > row) {
        *chunk = make_uint4(0u, 0u, 0u, 0u);
      } else {
        uint4 v = *chunk;
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ca = col0 + 2 * e;
          if (ca > row) w[e] &= 0u;
          else if (ca + 1 > row) w[e] &= 0x0000FFFFu;  // keep the low (even-column) element
        }
        *chunk = v;
      }
    }
  }
}

// TRMM: units are implicit, longest first: u -> (row tile R - 1 - u / NT, column tile u % NT).
template <bool TRMM>
__device__ __forceinline__ VUnit get_unit(const VUnit* __restrict__ units, int u, int r_tiles, int n_tiles_c,
                                          int k_blocks_total) {
  if (!TRMM) return units[u];
  const int r = r_tiles - 1 - u / n_tiles_c;
  const int kb = min(2 * r + 2, k_blocks_total);  // reduction k < 128 (r + 1)
  return VUnit{0, r * VM, (u % n_tiles_c) * VN, kb};
}

template <bool TRMM>
__global__ void __launch_bounds__(kVThreads, 1)
    vgemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const VUnit* __restrict__ units, const ProblemDims* __restrict__ dims, int32_t n_units,
                 int32_t m_max, int32_t k_max, __nv_bfloat16* __restrict__ c, int64_t ldc, int32_t r_tiles,
                 int32_t n_tiles_c, int32_t trmm_n, int32_t trmm_nc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* empty = full + VSTAGES;
  uint64_t* tmem_full = empty + VSTAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int k_blocks_total = (k_max + VK - 1) / VK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    for (int s = 0; s < VSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_ptr);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const VUnit w = get_unit<TRMM>(units, u, r_tiles, n_tiles_c, k_blocks_total);
        const int arow = w.p * m_max + w.m0;  // A viewed as [batch * M_max, K_max]
        const int brow0 = w.p * k_max;        // B viewed as [batch * K_max, N_max]
        for (int kb = 0; kb < w.kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          uint8_t* sa = smem + stage * kStageBytes;
          tma_load_2d(sa, &tm_a, &full[stage], kb * VK, arow);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            tma_load_2d(sa + kABytes + j * kBBoxBytes, &tm_b, &full[stage], w.n0 + 64 * j, brow0 + kb * VK);
          if (++stage == VSTAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // MMA issue (lane 0); the whole warp masks the diagonal-straddling A blocks of trmm
    constexpr uint32_t idesc = make_idesc_bf16(VM, VN, /*b_mn_major=*/true);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const VUnit w = get_unit<TRMM>(units, u, r_tiles, n_tiles_c, k_blocks_total);
      mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * VN;
      for (int kb = 0; kb < w.kb; ++kb) {
        mbar_wait(&full[stage], phase);
        uint8_t* sa = smem + stage * kStageBytes;
        if (TRMM && kb * VK + VK - 1 > w.m0) {  // the block reaches above the diagonal
          mask_upper_triangle(sa, w.m0, kb * VK, lane);
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
          __syncwarp();
        }
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sa);
          const uint32_t b_addr = a_addr + kABytes;
#pragma unroll
          for (int k = 0; k < VK / 16; ++k) {
            const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            // MN-major B: 16 k-rows (2 KB) per step; 64-column swizzle atoms 8 KB apart
            const uint64_t bd = make_sdesc_sw128(b_addr + k * 16 * 128, kBBoxBytes, 1024);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == VSTAGES) stage = 0, phase ^= 1;
      }
      if (lane == 0) umma_commit(&tmem_full[acc]);
      __syncwarp();
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
  } else {
    // epilogue: quadrant q = warp % 4 -> accumulator rows [32 q, 32 q + 32)
    const uint32_t q = warp & 3;
    const bool c_v8 = (reinterpret_cast<uintptr_t>(c) & 31u) == 0 && (ldc % 16) == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const VUnit w = get_unit<TRMM>(units, u, r_tiles, n_tiles_c, k_blocks_total);
      const int pm = TRMM ? trmm_n : dims[w.p].m, pn = TRMM ? trmm_nc : dims[w.p].n;
      const int row = w.m0 + static_cast<int>(q * 32 + lane);  // row of this thread inside problem p
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      __nv_bfloat16* crow = c + (static_cast<int64_t>(w.p) * m_max + row) * ldc;
#pragma unroll 1
      for (int cb = 0; cb < VN / 32; ++cb) {
        uint32_t r[32];
        CORA_TMEM_LD_32X32B_X32(tmem_base + ((q * 32) << 16) + acc * VN + cb * 32, r);
        tmem_ld_wait();
        if (w.kb == 0) {  // K_i == 0: no MMA ran for this unit, the accumulator holds stale data; C_i = 0
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = 0u;
        }
        const int col0 = w.n0 + cb * 32;
        if (row < pm && col0 < pn && c_v8 && col0 + 32 <= pn) {
          // 32-B stores: one full sector per lane
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const float* v = reinterpret_cast<const float*>(r) + g * 16;
            uint32_t wv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) wv[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
            st_global_v8(crow + col0 + g * 16, wv);
          }
        } else if (row < pm && col0 < pn) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int col = col0 + g * 8;
            const float* v = reinterpret_cast<const float*>(r) + g * 8;
            if (col + 8 <= pn) {
              *reinterpret_cast<uint4*>(crow + col) =
                  make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                             pack_bf16x2(v[6], v[7]));
            } else {
              for (int e = 0; e < 8 && col + e < pn; ++e) crow[col + e] = __float2bfloat16_rn(v[e]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

template <bool TRMM>
cudaError_t set_smem_attr() {
  static bool done[kMaxDevices] = {};
  const int dev = current_device();
  if (done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(vgemm_kernel<TRMM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

}  // namespace

// Serialised work list ("plan"): a 16-byte header {magic, batch, n_units, 0}, the units (16 B each: every
// 128 x 256 tile of every problem, longest reduction first, stable) and the problems' (M_i, N_i).  Built on
// the host into caller memory, copied verbatim into the device workspace by launch_vgemm.
constexpr int32_t kPlanMagic = 0x56474D31;  // "VGM1"
size_t vgemm_plan_bytes(int32_t batch, const int32_t* dims_host) {
  size_t units = 0;
  for (int i = 0; i < batch; ++i)
    units += static_cast<size_t>((dims_host[3 * i] + VM - 1) / VM) * ((dims_host[3 * i + 1] + VN - 1) / VN);
  return 16 + units * sizeof(VUnit) + static_cast<size_t>(batch) * sizeof(ProblemDims);
}

void vgemm_plan(int32_t batch, const int32_t* dims_host, void* plan_host) {
  std::vector<VUnit> units;
  for (int i = 0; i < batch; ++i) {
    const int m = dims_host[3 * i], n = dims_host[3 * i + 1], k = dims_host[3 * i + 2];
    const int kb = (k + VK - 1) / VK;
    for (int m0 = 0; m0 < m; m0 += VM)
      for (int n0 = 0; n0 < n; n0 += VN) units.push_back(VUnit{i, m0, n0, kb});
  }
  std::stable_sort(units.begin(), units.end(), [](const VUnit& x, const VUnit& y) { return x.kb > y.kb; });
  int32_t* h = static_cast<int32_t*>(plan_host);
  h[0] = kPlanMagic;
  h[1] = batch;
  h[2] = static_cast<int32_t>(units.size());
  h[3] = 0;
  uint8_t* p = static_cast<uint8_t*>(plan_host) + 16;
  if (!units.empty()) std::memcpy(p, units.data(), units.size() * sizeof(VUnit));
  ProblemDims* pd = reinterpret_cast<ProblemDims*>(p + units.size() * sizeof(VUnit));
  for (int i = 0; i < batch; ++i) pd[i] = ProblemDims{dims_host[3 * i], dims_host[3 * i + 1]};
}

bool vgemm_plan_valid(const void* plan_host, size_t ws_bytes) {
  const int32_t* h = static_cast<const int32_t*>(plan_host);
  if (h[0] != kPlanMagic || h[1] < 0 || h[2] < 0) return false;
  return 16 + static_cast<size_t>(h[2]) * sizeof(VUnit) + static_cast<size_t>(h[1]) * sizeof(ProblemDims) <= ws_bytes;
}

cudaError_t launch_vgemm(const void* plan_host, const void* a, const void* b, void* c, int32_t m_max, int32_t n_max,
                         int32_t k_max, void* ws, cudaStream_t stream) {
  const int32_t* h = static_cast<const int32_t*>(plan_host);
  const int32_t batch = h[1], n_units = h[2];
  if (n_units == 0) return cudaSuccess;
  // one asynchronous copy of the plan: from pinned caller memory it is a graph-capturable memcpy node
  const size_t bytes = 16 + static_cast<size_t>(n_units) * sizeof(VUnit) + static_cast<size_t>(batch) * sizeof(ProblemDims);
  cudaError_t e = cudaMemcpyAsync(ws, plan_host, bytes, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  uint8_t* w = static_cast<uint8_t*>(ws);
  const VUnit* d_units = reinterpret_cast<const VUnit*>(w + 16);
  const ProblemDims* d_dims = reinterpret_cast<const ProblemDims*>(w + 16 + static_cast<size_t>(n_units) * sizeof(VUnit));
  CUtensorMap ta, tb;
  if (!make_tmap_2d_bf16(&ta, a, k_max, static_cast<uint64_t>(batch) * m_max, static_cast<uint64_t>(k_max) * 2, VK,
                         VM, true) ||
      !make_tmap_2d_bf16(&tb, b, n_max, static_cast<uint64_t>(batch) * k_max, static_cast<uint64_t>(n_max) * 2, 64,
                         VK, true))
    return cudaErrorInvalidValue;
  if ((e = set_smem_attr<false>()) != cudaSuccess) return e;
  const int grid = std::min(static_cast<int>(n_units), device_sm_count());
  return launch_pdl(vgemm_kernel<false>, dim3(grid), dim3(kVThreads), kSmemBytes, stream, 1, ta, tb, d_units, d_dims,
                    static_cast<int>(n_units), m_max, k_max, static_cast<__nv_bfloat16*>(c), static_cast<int64_t>(n_max),
                    0, 0, 0, 0);
}

cudaError_t launch_trmm(const void* l, const void* b, void* c, int32_t n, int32_t n_cols, cudaStream_t stream) {
  if (n == 0 || n_cols == 0) return cudaSuccess;
  CUtensorMap ta, tb;
  if (!make_tmap_2d_bf16(&ta, l, n, n, static_cast<uint64_t>(n) * 2, VK, VM, true) ||
      !make_tmap_2d_bf16(&tb, b, n_cols, n, static_cast<uint64_t>(n_cols) * 2, 64, VK, true))
    return cudaErrorInvalidValue;
  cudaError_t e = set_smem_attr<true>();
  if (e != cudaSuccess) return e;
  const int r_tiles = (n + VM - 1) / VM, nt = (n_cols + VN - 1) / VN;
  const int n_units = r_tiles * nt;
  const int grid = std::min(n_units, device_sm_count());
  return launch_pdl(vgemm_kernel<true>, dim3(grid), dim3(kVThreads), kSmemBytes, stream, 1, ta, tb,
                    static_cast<const VUnit*>(nullptr), static_cast<const ProblemDims*>(nullptr), n_units, n, n,
                    static_cast<__nv_bfloat16*>(c), static_cast<int64_t>(n_cols), r_tiles, nt, n, n_cols);
}

}  // namespace cora
