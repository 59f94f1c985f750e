// Merged Linear on the 5th-gen tensor cores: a persistent, per-instance
// ("grouped") bf16 GEMM. tcgen05.mma accumulates in TMEM (two accumulator
// buffers, so one tile's epilogue overlaps the next tile's main loop), TMA
// streams operands through an mbarrier ring that runs continuously across
// tiles, and the fused epilogue y = act(acc + bias + residual) goes
// tcgen05.ld -> registers -> swizzled smem -> TMA bulk-tensor store.
//
// Replaces the reference's merged-Linear kernel `batch_matmul`
// (pkg/src/modelmerge/engine.py:215-235) for instance-packed shapes
// x (G, T, K) . W[g] -> y (G, T, N).
//
// D[i, j] = sum_k A[g, i, k] * B[g, j, k] over 128 x BN tiles, both operands
// K-major (G, rows, K). Orientation:
//   * normal  (SWAP=false): A = activations (i = token), B = weights (j = out
//     feature) — large T, tensor-bound merges.
//   * swapped (SWAP=true):  A = weights (i = out feature), B = activations
//     (j = token) — small T (batch-1 serving): the MMA's 128-row side is
//     filled by weight rows, so each weight byte is streamed once.
// Work units are (instance, A tile, B tile, K split). A grid of
// min(units, #SMs) CTAs walks them round-robin. K splits raise parallelism
// for low-tile-count shapes: each split writes an fp32 partial to an L2
// workspace, and the last arriver (per-tile semaphore) sums the partials in
// split order (deterministic), runs the epilogue and re-arms the semaphore.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer (one lane), warps 2..5 = epilogue (TMEM lane quarter = warp % 4).
#include "common.cuh"
#include "kernels.h"

namespace nf {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kGemmThreads = 192;
constexpr int kOutBlock = 64;  // features per 128-byte output block (bf16)
constexpr int kMaxSplits = 8;
#ifndef NF_GEMM_BUDGET_KB
#define NF_GEMM_BUDGET_KB 220  // smem for the operand ring + output staging
#endif
constexpr int64_t kCounterBytes = 64 * 1024;  // semaphores at the workspace head

#ifdef NF_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[4096];
NF_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define NF_TRACE(slot)                                                          \
  do {                                                                          \
    if (blockIdx.x == 0) g_gemm_trace[(slot)] = gtimer();                       \
  } while (0)
#else
#define NF_TRACE(slot) \
  do {                 \
  } while (0)
#endif

struct GemmParams {
  const float* bias;     // (G, features) fp32 or nullptr
  const void* residual;  // y-shaped bf16 or nullptr
  int64_t out_gstride;   // elements between instances of y
  int64_t out_ld;        // elements between tokens of y
  int rows_a, rows_b;    // valid rows of A / B
  int features;          // N (bias stride per instance)
  int tiles_a, tiles_b, groups;
  int splits, kb_total, kb_per_split, units;
  float* ws;             // split-K partials [tile][split][128][BN]
  unsigned* counters;    // [tile] arrival semaphores (zero between launches)
};

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOutBytes = kGemmBM * BN * 2;
  static constexpr int kStages =
      ((BN >= 256 ? 220 : NF_GEMM_BUDGET_KB) * 1024 - kOutBytes) / kStageBytes;
  static constexpr int kTmemCols = 2 * BN;  // two accumulator buffers
  static constexpr size_t kBytes =
      1024 + size_t(kStages) * kStageBytes + kOutBytes + 256;
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kTmemCols <= 512, "TMEM overflow");
};

// Byte offset of (token row t, feature f) inside the staged output tile made
// of 64-feature blocks, each `rows` x 128 B in the SWIZZLE_128B layout.
NF_DEVICE uint32_t stage_offset(int t, int f, int rows) {
  const int block = f >> 6;
  const int within = (f & 63) * 2;
  const int chunk = within >> 4;
  return uint32_t(block * rows * 128 + t * 128 + (((chunk ^ (t & 7)) << 4) | (within & 15)));
}

struct UnitCoord {
  int g, ta, tb, s, tile, kb0, kb1;
};

NF_DEVICE UnitCoord decode_unit(const GemmParams& p, int u, bool swap) {
  UnitCoord c;
  c.s = u % p.splits;
  c.tile = u / p.splits;
  // swapped: B (tokens) fastest; normal: A (token tiles) fastest, so CTAs
  // running concurrently share one weight tile in L2.
  if (swap) {
    c.tb = c.tile % p.tiles_b;
    c.ta = (c.tile / p.tiles_b) % p.tiles_a;
    c.g = c.tile / (p.tiles_b * p.tiles_a);
  } else {
    c.ta = c.tile % p.tiles_a;
    c.tb = (c.tile / p.tiles_a) % p.tiles_b;
    c.g = c.tile / (p.tiles_a * p.tiles_b);
  }
  c.kb0 = c.s * p.kb_per_split;
  c.kb1 = min(p.kb_total, c.kb0 + p.kb_per_split);
  return c;
}

template <int BN, bool SWAP, int ACT, bool HAS_RES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_grouped_gemm_tc(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_y, GemmParams p) {
  using C = GemmCfg<BN>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * C::kABytes;
  uint8_t* sOut = smem + kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + C::kOutBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_y);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) NF_TRACE(0);
  // Let the next kernel in the stream get scheduled as SMs free up; it waits
  // on griddepcontrol.wait for this grid's results before reading them.
  grid_dependents_launch();

  if (warp == 0) {
    if (lane == 0) {
      // Weights stream once: evict-first. Activations are re-read by sibling
      // CTAs: evict-last keeps them in L2.
      const uint64_t hint_a = SWAP ? kEvictFirst : kEvictLast;
      const uint64_t hint_b = SWAP ? kEvictLast : kEvictFirst;
      auto load_w = [&](int stage, const UnitCoord& c, int kb) {
        if (SWAP)
          tma_load_3d(sA + stage * C::kABytes, &map_a, &full[stage], kb * kGemmBK,
                      c.ta * kGemmBM, c.g, hint_a);
        else
          tma_load_3d(sB + stage * C::kBBytes, &map_b, &full[stage], kb * kGemmBK, c.tb * BN,
                      c.g, hint_b);
      };
      auto load_x = [&](int stage, const UnitCoord& c, int kb) {
        if (SWAP)
          tma_load_3d(sB + stage * C::kBBytes, &map_b, &full[stage], kb * kGemmBK, c.tb * BN,
                      c.g, hint_b);
        else
          tma_load_3d(sA + stage * C::kABytes, &map_a, &full[stage], kb * kGemmBK,
                      c.ta * kGemmBM, c.g, hint_a);
      };
      int it = 0;
      int u = blockIdx.x;
      int pre = 0;
      if (u < p.units) {
        // Under programmatic dependent launch the weights do not depend on
        // the previous kernel but the activations do: request the first
        // ring's worth of weight tiles before the dependency wait.
        const UnitCoord c = decode_unit(p, u, SWAP);
        pre = min(kStages, c.kb1 - c.kb0);
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], C::kStageBytes);
          load_w(i, c, c.kb0 + i);
        }
        grid_dependency_wait();
        for (int i = 0; i < pre; ++i) load_x(i, c, c.kb0 + i);
        it = pre;
      } else {
        grid_dependency_wait();
      }
      for (; u < p.units; u += gridDim.x) {
        const UnitCoord c = decode_unit(p, u, SWAP);
        for (int kb = c.kb0 + pre; kb < c.kb1; ++kb, ++it) {
          const int stage = it % kStages;
          mbar_wait(&empty[stage], ((it / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          load_w(stage, c, kb);
          load_x(stage, c, kb);
        }
        pre = 0;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16_f32(kGemmBM, BN);
    int it = 0, local = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++local) {
      const UnitCoord c = decode_unit(p, u, SWAP);
      const int acc = local & 1;
      mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
      for (int kb = c.kb0; kb < c.kb1; ++kb, ++it) {
        const int stage = it % kStages;
        mbar_wait(&full[stage], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kGemmBK / 16; ++kk)
            umma_f16_ss(d_tmem, make_sw128_kmajor_desc(a_base + kk * 32),
                        make_sw128_kmajor_desc(b_base + kk * 32), idesc,
                        (kb != c.kb0 || kk != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // accumulator row == TMEM lane
    const int etid = threadIdx.x - 64;    // 0..127
    const uint32_t stage_base = smem_u32(sOut);
    int local = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++local) {
      const UnitCoord c = decode_unit(p, u, SWAP);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      if (etid == 0) NF_TRACE(1 + 4 * local);
      const uint32_t t_row = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      const int m0 = c.ta * kGemmBM, n0 = c.tb * BN;
      float* part = nullptr;
      if (p.splits > 1) {
        // Publish this split's fp32 partial; the last arriver reduces.
        // Partials are stored column-major over TMEM lanes ([col][row]):
        // each warp store covers one contiguous 128-byte line.
        part = p.ws + (int64_t(c.tile) * p.splits) * kGemmBM * BN;
        float* mine = part + int64_t(c.s) * kGemmBM * BN + row;
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + uint32_t(cc), r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(mine + (cc + j) * kGemmBM, __uint_as_float(r[j]));
        }
        __threadfence();
        named_bar_sync(1, 128);
        if (etid == 0) NF_TRACE(3 + 4 * local);
        if (etid == 0) *last_flag = (atomicAdd(p.counters + c.tile, 1u) == unsigned(p.splits - 1));
        named_bar_sync(1, 128);
        if (!*last_flag) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          continue;
        }
        __threadfence();
      }
      const __nv_bfloat16* res =
          HAS_RES ? reinterpret_cast<const __nv_bfloat16*>(p.residual) +
                        int64_t(c.g) * p.out_gstride
                  : nullptr;
      const float* bias = p.bias ? p.bias + int64_t(c.g) * p.features : nullptr;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + uint32_t(cc), r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        }
        if (p.splits > 1) {
          // Deterministic reduction: splits summed in index order.
          float sum[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[j] = 0.f;
          for (int s2 = 0; s2 < p.splits; ++s2) {
            if (s2 == c.s) {
#pragma unroll
              for (int j = 0; j < 32; ++j) sum[j] += v[j];
            } else {
              const float* src = part + int64_t(s2) * kGemmBM * BN + row + cc * kGemmBM;
#pragma unroll
              for (int j = 0; j < 32; ++j) sum[j] += __ldcg(src + j * kGemmBM);
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = sum[j];
        }
        if (!SWAP) {
          // Thread = token row; 32 consecutive features n0+cc .. +31.
          const int tok = m0 + row;
          const int f0 = n0 + cc;
          if (bias) {
            if (f0 + 32 <= p.rows_b) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + f0 + j));
                v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (f0 + j < p.rows_b) v[j] += __ldg(bias + f0 + j);
            }
          }
          if (HAS_RES && tok < p.rows_a) {
            const __nv_bfloat16* rp = res + int64_t(tok) * p.out_ld + f0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (f0 + j < p.rows_b) v[j] += __bfloat162float(rp[j]);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_t<ACT>(v[j]);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(stage_base + stage_offset(row, cc + 8 * q, kGemmBM),
                         pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                         pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                         pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        } else {
          // Thread = feature row; 32 consecutive tokens. Neighbouring lanes
          // (features f, f^1) swap one value so each lane stores a packed
          // bf16 pair of adjacent features: 16 32-bit smem stores per chunk.
          const int feat = m0 + row;
          const float b = (bias && feat < p.rows_a) ? __ldg(bias + feat) : 0.0f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] += b;
            if (HAS_RES) {
              const int tok = n0 + cc + j;
              if (feat < p.rows_a && tok < p.rows_b)
                v[j] += __bfloat162float(res[int64_t(tok) * p.out_ld + feat]);
            }
            v[j] = act_t<ACT>(v[j]);
          }
          const bool odd = lane & 1;
          const int feven = row & ~1;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float send = odd ? v[j] : v[j + 1];
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const uint32_t packed = odd ? pack_bf16x2(recv, v[j + 1]) : pack_bf16x2(v[j], recv);
            const int t = cc + j + (odd ? 1 : 0);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(stage_base + stage_offset(t, feven, BN)),
                         "r"(packed)
                         : "memory");
          }
        }
      }
      // All TMEM reads of this buffer are done: hand it back to the MMA warp.
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (etid == 0) {
        if (!SWAP) {
#pragma unroll
          for (int b = 0; b < BN / kOutBlock; ++b)
            tma_store_3d(&map_y, sOut + b * kGemmBM * 128, n0 + b * kOutBlock, m0, c.g);
        } else {
#pragma unroll
          for (int b = 0; b < kGemmBM / kOutBlock; ++b)
            tma_store_3d(&map_y, sOut + b * BN * 128, m0 + b * kOutBlock, n0, c.g);
        }
        bulk_commit();
        if (p.splits > 1) p.counters[c.tile] = 0u;  // re-arm for the next launch
        bulk_wait_read0();                          // staging reusable
        NF_TRACE(4 + 4 * local);
      }
      named_bar_sync(1, 128);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) NF_TRACE(2);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  // Resolved once; the function pointer is immutable afterwards.
  static EncodeTiledFn fn = []() -> EncodeTiledFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D bf16 tensor (G, rows, inner) with inner contiguous -> tensor map with
// a (box_inner, box_rows, 1) SWIZZLE_128B box (box_inner * 2 == 128 bytes).
bool make_bf16_map(CUtensorMap* map, const void* base, int64_t G, int64_t rows, int64_t inner,
                   int box_inner, int box_rows, int64_t row_stride, int64_t g_stride) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  if (row_stride <= 0) row_stride = inner;
  if (g_stride <= 0) g_stride = rows * row_stride;
  if ((row_stride * 2) % 16 || (g_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(base) & 15))
    return false;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(G)};
  cuuint64_t strides[2] = {cuuint64_t(row_stride * 2), cuuint64_t(g_stride * 2)};
  cuuint32_t box[3] = {cuuint32_t(box_inner), cuuint32_t(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool SWAP, int ACT, bool HAS_RES>
static int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& my,
                     const GemmParams& p, int grid, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  auto kern = k_grouped_gemm_tc<BN, SWAP, ACT, HAS_RES>;
  static bool attr_done = false;  // idempotent attribute set; benign race
  if (!attr_done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kBytes));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled();
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, my, p);
  return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

template <int BN, bool SWAP, int ACT>
static int launch_tc_res(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& my,
                         const GemmParams& p, int grid, cudaStream_t stream) {
  if (p.residual) return launch_tc<BN, SWAP, ACT, true>(ma, mb, my, p, grid, stream);
  return launch_tc<BN, SWAP, ACT, false>(ma, mb, my, p, grid, stream);
}

template <int BN, bool SWAP>
static int launch_tc_act(int act, const CUtensorMap& ma, const CUtensorMap& mb,
                         const CUtensorMap& my, const GemmParams& p, int grid,
                         cudaStream_t stream) {
  switch (act) {
    case NF_ACT_RELU: return launch_tc_res<BN, SWAP, NF_ACT_RELU>(ma, mb, my, p, grid, stream);
    case NF_ACT_GELU: return launch_tc_res<BN, SWAP, NF_ACT_GELU>(ma, mb, my, p, grid, stream);
    case NF_ACT_TANH: return launch_tc_res<BN, SWAP, NF_ACT_TANH>(ma, mb, my, p, grid, stream);
    default: return launch_tc_res<BN, SWAP, NF_ACT_NONE>(ma, mb, my, p, grid, stream);
  }
}

static int pick_bn(int64_t T, int64_t N) {
  if (T <= 256) return T <= 64 ? 64 : (T <= 128 ? 128 : 256);
  return N >= 256 ? 256 : (N > 64 ? 128 : 64);
}

// Split-K factor: enough units to cover the SMs when the tile count is low,
// with at least 4 K blocks per split and a workspace that fits.
static int choose_splits(int64_t tiles, int kb_total, int bn, int64_t ws_bytes) {
  if (ws_bytes <= kCounterBytes || tiles >= 100 || tiles > kCounterBytes / 4) return 1;
  int s = int(kNumSMs / tiles);
  s = s < kMaxSplits ? s : kMaxSplits;
  // Each split adds a partial write + reduction to the critical path; only
  // worth it when every split still streams a long K range.
  s = s < kb_total / 64 ? s : kb_total / 64;
  while (s > 1 && tiles * s * int64_t(kGemmBM) * bn * 4 > ws_bytes - kCounterBytes) --s;
  return s < 1 ? 1 : s;
}

int64_t linear_workspace_bytes(int64_t G, int64_t T, int64_t K, int64_t N) {
  const int bn = pick_bn(T, N);
  const int64_t tiles_a = T <= 256 ? (N + kGemmBM - 1) / kGemmBM : (T + kGemmBM - 1) / kGemmBM;
  const int64_t tiles_b = T <= 256 ? (T + bn - 1) / bn : (N + bn - 1) / bn;
  const int64_t tiles = G * tiles_a * tiles_b;
  const int kb_total = int((K + kGemmBK - 1) / kGemmBK);
  const int s = choose_splits(tiles, kb_total, bn, INT64_MAX);
  if (s <= 1) return 0;
  return kCounterBytes + tiles * s * int64_t(kGemmBM) * bn * 4;
}

// Entry used by the C ABI. x rows at x + g*x_gs + t*x_ld (bf16); w (G, N, K)
// K-major bf16; bias fp32 (G, N) or null; y / residual rows at
// y + g*y_gs + t*y_ld (bf16). `ws` (zero-initialised once; the kernel
// restores its semaphores) enables split-K; null disables it.
int grouped_linear_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                      const float* bias, const void* residual, void* y, int64_t y_ld,
                      int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int out_dtype,
                      int act, void* ws, int64_t ws_bytes, cudaStream_t stream) {
  // TMA needs 16-byte aligned row strides for x, w and y.
  if (out_dtype != NF_BF16 || K % 8 != 0 || N % 8 != 0) return NF_ERR_UNSUPPORTED;
  if (G > 65535 || T > (int64_t(1) << 30) || N > (int64_t(1) << 30)) return NF_ERR_UNSUPPORTED;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255)) return NF_ERR_SHAPE;
  GemmParams p{};
  p.bias = bias;
  p.residual = residual;
  p.out_gstride = y_gs;
  p.out_ld = y_ld;
  p.features = int(N);
  p.groups = int(G);
  p.kb_total = int((K + kGemmBK - 1) / kGemmBK);
  const bool swap = T <= 256;
  const int bn = pick_bn(T, N);
  CUtensorMap ma, mb, my;
  if (swap) {
    if (!make_bf16_map(&ma, w, G, N, K, kGemmBK, kGemmBM, 0, 0) ||
        !make_bf16_map(&mb, x, G, T, K, kGemmBK, bn, x_ld, x_gs) ||
        !make_bf16_map(&my, y, G, T, N, kOutBlock, bn, y_ld, y_gs))
      return NF_ERR_UNSUPPORTED;
    p.rows_a = int(N);
    p.rows_b = int(T);
  } else {
    if (!make_bf16_map(&ma, x, G, T, K, kGemmBK, kGemmBM, x_ld, x_gs) ||
        !make_bf16_map(&mb, w, G, N, K, kGemmBK, bn, 0, 0) ||
        !make_bf16_map(&my, y, G, T, N, kOutBlock, kGemmBM, y_ld, y_gs))
      return NF_ERR_UNSUPPORTED;
    p.rows_a = int(T);
    p.rows_b = int(N);
  }
  p.tiles_a = (p.rows_a + kGemmBM - 1) / kGemmBM;
  p.tiles_b = (p.rows_b + bn - 1) / bn;
  const int64_t tiles = G * p.tiles_a * int64_t(p.tiles_b);
  p.splits = choose_splits(tiles, p.kb_total, bn, ws ? ws_bytes : 0);
  p.kb_per_split = (p.kb_total + p.splits - 1) / p.splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  if (tiles * p.splits > (int64_t(1) << 31) - 1) return NF_ERR_UNSUPPORTED;
  p.units = int(tiles * p.splits);
  p.counters = static_cast<unsigned*>(ws);
  p.ws = ws ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes) : nullptr;
  const int grid = p.units < kNumSMs ? p.units : kNumSMs;
#define NF_TC(BNV, SW) return launch_tc_act<BNV, SW>(act, ma, mb, my, p, grid, stream)
  if (swap) {
    if (bn == 64) NF_TC(64, true);
    if (bn == 128) NF_TC(128, true);
    NF_TC(256, true);
  }
  if (bn == 64) NF_TC(64, false);
  if (bn == 128) NF_TC(128, false);
  NF_TC(256, false);
#undef NF_TC
}

}  // namespace nf
