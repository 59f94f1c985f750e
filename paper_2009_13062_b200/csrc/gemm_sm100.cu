// Merged Linear on the 5th-gen tensor cores: a per-instance ("grouped")
// bf16 GEMM with tcgen05.mma accumulating in TMEM, operands staged by TMA
// (SWIZZLE_128B) through an mbarrier ring, and a fused bias/activation/
// residual epilogue (tcgen05.ld -> registers -> swizzled smem -> TMA store).
//
// Replaces the reference's merged-Linear kernel `batch_matmul`
// (pkg/src/modelmerge/engine.py:215-235) for instance-packed shapes
// x (G, T, K) . W[g] -> y (G, T, N).
//
// Computes D[i, j] = sum_k A[g, i, k] * B[g, j, k] for a 128 x BN tile where
// A and B are both K-major (G, rows, K) tensors. Two orientations:
//   * normal  (SWAP=false): A = activations (i = token), B = weights (j = out
//     feature). Used when T is large (tensor-bound merges).
//   * swapped (SWAP=true):  A = weights (i = out feature), B = activations
//     (j = token). Used at small T (batch-1 serving): the 128-row MMA M side
//     is filled by weight rows, so every weight byte is streamed from HBM
//     exactly once and the (tiny) activation tile is the one re-read, from L2.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer (one elected lane), warps 2..5 = epilogue (TMEM lane quarter =
// warp_id % 4). The epilogue stages the bf16 output tile in the (now idle)
// pipeline buffers as 64-feature x tokens blocks in the SWIZZLE_128B layout,
// then one thread writes each block with a TMA bulk-tensor store.
#include "common.cuh"
#include "kernels.h"

namespace nf {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kGemmThreads = 192;
constexpr int kOutBlock = 64;  // features per 128-byte output block (bf16)

#ifdef NF_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[4096];
NF_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define NF_TRACE(slot)                                                          \
  do {                                                                          \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)                  \
      g_gemm_trace[(slot)] = gtimer();                                          \
  } while (0)
#else
#define NF_TRACE(slot) \
  do {                 \
  } while (0)
#endif

struct GemmEpilogue {
  const float* bias;     // (G, features) fp32 or nullptr
  const void* residual;  // (G, T, N) bf16 or nullptr
  int64_t out_gstride;   // elements between instances (T * N)
  int64_t out_ld;        // elements between tokens (N)
  int rows_a;            // valid rows of operand A
  int rows_b;            // valid rows of operand B
  int features;          // N (bias stride per instance)
};

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr size_t kBytes = 1024 /*align slack*/ + size_t(kStages) * kStageBytes + 256;
  static_assert(kGemmBM * BN * 2 <= kStages * kStageBytes, "output staging must fit");
};

// Byte offset of (token row t, feature f) inside a staged output tile made of
// 64-feature blocks, each `rows` x 128 B with the SWIZZLE_128B chunk XOR.
NF_DEVICE uint32_t stage_offset(int t, int f, int rows) {
  const int block = f >> 6;
  const int within = (f & 63) * 2;
  const int chunk = within >> 4;
  return uint32_t(block * rows * 128 + t * 128 + (((chunk ^ (t & 7)) << 4) | (within & 15)));
}

template <int BN, bool SWAP, int ACT, bool HAS_RES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_grouped_gemm_tc(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_y, GemmEpilogue epi, int num_kb) {
  using S = GemmSmem<BN>;
  constexpr int kStages = S::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * S::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * S::kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kGemmBM;
  const int n0 = blockIdx.y * BN;
  const int g = blockIdx.z;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_y);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::kTmemCols);
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
      // Weights are streamed exactly once: evict-first. Activations are
      // re-read by sibling CTAs: evict-last keeps them in L2.
      const uint64_t hint_a = SWAP ? kEvictFirst : kEvictLast;
      const uint64_t hint_b = SWAP ? kEvictLast : kEvictFirst;
      // Under programmatic dependent launch the weight operand does not
      // depend on the previous kernel, but the activation operand does. So
      // the weight tiles of the first ring's worth of stages are requested
      // before the dependency wait (overlapping the previous kernel's tail),
      // and only the activation tiles wait for the producer grid.
      const int pre = num_kb < kStages ? num_kb : kStages;
      for (int kb = 0; kb < pre; ++kb) {
        mbar_arrive_expect_tx(&full[kb], S::kStageBytes);
        if (SWAP)
          tma_load_3d(sA + kb * S::kABytes, &map_a, &full[kb], kb * kGemmBK, m0, g, hint_a);
        else
          tma_load_3d(sB + kb * S::kBBytes, &map_b, &full[kb], kb * kGemmBK, n0, g, hint_b);
      }
      grid_dependency_wait();
      for (int kb = 0; kb < pre; ++kb) {
        if (SWAP)
          tma_load_3d(sB + kb * S::kBBytes, &map_b, &full[kb], kb * kGemmBK, n0, g, hint_b);
        else
          tma_load_3d(sA + kb * S::kABytes, &map_a, &full[kb], kb * kGemmBK, m0, g, hint_a);
      }
      for (int kb = pre; kb < num_kb; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        NF_TRACE(100 + kb);
        mbar_arrive_expect_tx(&full[s], S::kStageBytes);
        tma_load_3d(sA + s * S::kABytes, &map_a, &full[s], kb * kGemmBK, m0, g, hint_a);
        tma_load_3d(sB + s * S::kBBytes, &map_b, &full[s], kb * kGemmBK, n0, g, hint_b);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16_f32(kGemmBM, BN);
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (lane == 0) {
        NF_TRACE(1000 + kb);
        const uint32_t a_base = smem_u32(sA + s * S::kABytes);
        const uint32_t b_base = smem_u32(sB + s * S::kBBytes);
#pragma unroll
        for (int kk = 0; kk < kGemmBK / 16; ++kk) {
          // Advancing K by 16 bf16 = 32 bytes inside the 128-byte swizzle row.
          umma_f16_ss(tmem_base, make_sw128_kmajor_desc(a_base + kk * 32),
                      make_sw128_kmajor_desc(b_base + kk * 32), idesc, (kb | kk) != 0);
        }
        umma_commit(&empty[s]);  // frees the smem slot once these MMAs retire
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(tmem_full);
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // accumulator row == TMEM lane
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (threadIdx.x == 64) NF_TRACE(1);
    const uint32_t stage = smem_u32(smem);  // pipeline buffers are idle now
    const __nv_bfloat16* res =
        epi.residual
            ? reinterpret_cast<const __nv_bfloat16*>(epi.residual) + int64_t(g) * epi.out_gstride
            : nullptr;
    const float* bias = epi.bias ? epi.bias + int64_t(g) * epi.features : nullptr;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(c), r);
      tmem_ld_wait();
      if (threadIdx.x == 64) NF_TRACE(10 + c / 32);
      if (!SWAP) {
        // Thread = token row; 32 consecutive features n0+c .. n0+c+31.
        const int tok = m0 + row;
        const int f0 = n0 + c;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (bias) {
          if (f0 + 32 <= epi.rows_b) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + f0 + j));
              v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (f0 + j < epi.rows_b) v[j] += __ldg(bias + f0 + j);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = act_t<ACT>(v[j]);
        if (HAS_RES && tok < epi.rows_a) {
          const __nv_bfloat16* rp = res + int64_t(tok) * epi.out_ld + f0;
          if (f0 + 32 <= epi.rows_b) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = *reinterpret_cast<const uint4*>(rp + 8 * q);
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                v[8 * q + 2 * e] += f.x;
                v[8 * q + 2 * e + 1] += f.y;
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (f0 + j < epi.rows_b) v[j] += __bfloat162float(rp[j]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t addr = stage + stage_offset(row, c + 8 * q, kGemmBM);
          st_shared_v4(addr, pack_bf16x2(v[8 * q], v[8 * q + 1]),
                       pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                       pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                       pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        }
      } else {
        // Thread = feature row; 32 consecutive tokens n0+c .. n0+c+31. Lanes
        // hold consecutive features, so each smem row write is contiguous.
        const int feat = m0 + row;
        const float b = (bias && feat < epi.rows_a) ? __ldg(bias + feat) : 0.0f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float v = act_t<ACT>(__uint_as_float(r[j]) + b);
          const int tok = n0 + c + j;
          if (HAS_RES && feat < epi.rows_a && tok < epi.rows_b)
            v += __bfloat162float(res[int64_t(tok) * epi.out_ld + feat]);
          const __nv_bfloat16 h = __float2bfloat16_rn(v);
          st_shared_u16(stage + stage_offset(c + j, row, BN),
                        *reinterpret_cast<const uint16_t*>(&h));
        }
      }
    }
    if (threadIdx.x == 64) NF_TRACE(3);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 64) NF_TRACE(4);
    if (warp == 2 && lane == 0) {
      if (!SWAP) {
#pragma unroll
        for (int b = 0; b < BN / kOutBlock; ++b)
          tma_store_3d(&map_y, smem + b * kGemmBM * 128, n0 + b * kOutBlock, m0, g);
      } else {
#pragma unroll
        for (int b = 0; b < kGemmBM / kOutBlock; ++b)
          tma_store_3d(&map_y, smem + b * BN * 128, m0 + b * kOutBlock, n0, g);
      }
      bulk_commit();
      bulk_wait_read0();
      NF_TRACE(5);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) NF_TRACE(2);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S::kTmemCols);
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
                     const GemmEpilogue& epi, int rows_a, int rows_b, int G, int K,
                     cudaStream_t stream) {
  using S = GemmSmem<BN>;
  auto kern = k_grouped_gemm_tc<BN, SWAP, ACT, HAS_RES>;
  static bool attr_done = false;  // idempotent attribute set; benign race
  if (!attr_done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::kBytes));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((rows_a + kGemmBM - 1) / kGemmBM, (rows_b + BN - 1) / BN, G);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled();
  const int num_kb = (K + kGemmBK - 1) / kGemmBK;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, my, epi, num_kb);
  return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

template <int BN, bool SWAP, int ACT>
static int launch_tc_res(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& my,
                         const GemmEpilogue& epi, int rows_a, int rows_b, int G, int K,
                         cudaStream_t stream) {
  if (epi.residual)
    return launch_tc<BN, SWAP, ACT, true>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
  return launch_tc<BN, SWAP, ACT, false>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
}

template <int BN, bool SWAP>
static int launch_tc_act(int act, const CUtensorMap& ma, const CUtensorMap& mb,
                         const CUtensorMap& my, const GemmEpilogue& epi, int rows_a, int rows_b,
                         int G, int K, cudaStream_t stream) {
  switch (act) {
    case NF_ACT_RELU:
      return launch_tc_res<BN, SWAP, NF_ACT_RELU>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
    case NF_ACT_GELU:
      return launch_tc_res<BN, SWAP, NF_ACT_GELU>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
    case NF_ACT_TANH:
      return launch_tc_res<BN, SWAP, NF_ACT_TANH>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
    default:
      return launch_tc_res<BN, SWAP, NF_ACT_NONE>(ma, mb, my, epi, rows_a, rows_b, G, K, stream);
  }
}

// Entry used by the C ABI. x: (G, T, K) bf16; w: (G, N, K) bf16 K-major;
// bias fp32 (G, N) or null; y/residual: (G, T, N) bf16.
int grouped_linear_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                      const float* bias, const void* residual, void* y, int64_t y_ld,
                      int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int out_dtype,
                      int act, cudaStream_t stream) {
  // TMA needs 16-byte aligned row strides for x, w and y.
  if (out_dtype != NF_BF16 || K % 8 != 0 || N % 8 != 0) return NF_ERR_UNSUPPORTED;
  if (G > 65535 || T > (int64_t(1) << 30) || N > (int64_t(1) << 30)) return NF_ERR_UNSUPPORTED;
  GemmEpilogue epi;
  epi.bias = bias;
  epi.residual = residual;
  epi.out_gstride = y_gs;
  epi.out_ld = y_ld;
  epi.features = int(N);
  CUtensorMap ma, mb, my;
  if (T <= 256) {
    // Swapped: A = weights (rows N), B = activations (rows T).
    const int bn = T <= 64 ? 64 : (T <= 128 ? 128 : 256);
    if (!make_bf16_map(&ma, w, G, N, K, kGemmBK, kGemmBM, 0, 0) ||
        !make_bf16_map(&mb, x, G, T, K, kGemmBK, bn, x_ld, x_gs) ||
        !make_bf16_map(&my, y, G, T, N, kOutBlock, bn, y_ld, y_gs))
      return NF_ERR_UNSUPPORTED;
    epi.rows_a = int(N);
    epi.rows_b = int(T);
    if (bn == 64)
      return launch_tc_act<64, true>(act, ma, mb, my, epi, int(N), int(T), int(G), int(K), stream);
    if (bn == 128)
      return launch_tc_act<128, true>(act, ma, mb, my, epi, int(N), int(T), int(G), int(K),
                                      stream);
    return launch_tc_act<256, true>(act, ma, mb, my, epi, int(N), int(T), int(G), int(K), stream);
  }
  // Normal: A = activations (rows T), B = weights (rows N).
  const int bn = N >= 256 ? 256 : (N > 64 ? 128 : 64);
  if (!make_bf16_map(&ma, x, G, T, K, kGemmBK, kGemmBM, x_ld, x_gs) ||
      !make_bf16_map(&mb, w, G, N, K, kGemmBK, bn, 0, 0) ||
      !make_bf16_map(&my, y, G, T, N, kOutBlock, kGemmBM, y_ld, y_gs))
    return NF_ERR_UNSUPPORTED;
  epi.rows_a = int(T);
  epi.rows_b = int(N);
  if (bn == 64)
    return launch_tc_act<64, false>(act, ma, mb, my, epi, int(T), int(N), int(G), int(K), stream);
  if (bn == 128)
    return launch_tc_act<128, false>(act, ma, mb, my, epi, int(T), int(N), int(G), int(K), stream);
  return launch_tc_act<256, false>(act, ma, mb, my, epi, int(T), int(N), int(G), int(K), stream);
}

}  // namespace nf
