// Merged attention: softmax(Q K^T * scale) V per (instance*batch, head) over
// a fused QKV activation (..., S, 3*H*dh). Batched over instances: the merged
// graph packs instances on the leading axis, so M instances x B sequences x H
// heads are just independent CTAs.
//
// The reference IR cannot express attention; its oracle is the
// reference contraction order + `softmax` (engine.py:313-319), see
// oracle/kernels.py::attention.
//
// tcgen05 path (bf16, dh == 64, S <= 128): one CTA per (sequence, head).
//   TMA loads Q, K, V tiles (128 x 64, SWIZZLE_128B) straight out of the
//   fused QKV rows; S = Q K^T accumulates in TMEM (128 x 128 fp32); each
//   thread owns one query row, does the max/exp2/sum in registers and writes
//   unnormalised P (bf16) to smem in the K-major SWIZZLE_128B layout; V's
//   TMA tile is consumed in place as an MN-major operand; O = P V
//   accumulates in TMEM (128 x 64) and is scaled by 1/rowsum in the
//   epilogue. Scores never touch HBM.
// SIMT path (any S, dh <= 128, f32 or bf16): one warp per query row with an
//   online softmax, for shapes / dtypes the tensor-core path does not take.
#include "common.cuh"
#include "kernels.h"

namespace nf {

bool make_bf16_map(CUtensorMap* map, const void* base, int64_t G, int64_t rows, int64_t inner,
                   int box_inner, int box_rows, int64_t row_stride, int64_t g_stride);

#ifdef NF_ATTN_TRACE
__device__ unsigned long long g_attn_trace[64];
#define NF_ATRACE(slot)                                                               \
  do {                                                                                \
    if (blockIdx.x == 0) {                                                            \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_attn_trace[(slot)] = t_;                                                      \
    }                                                                                 \
  } while (0)
#else
#define NF_ATRACE(slot) \
  do {                  \
  } while (0)
#endif

namespace {

constexpr int kAttnS = 128;   // max keys / queries per CTA
constexpr int kAttnD = 64;    // head dim on the tensor-core path
constexpr int kTileBytes = kAttnS * kAttnD * 2;  // 16 KB

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn_attn() {
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

// qkv viewed as 4-D (dh, 3H, S, Bt); box (64, 1, 128, 1) = one 128 x 128 B
// head tile in the K-major SWIZZLE_128B layout.
bool make_qkv_map(CUtensorMap* map, const void* qkv, int64_t Bt, int64_t S, int64_t H) {
  EncodeTiledFn fn = encode_fn_attn();
  if (!fn) return false;
  const int64_t D = H * kAttnD;
  cuuint64_t dims[4] = {cuuint64_t(kAttnD), cuuint64_t(3 * H), cuuint64_t(S), cuuint64_t(Bt)};
  cuuint64_t strides[3] = {cuuint64_t(kAttnD * 2), cuuint64_t(3 * D * 2),
                           cuuint64_t(S * 3 * D * 2)};
  cuuint32_t box[4] = {kAttnD, 1, kAttnS, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(qkv), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Byte offset of (row r, k) in a K-major SWIZZLE_128B operand whose K extent
// is split into 64-element (128 B) blocks of `rows` rows each.
__device__ __forceinline__ uint32_t kmajor_off(int r, int k, int rows) {
  const int blk = k >> 6;
  const int within = (k & 63) * 2;
  return uint32_t(blk * rows * 128 + r * 128 + ((((within >> 4) ^ (r & 7)) << 4) | (within & 15)));
}

__global__ void __launch_bounds__(128, 2)
    k_attention_tc(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ out,
                   int S, int H, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + kTileBytes;
  uint8_t* sP = sV + kTileBytes;           // 128 rows x 128 keys, 2 k-blocks (32 KB)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * kTileBytes);
  uint64_t* bar_load = bars;
  uint64_t* bar_s = bars + 1;
  uint64_t* bar_o = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int bt = blockIdx.x / H;
  const int h = blockIdx.x % H;

  if (tid == 0) {
    tma_prefetch_desc(&map_qkv);
    mbar_init(bar_load, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) NF_ATRACE(0);
  const uint32_t tmem_s = tmem;        // columns [0, 128): scores
  const uint32_t tmem_o = tmem + 128;  // columns [128, 192): context

  if (tid == 0) {
    grid_dependency_wait();
    mbar_arrive_expect_tx(bar_load, 3 * kTileBytes);
    tma_load_4d(sQ, &map_qkv, bar_load, 0, h, 0, bt, kEvictFirst);
    tma_load_4d(sK, &map_qkv, bar_load, 0, H + h, 0, bt, kEvictFirst);
    tma_load_4d(sV, &map_qkv, bar_load, 0, 2 * H + h, 0, bt, kEvictFirst);
  }
  grid_dependents_launch();
  mbar_wait(bar_load, 0);
  if (tid == 0) NF_ATRACE(1);

  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 128);
    const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
    for (int kk = 0; kk < kAttnD / 16; ++kk)
      umma_f16_ss(tmem_s, make_sw128_kmajor_desc(qa + kk * 32),
                  make_sw128_kmajor_desc(ka + kk * 32), idesc, kk != 0);
    umma_commit(bar_s);
  }

  // Softmax over this thread's query row (TMEM lane = tid).
  mbar_wait(bar_s, 0);
  tc_fence_after();
  if (tid == 0) NF_ATRACE(2);
  float mx = -INFINITY;
  uint32_t r[4][32];  // this query row's 128 scores
#pragma unroll
  for (int c = 0; c < 4; ++c)
    tmem_ld_32x32b_x32(tmem_s + (uint32_t(warp * 32) << 16) + uint32_t(c * 32), r[c]);
  tmem_ld_wait();
  if (tid == 0) NF_ATRACE(10);
  // Branch-free: out-of-range keys (S < 128) are masked to -inf by select,
  // so every exp is independent straight-line code the scheduler can overlap.
  {
    float m8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) m8[q] = -INFINITY;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float v = __uint_as_float(r[c][j]);
        m8[j & 7] = fmaxf(m8[j & 7], (c * 32 + j < S) ? v : -INFINITY);
      }
#pragma unroll
    for (int q = 0; q < 8; ++q) mx = fmaxf(mx, m8[q]);
  }
  if (tid == 0) NF_ATRACE(11);
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t prow = smem_u32(sP);
  const float mxs = mx * scale_log2;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float x0 = (c * 32 + j < S) ? fmaf(__uint_as_float(r[c][j]), scale_log2, -mxs)
                                        : -INFINITY;
      const float x1 = (c * 32 + j + 1 < S)
                           ? fmaf(__uint_as_float(r[c][j + 1]), scale_log2, -mxs)
                           : -INFINITY;
      // Probabilities are rounded to the bf16 values the PV MMA consumes and
      // the normaliser sums exactly those values.
      const uint32_t packed = pack_bf16x2(ex2_approx(x0), ex2_approx(x1));
      s4[(j >> 1) & 3] += __uint_as_float(packed << 16) + __uint_as_float(packed & 0xffff0000u);
      pk[j >> 1] = packed;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_shared_v4(prow + kmajor_off(tid, c * 32 + q * 8, 128), pk[4 * q], pk[4 * q + 1],
                   pk[4 * q + 2], pk[4 * q + 3]);
  }
  const float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  if (tid == 0) NF_ATRACE(12);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) NF_ATRACE(3);

  if (tid == 0) {
    tc_fence_after();
    // B = V straight from its TMA tile: keys (the K dim) are 128-byte rows of
    // 64 dh values, i.e. the MN-major SWIZZLE_128B layout; 16 keys per MMA.
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 64, 0, 1);
    const uint32_t pa = smem_u32(sP), va = smem_u32(sV);
#pragma unroll
    for (int kk = 0; kk < kAttnS / 16; ++kk) {
      const int blk = kk >> 2, sub = kk & 3;
      umma_f16_ss(tmem_o, make_sw128_kmajor_desc(pa + blk * 128 * 128 + sub * 32),
                  make_sw128_mnmajor_desc(va + kk * 16 * 128, 8192, 1024), idesc, kk != 0);
    }
    umma_commit(bar_o);
  }
  mbar_wait(bar_o, 0);
  tc_fence_after();
  if (tid == 0) NF_ATRACE(4);
  {
    uint32_t o[2][32];
    tmem_ld_32x32b_x32(tmem_o + (uint32_t(warp * 32) << 16), o[0]);
    tmem_ld_32x32b_x32(tmem_o + (uint32_t(warp * 32) << 16) + 32, o[1]);
    tmem_ld_wait();
    if (tid < S) {
      const float inv = 1.0f / sum;
      const int64_t D = int64_t(H) * kAttnD;
      __nv_bfloat16* dst = out + (int64_t(bt) * S + tid) * D + int64_t(h) * kAttnD;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(o[c][8 * q]) * inv, __uint_as_float(o[c][8 * q + 1]) * inv);
          u.y = pack_bf16x2(__uint_as_float(o[c][8 * q + 2]) * inv, __uint_as_float(o[c][8 * q + 3]) * inv);
          u.z = pack_bf16x2(__uint_as_float(o[c][8 * q + 4]) * inv, __uint_as_float(o[c][8 * q + 5]) * inv);
          u.w = pack_bf16x2(__uint_as_float(o[c][8 * q + 6]) * inv, __uint_as_float(o[c][8 * q + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c * 32 + q * 8) = u;
        }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) NF_ATRACE(5);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

constexpr size_t kAttnSmem = 1024 + 5 * kTileBytes + 64;

// (An 8-warp persistent variant measured 3% slower on BERT-base N=32 B=8:
// two 4-warp CTAs per SM already overlap their softmax phases.)

// Persistent variant for many (sequence, head) units: each CTA walks units
// u = blockIdx.x, += gridDim.x over a double buffer of Q/K/V tiles; a
// buffer is refilled with the unit two ahead as soon as its unit's PV MMA
// retired; P (bf16 128 x 128) reuses the current unit's Q|K slots once
// S = Q K^T retired.
// 2 x 48 KB of tiles + barriers -> two CTAs per SM (256 TMEM cols each).
constexpr size_t kAttnPSmem = 1024 + 6 * kTileBytes + 128;

__global__ void __launch_bounds__(128, 2)
    k_attention_tc_persistent(const __grid_constant__ CUtensorMap map_qkv,
                              __nv_bfloat16* __restrict__ out, int S, int H, int units,
                              float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTileBytes);
  uint64_t* bar_load = bars;  // [2]
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_o = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) {
    tma_prefetch_desc(&map_qkv);
    mbar_init(&bar_load[0], 1);
    mbar_init(&bar_load[1], 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_s = tmem, tmem_o = tmem + 128;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;

  auto issue = [&](int u, int buf) {
    uint8_t* b = smem + buf * 3 * kTileBytes;
    const int bt = u / H, h = u % H;
    mbar_arrive_expect_tx(&bar_load[buf], 3 * kTileBytes);
    tma_load_4d(b, &map_qkv, &bar_load[buf], 0, h, 0, bt, kEvictFirst);
    tma_load_4d(b + kTileBytes, &map_qkv, &bar_load[buf], 0, H + h, 0, bt, kEvictFirst);
    tma_load_4d(b + 2 * kTileBytes, &map_qkv, &bar_load[buf], 0, 2 * H + h, 0, bt, kEvictFirst);
  };
  if (tid == 0) {
    grid_dependency_wait();
    if (int(blockIdx.x) < units) issue(blockIdx.x, 0);
    if (int(blockIdx.x + gridDim.x) < units) issue(blockIdx.x + gridDim.x, 1);
  }
  grid_dependents_launch();

  int i = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
    const int buf = i & 1;
    uint8_t* sQ = smem + buf * 3 * kTileBytes;
    uint8_t* sK = sQ + kTileBytes;
    uint8_t* sV = sK + kTileBytes;
    uint8_t* sP = sQ;  // Q|K, free once S is in TMEM
    const int bt = u / H, h = u % H;
    mbar_wait(&bar_load[buf], uint32_t(i >> 1) & 1u);
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = make_idesc_bf16_f32(128, 128);
      const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
      for (int kk = 0; kk < kAttnD / 16; ++kk)
        umma_f16_ss(tmem_s, make_sw128_kmajor_desc(qa + kk * 32),
                    make_sw128_kmajor_desc(ka + kk * 32), idesc, kk != 0);
      umma_commit(bar_s);
    }
    mbar_wait(bar_s, uint32_t(i) & 1u);
    tc_fence_after();
    uint32_t r[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem_s + lane_off + uint32_t(c * 32), r[c]);
    tmem_ld_wait();
    float mx = -INFINITY;
    {
      float m8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) m8[q] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j)
          m8[j & 7] = fmaxf(m8[j & 7], (c * 32 + j < S) ? __uint_as_float(r[c][j]) : -INFINITY);
#pragma unroll
      for (int q = 0; q < 8; ++q) mx = fmaxf(mx, m8[q]);
    }
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
    const uint32_t prow = smem_u32(sP);
    const float mxs = mx * scale_log2;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float x0 = (c * 32 + j < S) ? fmaf(__uint_as_float(r[c][j]), scale_log2, -mxs)
                                          : -INFINITY;
        const float x1 = (c * 32 + j + 1 < S)
                             ? fmaf(__uint_as_float(r[c][j + 1]), scale_log2, -mxs)
                             : -INFINITY;
        const uint32_t packed = pack_bf16x2(ex2_approx(x0), ex2_approx(x1));
        s4[(j >> 1) & 3] += __uint_as_float(packed << 16) + __uint_as_float(packed & 0xffff0000u);
        pk[j >> 1] = packed;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_shared_v4(prow + kmajor_off(tid, c * 32 + q * 8, 128), pk[4 * q], pk[4 * q + 1],
                     pk[4 * q + 2], pk[4 * q + 3]);
    }
    const float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();  // P written; S fully read
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = make_idesc_bf16_f32(128, 64, 0, 1);
      const uint32_t pa = smem_u32(sP), va = smem_u32(sV);
#pragma unroll
      for (int kk = 0; kk < kAttnS / 16; ++kk) {
        const int blk = kk >> 2, sub = kk & 3;
        umma_f16_ss(tmem_o, make_sw128_kmajor_desc(pa + blk * 128 * 128 + sub * 32),
                    make_sw128_mnmajor_desc(va + kk * 16 * 128, 8192, 1024), idesc, kk != 0);
      }
      umma_commit(bar_o);
    }
    mbar_wait(bar_o, uint32_t(i) & 1u);
    // this unit's Q | K (P) and V are consumed: the unit after next streams
    // into them during this epilogue and the next unit's work (two units'
    // tiles in flight instead of one)
    if (tid == 0 && u + 2 * int(gridDim.x) < units) issue(u + 2 * gridDim.x, buf);
    tc_fence_after();
    {
      uint32_t o[2][32];
      tmem_ld_32x32b_x32(tmem_o + lane_off, o[0]);
      tmem_ld_32x32b_x32(tmem_o + lane_off + 32, o[1]);
      tmem_ld_wait();
      if (tid < S) {
        const float inv = 1.0f / sum;
        const int64_t D = int64_t(H) * kAttnD;
        __nv_bfloat16* dst = out + (int64_t(bt) * S + tid) * D + int64_t(h) * kAttnD;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(o[c][8 * q]) * inv, __uint_as_float(o[c][8 * q + 1]) * inv);
            w.y = pack_bf16x2(__uint_as_float(o[c][8 * q + 2]) * inv, __uint_as_float(o[c][8 * q + 3]) * inv);
            w.z = pack_bf16x2(__uint_as_float(o[c][8 * q + 4]) * inv, __uint_as_float(o[c][8 * q + 5]) * inv);
            w.w = pack_bf16x2(__uint_as_float(o[c][8 * q + 6]) * inv, __uint_as_float(o[c][8 * q + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + q * 8) = w;
          }
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM S/O and this buffer's smem are free for the next unit
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------
// SIMT fallback: one warp per (sequence, head, query), online softmax.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_attention_simt(const T* __restrict__ qkv, T* __restrict__ out, int64_t Bt,
                                 int S, int H, int dh, float scale) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t D = int64_t(H) * dh;
  const int64_t units = Bt * H * S;
  for (int64_t u = w; u < units; u += nw) {
    const int i = int(u % S);
    const int h = int((u / S) % H);
    const int64_t b = u / (int64_t(S) * H);
    const T* base = qkv + b * S * 3 * D;
    const T* q = base + int64_t(i) * 3 * D + int64_t(h) * dh;
    float qv[4], acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = lane + 32 * e;
      qv[e] = d < dh ? to_f32(q[d]) : 0.f;
      acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < S; ++j) {
      const T* k = base + int64_t(j) * 3 * D + D + int64_t(h) * dh;
      const T* v = k + D;
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = lane + 32 * e;
        if (d < dh) dot += qv[e] * to_f32(k[d]);
      }
      dot = warp_sum(dot) * scale;
      const float mn = fmaxf(m, dot);
      const float corr = expf(m - mn);
      const float p = expf(dot - mn);
      l = l * corr + p;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = lane + 32 * e;
        acc[e] = acc[e] * corr + (d < dh ? p * to_f32(v[d]) : 0.f);
      }
      m = mn;
    }
    T* o = out + (b * S + i) * D + int64_t(h) * dh;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = lane + 32 * e;
      if (d < dh) o[d] = from_f32<T>(acc[e] / l);
    }
  }
}

// XLNet relative attention (attn_type "bi", no segments / mask): warp per
// (sequence, head, query i), online softmax over keys j of
//   score = ((q + r_w_bias) . k_j + (q + r_r_bias) . kr_{S - i + j}) * scale
// where kr = the projected positional keys (2S rows per sequence) and the
// index S - i + j is transformers' rel_shift_bnij. Biases are per instance:
// sequence b belongs to instance b / seqs_per_bias.
template <typename T>
__global__ void k_rel_attention_simt(const T* __restrict__ qkv, const T* __restrict__ r,
                                     const float* __restrict__ rwb, const float* __restrict__ rrb,
                                     T* __restrict__ out, int64_t Bt, int S, int H, int dh,
                                     int seqs_per_bias, int seqs_per_r, float scale) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t D = int64_t(H) * dh;
  const int64_t units = Bt * H * S;
  for (int64_t u = w; u < units; u += nw) {
    const int i = int(u % S);
    const int h = int((u / S) % H);
    const int64_t b = u / (int64_t(S) * H);
    const int64_t inst = b / seqs_per_bias;
    const T* base = qkv + b * S * 3 * D;
    const T* rb = r + (b / seqs_per_r) * 2 * S * D + int64_t(h) * dh;
    const T* q = base + int64_t(i) * 3 * D + int64_t(h) * dh;
    const float* bw = rwb + (inst * H + h) * dh;
    const float* br = rrb + (inst * H + h) * dh;
    float qw[4], qr[4], acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = lane + 32 * e;
      const float qv = d < dh ? to_f32(q[d]) : 0.f;
      qw[e] = d < dh ? qv + bw[d] : 0.f;
      qr[e] = d < dh ? qv + br[d] : 0.f;
      acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < S; ++j) {
      const T* k = base + int64_t(j) * 3 * D + D + int64_t(h) * dh;
      const T* v = k + D;
      const T* kr = rb + int64_t(S - i + j) * D;
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = lane + 32 * e;
        if (d < dh) dot += qw[e] * to_f32(k[d]) + qr[e] * to_f32(kr[d]);
      }
      dot = warp_sum(dot) * scale;
      const float mn = fmaxf(m, dot);
      const float corr = expf(m - mn);
      const float p = expf(dot - mn);
      l = l * corr + p;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = lane + 32 * e;
        acc[e] = acc[e] * corr + (d < dh ? p * to_f32(v[d]) : 0.f);
      }
      m = mn;
    }
    T* o = out + (b * S + i) * D + int64_t(h) * dh;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = lane + 32 * e;
      if (d < dh) o[d] = from_f32<T>(acc[e] / l);
    }
  }
}

// ---------------------------------------------------------------------------
// XLNet relative attention on the tensor cores (bf16, dh == 64, S == 128).
// One CTA per (sequence, head), 128 threads, thread = query row i:
//   AC  = Q K^T                      tcgen05 -> TMEM cols [0,128) -> registers
//   raw = Q KR^T (KR = 2S = 256 rows) tcgen05 -> TMEM cols [0,256)
//   score[i][j] = (AC + bw[j] + raw[i][S-i+j] + cr[S-i+j]) * scale
// where bw[j] = r_w_bias . k_j and cr[p] = r_r_bias . kr_p (fp32 dot
// products, so (q + bias) is never rounded to bf16). The rel-shift
// raw[i][S-i+j] differs per TMEM lane; each warp stages a 32 x 64 window of
// raw through a padded smem buffer (pitch 68 words: 128-bit stores and the
// skewed scalar reads are both bank-conflict free) and reads it back
// diagonally. P overwrites KR's smem once the raw MMA retired; O = P V
// reuses TMEM cols [0,64). 256 TMEM cols + ~86 KB smem -> 2 CTAs per SM.
// ---------------------------------------------------------------------------
constexpr int kRelPitch = 68;                           // words per staged row

// positional keys r viewed as 4-D (dh, H, 2S, Bt); box (64, 1, 128, 1).
bool make_r_map(CUtensorMap* map, const void* r, int64_t Bt, int64_t S, int64_t H) {
  EncodeTiledFn fn = encode_fn_attn();
  if (!fn) return false;
  const int64_t D = H * kAttnD;
  cuuint64_t dims[4] = {cuuint64_t(kAttnD), cuuint64_t(H), cuuint64_t(2 * S), cuuint64_t(Bt)};
  cuuint64_t strides[3] = {cuuint64_t(kAttnD * 2), cuuint64_t(D * 2), cuuint64_t(2 * S * D * 2)};
  cuuint32_t box[4] = {kAttnD, 1, kAttnS, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(r), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 dot of a (64-element, fp32) bias vector with row `row` of a K-major
// SWIZZLE_128B bf16 tile.
__device__ __forceinline__ float bias_dot_row(const uint8_t* tile, int row, const float* bias) {
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 u = *reinterpret_cast<const uint4*>(tile + row * 128 + ((c ^ (row & 7)) << 4));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc = fmaf(__uint_as_float(w[e] << 16), bias[c * 8 + 2 * e], acc);
      acc = fmaf(__uint_as_float(w[e] & 0xffff0000u), bias[c * 8 + 2 * e + 1], acc);
    }
  }
  return acc;
}

// One CTA per (sequence, head), two CTAs per SM, 8 warps: warps w
// and w + 4 share TMEM lane quarter w & 3 and split the 128 key columns in
// halves, so each thread holds 64 scores (no spills), the rel-shift windows
// of the two halves run in parallel, and the row max / sum combine through
// shared memory. Shift windows: warps 0-3 in the Q|K|pad region, warps 4-7
// in KR + its 4 KB tail (both free once the raw MMA retired).
constexpr size_t kRel8Smem = 1024 + 2 * kTileBytes + 4096 + kTileBytes + 2 * kTileBytes + 4096 +
                             (128 + 256 + 128 + 4 * 128) * 4 + 64;

__global__ void __launch_bounds__(256, 2)
    k_rel_attention_tc8(const __grid_constant__ CUtensorMap map_qkv,
                        const __grid_constant__ CUtensorMap map_r, const float* __restrict__ rwb,
                        const float* __restrict__ rrb, __nv_bfloat16* __restrict__ out, int H,
                        int seqs_per_bias, int seqs_per_r, float scale_log2) {
  constexpr int S = kAttnS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + kTileBytes + 4096;
  uint8_t* sKR = sV + kTileBytes;  // 256 rows; later P (128 x 128) + shift windows
  float* sBw = reinterpret_cast<float*>(sKR + 2 * kTileBytes + 4096);
  float* sCr = sBw + 128;
  float* sRb = sCr + 256;   // r_w_bias | r_r_bias
  float* sMax = sRb + 128;  // [2][128]
  float* sSum = sMax + 256; // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSum + 256);
  uint64_t* bar_load = bars;
  uint64_t* bar_s = bars + 1;
  uint64_t* bar_bd = bars + 2;
  uint64_t* bar_o = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int quarter = warp & 3;
  const int half = warp >> 2;  // key columns [64*half, 64*half + 64)
  const int i_row = quarter * 32 + lane;
  const int bt = blockIdx.x / H;
  const int h = blockIdx.x % H;
  const int inst = bt / seqs_per_bias;

  if (tid == 0) {
    tma_prefetch_desc(&map_qkv);
    tma_prefetch_desc(&map_r);
    mbar_init(bar_load, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_bd, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);

  if (tid == 0) {
    grid_dependency_wait();
    mbar_arrive_expect_tx(bar_load, 5 * kTileBytes);
    tma_load_4d(sQ, &map_qkv, bar_load, 0, h, 0, bt, kEvictFirst);
    tma_load_4d(sK, &map_qkv, bar_load, 0, H + h, 0, bt, kEvictFirst);
    tma_load_4d(sV, &map_qkv, bar_load, 0, 2 * H + h, 0, bt, kEvictFirst);
    tma_load_4d(sKR, &map_r, bar_load, 0, h, 0, bt / seqs_per_r, kEvictLast);
    tma_load_4d(sKR + kTileBytes, &map_r, bar_load, 0, h, S, bt / seqs_per_r, kEvictLast);
  }
  grid_dependents_launch();
  if (tid < 64) {
    const float* src = tid < 32 ? rwb : rrb;
    const int d = (tid & 31) * 2;
    const float2 v = *reinterpret_cast<const float2*>(src + (int64_t(inst) * H + h) * kAttnD + d);
    sRb[(tid < 32 ? 0 : 64) + d] = v.x;
    sRb[(tid < 32 ? 0 : 64) + d + 1] = v.y;
  }
  mbar_wait(bar_load, 0);

  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 128);
    const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
    for (int kk = 0; kk < kAttnD / 16; ++kk)
      umma_f16_ss(tmem, make_sw128_kmajor_desc(qa + kk * 32),
                  make_sw128_kmajor_desc(ka + kk * 32), idesc, kk != 0);
    umma_commit(bar_s);
  }
  __syncthreads();  // bias vectors in smem
  // bias . key rows (fp32): bw for the 128 keys, cr for the 256 positions
  if (tid < 128) {
    sBw[tid] = bias_dot_row(sK, tid, sRb);
    sCr[tid] = bias_dot_row(sKR, tid, sRb + 64);
  } else {
    sCr[tid] = bias_dot_row(sKR, tid, sRb + 64);
  }

  mbar_wait(bar_s, 0);
  tc_fence_after();
  uint32_t r[2][32];  // AC of this row, key columns 64*half ..
#pragma unroll
  for (int c = 0; c < 2; ++c) tmem_ld_32x32b_x32(lane_base + uint32_t(64 * half + c * 32), r[c]);
  tmem_ld_wait();
  tc_fence_before();
  __syncthreads();  // AC consumed; bias vectors visible

  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 256);
    const uint32_t qa = smem_u32(sQ), ra = smem_u32(sKR);
#pragma unroll
    for (int kk = 0; kk < kAttnD / 16; ++kk)
      umma_f16_ss(tmem, make_sw128_kmajor_desc(qa + kk * 32),
                  make_sw128_kmajor_desc(ra + kk * 32), idesc, kk != 0);
    umma_commit(bar_bd);
  }
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      r[c][j] = __float_as_uint(__uint_as_float(r[c][j]) + sBw[64 * half + c * 32 + j]);

  mbar_wait(bar_bd, 0);
  tc_fence_after();
  uint8_t* wbuf = (half == 0 ? sQ : sKR) + quarter * 32 * kRelPitch * 4;
  const uint32_t stage_w = smem_u32(wbuf);
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int c = 2 * half + cc;             // global 32-key chunk
    const int p0 = 97 - 32 * quarter + 32 * c;  // window start for lane 31, jj 0
    const int base = p0 < 192 ? p0 : 192;
    const int shift = 31 - lane + (p0 - base);
    __syncwarp();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      uint32_t wv[32];
      tmem_ld_32x32b_x32(lane_base + uint32_t(base + 32 * hh), wv);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_shared_v4(stage_w + uint32_t((lane * kRelPitch + 32 * hh + 4 * q) * 4), wv[4 * q],
                     wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
    }
    __syncwarp();
    const float* row = reinterpret_cast<const float*>(wbuf) + lane * kRelPitch + shift;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int p = S - i_row + c * 32 + jj;
      r[cc][jj] = __float_as_uint(__uint_as_float(r[cc][jj]) + row[jj] + sCr[p]);
    }
  }
  float mx = -INFINITY;
  {
    float m8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) m8[q] = -INFINITY;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int j = 0; j < 32; ++j) m8[j & 7] = fmaxf(m8[j & 7], __uint_as_float(r[c][j]));
#pragma unroll
    for (int q = 0; q < 8; ++q) mx = fmaxf(mx, m8[q]);
  }
  sMax[half * 128 + i_row] = mx;
  tc_fence_before();
  __syncthreads();  // both halves' maxima; every raw TMEM / window read done
  mx = fmaxf(sMax[i_row], sMax[128 + i_row]);
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t prow = smem_u32(sKR);  // P overwrites KR (and the half-1 windows)
  const float mxs = mx * scale_log2;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int c = 2 * half + cc;
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float x0 = fmaf(__uint_as_float(r[cc][j]), scale_log2, -mxs);
      const float x1 = fmaf(__uint_as_float(r[cc][j + 1]), scale_log2, -mxs);
      const uint32_t packed = pack_bf16x2(ex2_approx(x0), ex2_approx(x1));
      s4[(j >> 1) & 3] += __uint_as_float(packed << 16) + __uint_as_float(packed & 0xffff0000u);
      pk[j >> 1] = packed;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_shared_v4(prow + kmajor_off(i_row, c * 32 + q * 8, 128), pk[4 * q], pk[4 * q + 1],
                   pk[4 * q + 2], pk[4 * q + 3]);
  }
  sSum[half * 128 + i_row] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();  // P complete

  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 64, 0, 1);
    const uint32_t pa = smem_u32(sKR), va = smem_u32(sV);
#pragma unroll
    for (int kk = 0; kk < kAttnS / 16; ++kk) {
      const int blk = kk >> 2, sub = kk & 3;
      umma_f16_ss(tmem, make_sw128_kmajor_desc(pa + blk * 128 * 128 + sub * 32),
                  make_sw128_mnmajor_desc(va + kk * 16 * 128, 8192, 1024), idesc, kk != 0);
    }
    umma_commit(bar_o);
  }
  mbar_wait(bar_o, 0);
  tc_fence_after();
  {
    uint32_t o[32];
    tmem_ld_32x32b_x32(lane_base + uint32_t(32 * half), o);
    tmem_ld_wait();
    const float inv = 1.0f / (sSum[i_row] + sSum[128 + i_row]);
    const int64_t D = int64_t(H) * kAttnD;
    __nv_bfloat16* dst = out + (int64_t(bt) * S + i_row) * D + int64_t(h) * kAttnD + 32 * half;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16x2(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
      u.y = pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
      u.z = pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
      u.w = pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
      *reinterpret_cast<uint4*>(dst + q * 8) = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace

int rel_attention(const void* qkv, const void* r, const float* rwb, const float* rrb, void* out,
                  int64_t Bt, int64_t S, int64_t H, int64_t dh, int64_t seqs_per_bias,
                  int64_t seqs_per_r, float scale, int dtype, int mode, cudaStream_t stream) {
  if (Bt < 1 || S < 1 || H < 1 || dh < 1 || seqs_per_bias < 1 || Bt % seqs_per_bias ||
      seqs_per_r < 1 || Bt % seqs_per_r)
    return NF_ERR_SHAPE;
  if (dh > 128) return NF_ERR_UNSUPPORTED;
  const uintptr_t al = reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(r) |
                       reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(rwb) |
                       reinterpret_cast<uintptr_t>(rrb);
  if (dtype == NF_BF16 && mode == NF_MODE_FAST && dh == kAttnD && S == kAttnS && (al & 15) == 0 &&
      Bt * H <= (int64_t(1) << 31) - 1) {
    CUtensorMap mq, mr;
    if (!make_qkv_map(&mq, qkv, Bt, S, H) || !make_r_map(&mr, r, Bt / seqs_per_r, S, H))
      return NF_ERR_LAUNCH;
    // 8 warps, one CTA per (sequence, head), two CTAs per SM. Measured
    // faster than a 4-warp kernel (92 vs 79 us per XLNet-base layer at 1536
    // units) and than a persistent double-buffered one.
    static SmemAttrOnce smem_attr;
    smem_attr.set(k_rel_attention_tc8, int(kRel8Smem));
    const int units = int(Bt * H);
    const float scale_log2 = scale * 1.4426950408889634f;
    cudaError_t e = launch_pdl(k_rel_attention_tc8, dim3(units), dim3(256), kRel8Smem, stream, mq,
                               mr, rwb, rrb, static_cast<__nv_bfloat16*>(out), int(H),
                               int(seqs_per_bias), int(seqs_per_r), scale_log2);
    return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
  }
  const int64_t warps = Bt * H * S;
  int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 32) blocks = int64_t(kNumSMs) * 32;
  if (dtype == NF_F32)
    launch_pdl(k_rel_attention_simt<float>, dim3(unsigned(blocks)), dim3(256), 0, stream,
               static_cast<const float*>(qkv), static_cast<const float*>(r), rwb, rrb,
               static_cast<float*>(out), Bt, int(S), int(H), int(dh), int(seqs_per_bias),
               int(seqs_per_r), scale);
  else if (dtype == NF_BF16)
    launch_pdl(k_rel_attention_simt<__nv_bfloat16>, dim3(unsigned(blocks)), dim3(256), 0, stream,
               static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(r), rwb,
               rrb, static_cast<__nv_bfloat16*>(out), Bt, int(S), int(H), int(dh),
               int(seqs_per_bias), int(seqs_per_r), scale);
  else
    return NF_ERR_UNSUPPORTED;
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

int attention(const void* qkv, void* out, int64_t Bt, int64_t S, int64_t H, int64_t dh,
              float scale, int dtype, int mode, cudaStream_t stream) {
  if (Bt < 1 || S < 1 || H < 1 || dh < 1) return NF_ERR_SHAPE;
  if (dh > 128) return NF_ERR_UNSUPPORTED;
  const uintptr_t al = reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(out);
  if (dtype == NF_BF16 && mode == NF_MODE_FAST && dh == kAttnD && S <= kAttnS && (al & 15) == 0 &&
      Bt * H <= (int64_t(1) << 31) - 1) {
    CUtensorMap map;
    if (!make_qkv_map(&map, qkv, Bt, S, H)) return NF_ERR_LAUNCH;
    const int64_t units = Bt * H;
    if (units > 2 * kNumSMs) {
      static SmemAttrOnce pattr;
      pattr.set(k_attention_tc_persistent, int(kAttnPSmem));
      const int grid = 2 * kNumSMs;
      const float sl2 = scale * 1.4426950408889634f;
      cudaError_t e = launch_pdl(k_attention_tc_persistent, dim3(grid), dim3(128), kAttnPSmem,
                                 stream, map, static_cast<__nv_bfloat16*>(out), int(S), int(H),
                                 int(units), sl2);
      return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
    }
    static SmemAttrOnce smem_attr;
    smem_attr.set(k_attention_tc, int(kAttnSmem));
    const float scale_log2 = scale * 1.4426950408889634f;
    cudaError_t e = launch_pdl(k_attention_tc, dim3(unsigned(Bt * H)), dim3(128), kAttnSmem,
                               stream, map, static_cast<__nv_bfloat16*>(out), int(S), int(H),
                               scale_log2);
    return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
  }
  const int64_t warps = Bt * H * S;
  int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 32) blocks = int64_t(kNumSMs) * 32;
  if (dtype == NF_F32)
    launch_pdl(k_attention_simt<float>, dim3(unsigned(blocks)), dim3(256), 0, stream, 
        static_cast<const float*>(qkv), static_cast<float*>(out), Bt, int(S), int(H), int(dh),
        scale);
  else if (dtype == NF_BF16)
    launch_pdl(k_attention_simt<__nv_bfloat16>, dim3(unsigned(blocks)), dim3(256), 0, stream, 
        static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(out), Bt, int(S),
        int(H), int(dh), scale);
  else
    return NF_ERR_UNSUPPORTED;
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

}  // namespace nf
