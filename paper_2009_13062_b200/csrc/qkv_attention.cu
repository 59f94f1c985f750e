// Fused merged QKV projection + attention for batch-1 encoders (one CTA per
// (instance, head)): the projection  [Q|K|V]_h = x_g · W_g[h]^T + b  runs on
// tcgen05 with M = 128 tokens, N = 192 (the head's 64 q, 64 k and 64 v
// features), K = d_model streamed by TMA; its epilogue writes Q, K, V as
// K-major bf16 tiles straight into shared memory, where the attention of
// k_attention_tc continues (S = QK^T in TMEM, register softmax, P·V). The
// per-head QKV activations never reach HBM and one launch replaces two.
//
// Replaces, for the merged graph's MatMul(qkv) -> Attention pair at batch 1,
// the reference-side composition `batch_matmul` (engine.py:215-235) followed
// by the attention restatement (oracle/kernels.py::attention).
#include "common.cuh"
#include "kernels.h"

namespace nf {

bool make_bf16_map(CUtensorMap* map, const void* base, int64_t G, int64_t rows, int64_t inner,
                   int box_inner, int box_rows, int64_t row_stride, int64_t g_stride);
bool make_bf16_map_kpt2(CUtensorMap* map, const void* base, int64_t G, int64_t rows, int64_t K,
                        int box_rows, int64_t row_stride, int64_t g_stride, int kpt);

namespace {

constexpr int kQS = 128;                 // tokens (= queries = keys)
constexpr int kQD = 64;                  // head dim
constexpr int kQTile = kQS * kQD * 2;    // 16 KB: one 128 x 64 bf16 tile
// Each ring stage holds two 64-wide k-blocks, delivered by one 4-D TMA box
// per operand (the projection main loop is bound by a per-transaction cost):
// x (128 tokens) and the head's 192 weight rows, stored head-major
// (G, H, [q|k|v], 64, D) so that they are one contiguous box.
constexpr int kQKPT = 2;
constexpr int kQStages = 2;
constexpr int kQABytes = kQTile * kQKPT;         // x: 2 x (128 tokens x 64 K)
constexpr int kQBBytes = 3 * kQD * 128 * kQKPT;  // w: 2 x (192 rows x 64 K) = 48 KB
constexpr int kQStageBytes = kQABytes + kQBBytes;
// + bias and folded-LN column sums of the head's 192 features (fp32)
constexpr size_t kQSmem = 1024 + size_t(kQStages) * kQStageBytes + 3 * kQTile + 256 + 2 * 192 * 4;

__device__ __forceinline__ uint32_t sw128_off(int r, int chunk16) {
  return uint32_t(r * 128 + ((chunk16 ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(192, 1)
    k_qkv_attention_tc(const __grid_constant__ CUtensorMap map_x,
                       const __grid_constant__ CUtensorMap map_w, const float* __restrict__ bias,
                       __nv_bfloat16* __restrict__ out, int H, int kb_total, float scale_log2,
                       const float2* nin_stats,
                       const float* nin_colsum, int nin_parts, float nin_eps,
                       const unsigned* dep, unsigned dep_target, unsigned* done) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* sQ = smem + kQStages * kQStageBytes;
  uint8_t* sK = sQ + kQTile;
  uint8_t* sV = sK + kQTile;
  uint8_t* sP = sQ;  // 128 x 128 bf16 = Q|K once S = QK^T retired
  uint64_t* full = reinterpret_cast<uint64_t*>(sV + kQTile);
  uint64_t* empty = full + kQStages;
  uint64_t* bar_acc = empty + kQStages;
  uint64_t* bar_s = bar_acc + 1;
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_o + 1);
  float* sBias = reinterpret_cast<float*>(sV + kQTile + 256);  // [192]
  float* sCs = sBias + 192;                                     // [192]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x / H;
  const int h = blockIdx.x % H;
  const int D = H * kQD;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_x);
    tma_prefetch_desc(&map_w);
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bar_acc, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // cols [0,192): projection; then S [0,128), O [128,192)
  grid_dependents_launch();

  if (warp == 0) {
    if (lane == 0) {
      auto load_w = [&](int stage, int st) {
        tma_load_4d(ring + stage * kQStageBytes + kQABytes, &map_w, &full[stage], 0,
                    h * 3 * kQD, st * kQKPT, g, kEvictFirst);
      };
      auto load_x = [&](int stage, int st) {
        tma_load_4d(ring + stage * kQStageBytes, &map_x, &full[stage], 0, 0, st * kQKPT, g,
                    kEvictLast);
      };
      const int n_st = (kb_total + kQKPT - 1) / kQKPT;
      // weights do not depend on the previous kernel: first ring before the wait
      const int pre = n_st < kQStages ? n_st : kQStages;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], kQStageBytes);
        load_w(i, i);
      }
      // x (and its statistics) come from the previous launch -- or, when it
      // is a chained launch that counts instance g's stored output tiles,
      // from that counter: this head starts as soon as ITS instance is done
      if (dep) wait_counter(dep + g, dep_target);
      else grid_dependency_wait();
      for (int i = 0; i < pre; ++i) load_x(i, i);
      for (int st = pre; st < n_st; ++st) {
        const int stage = st % kQStages;
        mbar_wait(&empty[stage], ((st / kQStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[stage], kQStageBytes);
        load_w(stage, st);
        load_x(stage, st);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16_f32(128, 3 * kQD);
    const int n_st = (kb_total + kQKPT - 1) / kQKPT;
    for (int st = 0; st < n_st; ++st) {
      const int stage = st % kQStages;
      mbar_wait(&full[stage], (st / kQStages) & 1);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int hk = 0; hk < kQKPT; ++hk) {
          const int kb = st * kQKPT + hk;
          if (kb >= kb_total) break;
          const uint32_t a = smem_u32(ring + stage * kQStageBytes) + hk * kQTile;
          const uint32_t b = smem_u32(ring + stage * kQStageBytes + kQABytes) + hk * (3 * kQD * 128);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_ss(tmem, make_sw128_kmajor_desc(a + kk * 32),
                        make_sw128_kmajor_desc(b + kk * 32), idesc, (kb | kk) != 0);
        }
        umma_commit(&empty[stage]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(bar_acc);
    __syncwarp();
  } else {
    // -------- warps 2..5: projection epilogue, then attention (thread = token)
    const int t = (warp & 3) * 32 + lane;  // TMEM lane == token row
    const int etid = threadIdx.x - 64;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const float* bq = bias ? bias + int64_t(g) * 3 * D : nullptr;
    // folded LayerNorm of x (GemmParams::nin_*): y = rstd * (x W'^T - mean * colsum) + b'
    const float* csq = nin_stats ? nin_colsum + int64_t(g) * 3 * D : nullptr;
    // The head's bias / column sums into smem while the projection runs (cold
    // L2 misses off the epilogue's critical path).
    for (int i = etid; i < 3 * kQD; i += 128) {
      const int64_t f = int64_t(i / kQD) * D + h * kQD + (i % kQD);
      sBias[i] = bq ? __ldg(bq + f) : 0.f;
      sCs[i] = csq ? __ldg(csq + f) : 0.f;
    }
    float2 ms = make_float2(0.f, 1.f);
    if (nin_stats) {
      // the stats come from the previous launch (or its instance-g counter)
      if (dep) {
        if (etid == 0) wait_counter(dep + g, dep_target);
        named_bar_sync(1, 128);
      } else {
        grid_dependency_wait();
      }
      ms = fold_stats(nin_stats, nin_parts, kQS, g, t, 1.0f / float(D), nin_eps);
    }
    named_bar_sync(1, 128);
    mbar_wait(bar_acc, 0);
    tc_fence_after();
    // features [0,64) q, [64,128) k, [128,192) v of head h -> K-major tiles
#pragma unroll 1
    for (int c = 0; c < 6; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + lane_off + uint32_t(c * 32), r);
      tmem_ld_wait();
      const int part = c >> 1;                  // 0 q, 1 k, 2 v
      const int f0 = (c & 1) * 32;              // column within the head
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (csq) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = ms.y * fmaf(-ms.x, sCs[c * 32 + j], v[j]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += sBias[c * 32 + j];
      uint8_t* tile = part == 0 ? sQ : (part == 1 ? sK : sV);
      const uint32_t base = smem_u32(tile);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_shared_v4(base + sw128_off(t, (f0 >> 3) + q), pack_bf16x2(v[8 * q], v[8 * q + 1]),
                     pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                     pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                     pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
    }
    fence_proxy_async_smem();  // generic smem writes -> tensor-core reads
    tc_fence_before();
    named_bar_sync(1, 128);
    if (etid == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = make_idesc_bf16_f32(128, 128);
      const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
      for (int kk = 0; kk < kQD / 16; ++kk)
        umma_f16_ss(tmem, make_sw128_kmajor_desc(qa + kk * 32), make_sw128_kmajor_desc(ka + kk * 32),
                    idesc, kk != 0);
      umma_commit(bar_s);
    }
    mbar_wait(bar_s, 0);
    tc_fence_after();
    uint32_t s[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem + lane_off + uint32_t(c * 32), s[c]);
    tmem_ld_wait();
    float mx = -INFINITY;
    {
      float m8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) m8[q] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j) m8[j & 7] = fmaxf(m8[j & 7], __uint_as_float(s[c][j]));
#pragma unroll
      for (int q = 0; q < 8; ++q) mx = fmaxf(mx, m8[q]);
    }
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
    const float mxs = mx * scale_log2;
    const uint32_t prow = smem_u32(sP);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float x0 = fmaf(__uint_as_float(s[c][j]), scale_log2, -mxs);
        const float x1 = fmaf(__uint_as_float(s[c][j + 1]), scale_log2, -mxs);
        const uint32_t packed = pack_bf16x2(ex2_approx(x0), ex2_approx(x1));
        s4[(j >> 1) & 3] += __uint_as_float(packed << 16) + __uint_as_float(packed & 0xffff0000u);
        pk[j >> 1] = packed;
      }
      // P row t, keys c*32 .. c*32+31: K-major over keys, 2 blocks of 64
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int key = c * 32 + q * 8;
        st_shared_v4(prow + uint32_t((key >> 6) * kQS * 128) + sw128_off(t, (key & 63) >> 3),
                     pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
    const float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    fence_proxy_async_smem();
    tc_fence_before();
    named_bar_sync(1, 128);
    if (etid == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = make_idesc_bf16_f32(128, kQD, 0, 1);
      const uint32_t pa = smem_u32(sP), va = smem_u32(sV);
#pragma unroll
      for (int kk = 0; kk < kQS / 16; ++kk) {
        const int blk = kk >> 2, sub = kk & 3;
        umma_f16_ss(tmem + 128, make_sw128_kmajor_desc(pa + blk * kQS * 128 + sub * 32),
                    make_sw128_mnmajor_desc(va + kk * 16 * 128, 8192, 1024), idesc, kk != 0);
      }
      umma_commit(bar_o);
    }
    mbar_wait(bar_o, 0);
    tc_fence_after();
    {
      uint32_t o[2][32];
      tmem_ld_32x32b_x32(tmem + lane_off + 128, o[0]);
      tmem_ld_32x32b_x32(tmem + lane_off + 160, o[1]);
      tmem_ld_wait();
      const float inv = 1.0f / sum;
      __nv_bfloat16* dst = out + (int64_t(g) * kQS + t) * D + int64_t(h) * kQD;
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
    if (done) {
      // this head's context is stored: count it for instance g (a chained
      // launch's first op starts g's units at H heads)
      named_bar_sync(1, 128);
      if (etid == 0) publish_count(done + g);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace

// x (G, 128, D) bf16 rows (x_ld / x_gs element strides), w (G, 3D, D) K-major
// bf16 with head-major rows: row h*192 + part*64 + j = feature part*D + h*64 + j
// (part 0 q, 1 k, 2 v), bias (G, 3D) fp32 in feature order or
// null; out (G, 128, D) bf16 context. heads * 64 == D.
int qkv_attention_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w, const float* bias,
                     void* out, int64_t G, int64_t S, int64_t D, int64_t heads, float scale,
                     cudaStream_t stream, const NormFold* fold, const unsigned* dep,
                     unsigned dep_target, unsigned* done) {
  if (G < 1 || heads < 1 || D != heads * kQD) return NF_ERR_SHAPE;
  const float2* nin = fold ? reinterpret_cast<const float2*>(fold->in_stats) : nullptr;
  if (nin && (!fold->in_colsum || fold->in_parts < 1)) return NF_ERR_SHAPE;
  if (S != kQS || D % 64 || G * heads > (int64_t(1) << 31) - 1) return NF_ERR_UNSUPPORTED;
  CUtensorMap mx, mw;
  if (!make_bf16_map_kpt2(&mx, x, G, S, D, kQS, x_ld, x_gs, kQKPT) ||
      !make_bf16_map_kpt2(&mw, w, G, 3 * D, D, 3 * kQD, 0, 0, kQKPT))
    return NF_ERR_UNSUPPORTED;
  static SmemAttrOnce smem_attr;
  smem_attr.set(k_qkv_attention_tc, int(kQSmem));
  const float sl2 = scale * 1.4426950408889634f;
  cudaError_t e = launch_pdl(k_qkv_attention_tc, dim3(unsigned(G * heads)), dim3(192), kQSmem,
                             stream, mx, mw, bias, static_cast<__nv_bfloat16*>(out), int(heads),
                             int(D / 64), sl2, nin,
                             nin ? fold->in_colsum : nullptr, nin ? fold->in_parts : 0,
                             nin ? fold->in_eps : 0.f, dep, dep_target, done);
  return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

}  // namespace nf
