// fp32 merged convolution on the 5th-gen tensor cores: 3xTF32 implicit GEMM.
//
// Replaces the reference's `grouped_conv2d` / `conv2d` (pkg/src/modelmerge/
// engine.py:122-191) for the fp32 configuration (BASELINE configs[0],
// ResNet-50 merged N=2, fp32, gate 1e-4 normwise) with BatchNorm folded into
// the weights and bias, and residual + ReLU fused into the epilogue.
//
// TF32 keeps 10 mantissa bits, so one TF32 product is good to ~2^-11 — not
// enough for a 1e-4 gate through 50 layers. Each fp32 operand is split
// exactly into hi = x with the low 13 mantissa bits cleared (a TF32 value)
// and lo = x - hi (exact in fp32, |lo| < 2^-10 |x|), and the accumulator
// takes three tcgen05.mma kind::tf32 products per K step:
//     acc += lo_a * hi_b + hi_a * lo_b + hi_a * hi_b
// (the dropped lo_a * lo_b term and lo's own TF32 truncation are ~2^-20 of
// |a b|), accumulating in fp32 in TMEM.
//
// Tile: 128 output pixels (M) x BN output channels (N) of one group; K =
// (kh, kw, c) in 128-byte blocks of 32 fp32. Warp roles (320 threads):
//   warp 0      TMA producer: weight blocks hi and lo (pre-split on the host,
//               (2G, Cout/G, Kpad): hi groups [0, G), lo groups [G, 2G))
//   warp 1      TMEM owner + single-thread MMA issuer
//   warps 2-5   epilogue: TMEM -> registers, split-K fix-up, bias, residual,
//               ReLU, 16-byte fp32 stores (thread = pixel row, NHWC)
//   warps 6-9   im2col gather: cp.async 16-byte channel chunks of the NHWC
//               input (zero-filled outside the image) into the A-hi slot,
//               then an in-place split pass writes hi back and lo into the
//               A-lo slot (each thread splits exactly the chunks it copied)
// One work unit (tile x K split) per CTA; split-K partials reduce in split
// order in an L2 workspace (deterministic), like the bf16 GEMM.
#include "common.cuh"
#include "kernels.h"

namespace nf {

#ifdef NF_TF32_TRACE
// Per-CTA timeline (globaltimer ns) of the last launch, tools/tf32_trace.cu:
// 0 entry, 1 setup done, 2 first stage landed, 3 last MMA issued, 4 accumulator
// ready, 5 partial published, 6 all partials in
__device__ unsigned long long g_tf32_trace[148 * 8];
#define NF_TT(slot)                                                                   \
  do {                                                                                \
    if (blockIdx.x < 148) {                                                           \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_tf32_trace[blockIdx.x * 8 + (slot)] = t_;                                     \
    }                                                                                 \
  } while (0)
#else
#define NF_TT(slot) \
  do {              \
  } while (0)
#endif

namespace {

constexpr int kTM = 128;           // output pixels per tile
constexpr int kTK = 32;            // fp32 elements per 128-byte K block
constexpr int kTThreads = 320;     // TMA + MMA warps, 4 epilogue, 4 gather warps
constexpr int kTEpi = 128;
constexpr int kTGather = 128;
constexpr int kTMaxSplits = 16;  // batch-1 layer3/4 convs: few tiles, long K
constexpr int64_t kTCounterBytes = 64 * 1024;
constexpr int kTLeaveOff = 8192;  // second semaphore bank: [tile] splits done reducing

template <int BN>
struct TfCfg {
  static constexpr int kA = kTM * 128;  // one A half (hi or lo)
  static constexpr int kB = BN * 128;   // one B half
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kStages = (220 * 1024) / kStage;
  static constexpr size_t kBytes = 1024 + size_t(kStages) * kStage + 512;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  // cp.async groups in flight per gather thread; < kStages, or the gather
  // would wait on a slot whose fill it has not yet published
  static constexpr int kLag = kStages - 1 < 3 ? kStages - 1 : 3;
  static_assert(kStages >= 3 && kStages <= 16, "ring depth");
};

struct TfParams {
  const float* x;        // NHWC input, C channels (group g: channels [g*cg, (g+1)*cg))
  const float* bias;     // (Cout) fp32 or null (BN shift folded in)
  const float* residual; // NHWC like y, or null
  float* y;              // NHWC (N, Ho, Wo, Cout)
  int H, W, C, cg, k, S, P, Ho, Wo, pix, coutg, Cout, G, relu;
  int kb_total, kb_per_split, splits, tiles_m, tiles_n, units;
  FastDiv fd_cg, fd_k, fd_Wo, fd_Ho;  // gather divisors
  float* ws;             // split-K partials [tile][split][BN][128]
  unsigned* counters;    // [tile] arrival semaphores (zero between launches)
};

// kind::tf32, fp32 accumulate: D fmt [4,6)=1, A/B fmt [7,10)/[10,13)=2 (TF32),
// K-major operands, N>>3 at [17,23), M>>4 at [24,29).
constexpr uint32_t make_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}

// hi = x with the low 13 mantissa bits cleared (exactly representable in
// TF32, so the tensor core's truncation is the identity), lo = x - hi (exact).
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t& hi, uint32_t& lo) {
  hi = x & 0xFFFFE000u;
  lo = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi));
}

template <int BN>
__global__ void __launch_bounds__(kTThreads, 1)
    k_conv_tf32x3(const __grid_constant__ CUtensorMap map_w, TfParams p) {
  using C = TfCfg<BN>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  // stage s: [A hi | A lo | B hi | B lo]
  auto a_hi = [&](int s) { return smem + size_t(s) * C::kStage; };
  auto a_lo = [&](int s) { return smem + size_t(s) * C::kStage + C::kA; };
  auto b_hi = [&](int s) { return smem + size_t(s) * C::kStage + 2 * C::kA; };
  auto b_lo = [&](int s) { return smem + size_t(s) * C::kStage + 2 * C::kA + C::kB; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(kStages) * C::kStage);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x;
  const int split = u % p.splits;
  const int tile = u / p.splits;
  const int tm = tile % p.tiles_m;
  const int tn = (tile / p.tiles_m) % p.tiles_n;
  const int g = tile / (p.tiles_m * p.tiles_n);
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) NF_TT(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + kTGather);  // producer's expect_tx + every gather thread
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) NF_TT(1);
  grid_dependents_launch();

  if (warp == 0) {
    // weights do not depend on the previous kernel: no dependency wait
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], 2 * C::kB);
        const int kc = (kb0 + i) * kTK;
        tma_load_3d(b_hi(s), &map_w, &full[s], kc, tn * BN, g, kEvictFirst);
        tma_load_3d(b_lo(s), &map_w, &full[s], kc, tn * BN, p.G + g, kEvictFirst);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_tf32(kTM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      mbar_wait(&full[s], (i / kStages) & 1);
      tc_fence_after();
      if (lane == 0 && i == 0) NF_TT(2);
      if (lane == 0) {
        const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(s));
        const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // 8 TF32 (32 bytes) per MMA
          const uint32_t o = kk * 32;
          umma_tf32(tmem_base, make_sw128_kmajor_desc(al + o), make_sw128_kmajor_desc(bh + o),
                    idesc, (i | kk) ? 1u : 0u);
          umma_tf32(tmem_base, make_sw128_kmajor_desc(ah + o), make_sw128_kmajor_desc(bl + o),
                    idesc, 1u);
          umma_tf32(tmem_base, make_sw128_kmajor_desc(ah + o), make_sw128_kmajor_desc(bh + o),
                    idesc, 1u);
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(tfull);
    if (lane == 0) NF_TT(3);
    __syncwarp();
  } else if (warp < 2 + kTEpi / 32) {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int etid = threadIdx.x - 64;
    const int pix = tm * kTM + row;
    const bool pix_ok = pix < p.pix;
    const int c0 = g * p.coutg + tn * BN;  // first output channel of the tile
    grid_dependency_wait();                // residual / y / workspace follow the producer grid
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (etid == 0) NF_TT(4);
    const uint32_t t_row = tmem_base + (uint32_t(quarter * 32) << 16);
    // bias / residual / ReLU and the 16-byte NHWC stores of 4 channels
    auto store4 = [&](int chl, float4 v4) {  // chl: channel offset within the tile
      if (!pix_ok || tn * BN + chl >= p.coutg) return;
      const int ch = c0 + chl;
      if (p.bias) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + ch));
        v4.x += b4.x; v4.y += b4.y; v4.z += b4.z; v4.w += b4.w;
      }
      const int64_t off = int64_t(pix) * p.Cout + ch;
      if (p.residual) {
        const float4 r4 = __ldcg(reinterpret_cast<const float4*>(p.residual + off));
        v4.x += r4.x; v4.y += r4.y; v4.z += r4.z; v4.w += r4.w;
      }
      if (p.relu) {
        v4.x = fmaxf(v4.x, 0.f); v4.y = fmaxf(v4.y, 0.f);
        v4.z = fmaxf(v4.z, 0.f); v4.w = fmaxf(v4.w, 0.f);
      }
      *reinterpret_cast<float4*>(p.y + off) = v4;
    };
    if (p.splits == 1) {
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + uint32_t(cc), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          store4(cc + j, make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                     __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
      }
    } else {
      // Split-K: every split publishes its fp32 partial ([split][col][row]
      // in an L2 workspace), waits until all splits of the tile have, then
      // reduces and stores ITS OWN slice of the tile's columns, summing the
      // partials in split order (deterministic). The split CTAs of a tile
      // are co-resident (units <= #SMs, one CTA per SM), so the wait is
      // safe; the reduction is spread over the splits instead of serialised
      // in the last arriver (16 splits: 1 MB of L2 reads for one CTA).
      float* part = p.ws + int64_t(tile) * p.splits * BN * kTM;
      float* mine = part + int64_t(split) * BN * kTM + row;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + uint32_t(cc), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) __stcg(mine + (cc + j) * kTM, __uint_as_float(r[j]));
      }
      named_bar_sync(1, kTEpi);
      unsigned* arrive = p.counters + tile;
      unsigned* leave = p.counters + kTLeaveOff + tile;
      if (etid == 0) {
        NF_TT(5);
        publish_count(arrive);  // releases the CTA's partials (after the barrier)
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(arrive) : "memory");
          if (seen < unsigned(p.splits)) __nanosleep(64);
        } while (seen < unsigned(p.splits));
      }
      named_bar_sync(1, kTEpi);
      if (etid == 0) NF_TT(6);
      // columns [c_lo, c_hi) of the tile, a multiple of 4 per split
      const int per = ((BN / 4 + p.splits - 1) / p.splits) * 4;
      const int c_lo = split * per, c_hi = min(BN, c_lo + per);
#pragma unroll 1
      for (int cc = c_lo; cc < c_hi; cc += 4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s2 = 0; s2 < p.splits; ++s2) {
          const float* src = part + int64_t(s2) * BN * kTM + int64_t(cc) * kTM + row;
          acc.x += __ldcg(src);
          acc.y += __ldcg(src + kTM);
          acc.z += __ldcg(src + 2 * kTM);
          acc.w += __ldcg(src + 3 * kTM);
        }
        store4(cc, acc);
      }
      named_bar_sync(1, kTEpi);
      // the last split out re-arms both counters for the next launch (every
      // split has passed its wait on `arrive` by then)
      if (etid == 0 && atomicAdd(leave, 1u) == unsigned(p.splits - 1)) {
        *arrive = 0u;
        *leave = 0u;
      }
    }
  } else {
    // --------------------------- im2col gather ----------------------------
    const int gt = threadIdx.x - (64 + kTEpi);
    const int j = gt & 7;    // 16-byte chunk (4 channels) of the 128-byte K row
    const int rb = gt >> 3;  // rows rb + 16 * i
    const float* xg = p.x + int64_t(g) * p.cg;
    int ih0[8], iw0[8], base[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int px = tm * kTM + rb + 16 * i;
      const int t2 = p.fd_Wo.div(px);
      const int ow = px - t2 * p.Wo;
      const int n = p.fd_Ho.div(t2);
      const int oh = t2 - n * p.Ho;
      ih0[i] = px < p.pix ? oh * p.S - p.P : -(1 << 20);
      iw0[i] = ow * p.S - p.P;
      base[i] = n * p.H * p.W;
    }
    const int taps = p.k * p.k;
    auto chunk_off = [&](int i) {
      const int r = rb + 16 * i;
      return uint32_t(r * 128) + (uint32_t(j ^ (r & 7)) << 4);
    };
    // split pass of a landed stage: hi in place, lo into the A-lo slot
    auto split_stage = [&](int s) {
      const uint32_t h0 = smem_u32(a_hi(s)), l0 = smem_u32(a_lo(s));
      // the eight 16-byte reads first, then split + write back: one
      // shared-memory latency per stage instead of eight in series
      uint32_t w[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                     : "r"(h0 + chunk_off(i)));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t o = chunk_off(i);
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(w[i][e], hi[e], lo[e]);
        st_shared_v4(h0 + o, hi[0], hi[1], hi[2], hi[3]);
        st_shared_v4(l0 + o, lo[0], lo[1], lo[2], lo[3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    };
    grid_dependency_wait();  // x is the previous kernel's output
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      const int k0 = (kb0 + i) * kTK + j * 4;
      const int tap = p.fd_cg.div(k0);
      const int ch = k0 - tap * p.cg;
      const int kh = p.fd_k.div(tap);
      const int kw = tap - kh * p.k;
      const bool tap_ok = tap < taps;
      const uint32_t dst0 = smem_u32(a_hi(s));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int ih = ih0[q] + kh, iw = iw0[q] + kw;
        const bool ok = tap_ok && ih >= 0 && ih < p.H && iw >= 0 && iw < p.W;
        const float* src = ok ? xg + (int64_t(base[q]) + ih * p.W + iw) * p.C + ch : p.x;
        cp_async16(dst0 + chunk_off(q), src, ok ? 16 : 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (i >= C::kLag) {
        asm volatile("cp.async.wait_group %0;" ::"n"(C::kLag) : "memory");
        split_stage((i - C::kLag) % kStages);
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (int i = max(nkb - C::kLag, 0); i < nkb; ++i) split_stage(i % kStages);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

bool make_f32_map(CUtensorMap* map, const void* base, int64_t G2, int64_t rows, int64_t inner,
                  int box_rows) {
  // fp32 (2G, rows, inner) weights, box (32, box_rows, 1), SWIZZLE_128B
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = []() -> EncodeFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeFn>(f);
  }();
  if (!fn || (inner * 4) % 16 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(G2)};
  cuuint64_t strides[2] = {cuuint64_t(inner * 4), cuuint64_t(rows * inner * 4)};
  cuuint32_t box[3] = {cuuint32_t(kTK), cuuint32_t(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TfPlan {
  int bn, tiles_m, tiles_n, splits, kb_total;
};

TfPlan tf_plan(int64_t pix, int64_t coutg, int64_t G, int64_t Kpad, int64_t ws_bytes) {
  TfPlan t;
  t.bn = coutg <= 32 ? 32 : (coutg <= 64 ? 64 : 128);
  t.tiles_m = int((pix + kTM - 1) / kTM);
  t.tiles_n = int((coutg + t.bn - 1) / t.bn);
  t.kb_total = int((Kpad + kTK - 1) / kTK);
  const int64_t tiles = G * t.tiles_m * t.tiles_n;
  int s = 1;
  if (ws_bytes > kTCounterBytes && tiles < kNumSMs && tiles <= kTLeaveOff) {
    s = int(kNumSMs / tiles);
    s = s < kTMaxSplits ? s : kTMaxSplits;
    s = s < t.kb_total / 4 ? s : t.kb_total / 4;  // >= 4 K blocks per split
    while (s > 1 && tiles * s * int64_t(kTM) * t.bn * 4 > ws_bytes - kTCounterBytes) --s;
    if (s < 1) s = 1;
  }
  t.splits = s;
  return t;
}

template <int BN>
int launch_tf32(const CUtensorMap& mw, const TfParams& p, cudaStream_t stream) {
  static SmemAttrOnce smem_attr;
  smem_attr.set(k_conv_tf32x3<BN>, int(TfCfg<BN>::kBytes));
  cudaError_t e = launch_pdl(k_conv_tf32x3<BN>, dim3(p.units), dim3(kTThreads),
                             TfCfg<BN>::kBytes, stream, mw, p);
  return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

}  // namespace

int64_t conv_tf32_workspace_bytes(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                  int64_t G, int64_t k, int64_t stride, int64_t pad,
                                  int64_t Kpad) {
  if (G < 1 || C % G || Cout % G || stride < 1) return 0;
  const int64_t Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const TfPlan t = tf_plan(N * Ho * Wo, Cout / G, G, Kpad, INT64_MAX);
  if (t.splits <= 1) return 0;
  return kTCounterBytes + G * t.tiles_m * t.tiles_n * int64_t(t.splits) * kTM * t.bn * 4;
}

// x NHWC fp32 (C = G * cg, cg % 4 == 0), w (2G, Cout/G, Kpad) fp32 K-major
// with K = (kh, kw, c): [0, G) the TF32 hi parts, [G, 2G) the lo parts;
// bias (Cout) fp32 or null; residual / y NHWC fp32 (N, Ho, Wo, Cout).
int grouped_conv_tf32(const void* x, const void* w, const float* bias, const void* residual,
                      void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                      int pad, int Kpad, int relu, void* ws, int64_t ws_bytes,
                      cudaStream_t stream) {
  if (N < 1 || H < 1 || W < 1 || G < 1 || C % G || Cout % G || k < 1 || stride < 1 || pad < 0)
    return NF_ERR_SHAPE;
  const int cg = C / G, coutg = Cout / G;
  if (cg % 4 || coutg % 4 || Kpad % kTK || Kpad < k * k * cg) return NF_ERR_UNSUPPORTED;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1) return NF_ERR_SHAPE;
  const int64_t pix = int64_t(N) * Ho * Wo;
  if (pix > (int64_t(1) << 30) || int64_t(N) * H * W * C > (int64_t(1) << 31))
    return NF_ERR_UNSUPPORTED;
  const uintptr_t al = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                       reinterpret_cast<uintptr_t>(residual) | reinterpret_cast<uintptr_t>(bias);
  if (al & 15) return NF_ERR_UNSUPPORTED;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255)) return NF_ERR_SHAPE;
  const TfPlan t = tf_plan(pix, coutg, G, Kpad, ws ? ws_bytes : 0);
  TfParams p{};
  p.x = static_cast<const float*>(x);
  p.bias = bias;
  p.residual = static_cast<const float*>(residual);
  p.y = static_cast<float*>(y);
  p.H = H; p.W = W; p.C = C; p.cg = cg; p.k = k; p.S = stride; p.P = pad;
  p.Ho = Ho; p.Wo = Wo; p.pix = int(pix); p.coutg = coutg; p.Cout = Cout; p.G = G;
  p.relu = relu;
  p.fd_cg = FastDiv::make(cg);
  p.fd_k = FastDiv::make(k);
  p.fd_Wo = FastDiv::make(Wo);
  p.fd_Ho = FastDiv::make(Ho);
  p.kb_total = t.kb_total;
  p.kb_per_split = (t.kb_total + t.splits - 1) / t.splits;
  p.splits = (t.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.tiles_m = t.tiles_m;
  p.tiles_n = t.tiles_n;
  const int64_t units = int64_t(G) * t.tiles_m * t.tiles_n * p.splits;
  if (units > (int64_t(1) << 31) - 1) return NF_ERR_UNSUPPORTED;
  p.units = int(units);
  p.counters = static_cast<unsigned*>(ws);
  p.ws = ws ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kTCounterBytes) : nullptr;
  CUtensorMap mw;
  if (!make_f32_map(&mw, w, 2 * G, coutg, Kpad, t.bn)) return NF_ERR_UNSUPPORTED;
  if (t.bn == 32) return launch_tf32<32>(mw, p, stream);
  if (t.bn == 64) return launch_tf32<64>(mw, p, stream);
  return launch_tf32<128>(mw, p, stream);
}

}  // namespace nf
