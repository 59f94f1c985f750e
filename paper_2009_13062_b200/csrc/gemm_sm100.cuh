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
//
// Implicit-GEMM convolution (GATHER = 16 or 8): the activation operand is
// not a TMA tile but im2col rows gathered straight from the NHWC input by
// four extra warps (6..9) with cp.async (16- or 8-byte channel chunks,
// zero-filled outside the image / past the last tap) into the same
// SWIZZLE_128B K-major layout; K = (kh, kw, c) padded to 64. Weights still
// stream by TMA. Replaces the reference's `grouped_conv2d`
// (engine.py:155-191) without materialising im2col in HBM.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace nf {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kGemmThreads = 192;  // TMA warp + MMA warp + 4 epilogue warps
// Wide tiles get 8 epilogue warps (two per TMEM lane quarter, each taking
// half of the columns): the GELU / residual epilogue of a 128x256 tile then
// keeps up with the next tile's main loop.
template <int BN>
constexpr int epi_warps() { return BN >= 128 ? 8 : 4; }
template <int BN, int GATHER>
constexpr int gemm_threads() { return 64 + 32 * epi_warps<BN>() + (GATHER ? 128 : 0); }
constexpr int kGatherThreads = 128;
constexpr int kGatherLag = 8;  // cp.async groups in flight per gather thread
constexpr int kOutBlock = 64;  // features per 128-byte output block (bf16)
constexpr int kMaxSplits = 8;
#ifndef NF_GEMM_BUDGET_KB
#define NF_GEMM_BUDGET_KB 220  // smem for the operand ring + output staging
#endif
constexpr int64_t kCounterBytes = 64 * 1024;  // semaphores at the workspace head
static __device__ float g_zero_bias[1];  // bias operand of bias-free launches

#ifdef NF_GEMM_TRACE
// Per-CTA pipeline timestamps (globaltimer ns), 8 slots per CTA:
// 0 entry, 1 setup done, 2 first stage landed (MMA warp), 3 last MMA
// committed, 4 first accumulator ready (epilogue), 5 epilogue done, 6 exit.
__device__ unsigned long long g_gemm_trace[148 * 8];
NF_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define NF_TRACE(slot)                                                          \
  do {                                                                          \
    if (blockIdx.x < 148) g_gemm_trace[blockIdx.x * 8 + (slot)] = gtimer();     \
  } while (0)
// Stall accounting (ns spent in mbarrier waits, per CTA and role):
// 0 producer<-empty, 1 mma<-full, 2 mma<-tempty, 3 epilogue<-tfull, 4 epilogue busy
__device__ unsigned long long g_gemm_wait[148 * 8];
#define NF_WAIT_BEGIN() const unsigned long long nf_w0_ = gtimer()
#define NF_WAIT_END(slot)                                                       \
  do {                                                                          \
    if (blockIdx.x < 148) g_gemm_wait[blockIdx.x * 8 + (slot)] += gtimer() - nf_w0_; \
  } while (0)
#else
#define NF_WAIT_BEGIN() do {} while (0)
#define NF_WAIT_END(slot) do {} while (0)
#define NF_TRACE(slot) \
  do {                 \
  } while (0)
#endif

struct GemmParams {
  int act;               // fused epilogue activation (NF_ACT_*)
  const float* bias;     // (G, features) fp32 or nullptr
  const void* residual;  // y-shaped bf16 or nullptr
  int64_t out_gstride;   // elements between instances of y
  int64_t out_ld;        // elements between tokens of y
  int rows_a, rows_b;    // valid rows of A / B
  int features;          // N (bias stride per instance)
  int tiles_a, tiles_b, groups;
  int splits, kb_total, kb_per_split, units;
  // divisors of the unit decode / conv gather (gemm_params_finalize)
  FastDiv fd_splits, fd_ta, fd_tb, fd_cWo, fd_cHo, fd_cCg, fd_cK;
  float* ws;             // split-K partials [tile][split][128][BN]
  unsigned* counters;    // [tile] arrival semaphores (zero between launches)
  void* y_direct;        // y for tiles stored straight from registers (!kStaged)
  // implicit-GEMM conv geometry (GATHER kernels only)
  const __nv_bfloat16* cx;  // NHWC input
  int cH, cW, cC, cCg, cK, cS, cP, cHo, cWo;
  int halo_w, halo_bytes;    // GATHER == 1: halo box width, bytes per buffer (1 KB aligned)
  int halo_cpp;              // channels per halo pixel (cg, or 8 for cg == 4: 16-byte boxes)
  uint32_t halo_tx;          // bytes one halo TMA box delivers
  // Folded LayerNorms (swapped staged tiles): LN(v) over an instance's D
  // features per token is never materialised; its producer writes per-token
  // statistics (sum, centred sum of squares M2) of each of its 128-feature
  // tiles, [g][part][token], and consumers merge them (Chan et al.) and
  // rebuild the normalised value.
  //  in : B operand (tokens) = LN(x); the weights carry gamma, the bias beta,
  //       colsum[g][n] = sum_k W'[g][n][k]:  y = rstd * (x W'^T - mean * colsum) + b'
  //  res: residual = LN(r) = (r - mean) * rstd * gamma[n] + beta[n]
  //  out: this launch's output tiles feed a later LN: write their partial sums
  const float2* nin_stats;
  const float* nin_colsum;
  int nin_parts;
  float nin_inv_d, nin_eps;
  const float2* nres_stats;
  const float* nres_gamma;
  const float* nres_beta;
  int nres_parts;
  float nres_inv_d, nres_eps;
  float2* nout_stats;
  // Per-instance launch linking (CNN plans; all null = wait for the whole
  // previous launch as usual). The instance of a unit is g / link_gpi.
  // dep_x / dep_r: [instance] counters of stored tiles of the launches that
  // produced the activations / the residual -- a unit starts once its
  // instance reached the target, not once the previous launch finished.
  // done: this launch's [instance] counter, bumped per stored output tile.
  const unsigned* dep_x;
  const unsigned* dep_r;
  unsigned* done;
  unsigned dep_x_target, dep_r_target;
  int link_gpi;
};


// Persistent grid with equal units per CTA: the waves one CTA per slot
// needs, spread evenly (e.g. 192 units on 148 SMs: 96 CTAs x 2).
inline int balanced_grid(int64_t units, int slots) {
  if (units <= slots) return int(units);
  const int64_t waves = (units + slots - 1) / slots;
  return int((units + waves - 1) / waves);
}

#ifndef NF_GEMM_LITE_KB
#define NF_GEMM_LITE_KB 100  // swapped (weight-streaming) tiles: 2 CTAs per SM
#endif

// Output path of a tile configuration: staged = registers -> swizzled smem ->
// TMA store for tiles of >= 64 columns; narrow tiles (grouped convs with
// 4..32 channels per group) store straight from registers. (Direct stores
// from swapped tiles measured slower: 4 us vs 1.8 us per 128x128 epilogue.)
template <int BN, bool SWAP>
struct GemmOut {
  static constexpr bool kStaged = BN >= 64;
};

#ifndef NF_GEMM_PAIR_KB
#define NF_GEMM_PAIR_KB 225  // CTA-pair 128 x 256 tiles: 5 stages of 32 KB + 64 KB staging
#endif
#ifndef NF_GEMM_GATHER_KB
#define NF_GEMM_GATHER_KB NF_GEMM_BUDGET_KB
#endif
#ifndef NF_GEMM_HALO_KB
#define NF_GEMM_HALO_KB 120  // operand ring of halo-gather convs (2 halo buffers follow)
#endif

// KPT: k-blocks per TMA transaction / ring stage (2: one 4-D box per operand
// covers two 64-wide k-blocks).
template <int BN, bool SWAP, bool PAIR = false, int GATHER = 0, int KPT = 1>
struct GemmCfg {
  static constexpr bool kStaged = GemmOut<BN, SWAP>::kStaged;
  static constexpr int kABytes = kGemmBM * kGemmBK * 2 * KPT;
  static constexpr int kBBytes = (PAIR ? BN / 2 : BN) * kGemmBK * 2 * KPT;  // pair: half of B each
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOutBytes = kStaged ? kGemmBM * BN * 2 : 0;
  // Swapped tiles stream weights at batch 1: a small footprint lets the next
  // kernel's CTA (programmatic dependent launch) sit beside this one and
  // prefetch its own weights while this one drains.
#ifndef NF_GEMM_SWAP_KB
#define NF_GEMM_SWAP_KB NF_GEMM_BUDGET_KB
#endif
  // Gather (implicit-GEMM conv) kernels may trade ring depth for L1: the
  // 3x3 taps re-read each input pixel up to 9 times.
  static constexpr int kMinKB = (3 * kStageBytes + kOutBytes + 1023) / 1024;
  static constexpr int kBudgetKB =
      GATHER == 1 ? (NF_GEMM_HALO_KB > kMinKB ? NF_GEMM_HALO_KB : kMinKB)
      : GATHER ? (NF_GEMM_GATHER_KB > kMinKB ? NF_GEMM_GATHER_KB : kMinKB)
      : KPT > 1 ? 225
      : BN >= 256 ? (PAIR ? NF_GEMM_PAIR_KB : 220)
                  : (SWAP ? (kStaged ? NF_GEMM_SWAP_KB : NF_GEMM_LITE_KB) : NF_GEMM_BUDGET_KB);
  static constexpr int kStages = (kBudgetKB * 1024 - kOutBytes) / kStageBytes;
  // two accumulator buffers; tcgen05.alloc takes a power of two >= 32
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                   : 2 * BN <= 256 ? 256 : 512;
  // folded-LN per-token (mean, rstd) of the B operand and of the residual
  static constexpr int kNormBytes =
      (SWAP && kStaged && !PAIR && !GATHER) ? (KPT > 1 ? 2 : 4) * BN * 4 : 0;
  // KPT > 1 leaves room for one (mean, rstd) pair: input OR residual fold
  static constexpr int kResNormOff = KPT > 1 ? 0 : 2 * BN;
  static constexpr size_t kBytes =
      1024 + size_t(kStages) * kStageBytes + kOutBytes + 512 + kNormBytes;
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kStages <= 32, "barrier array");
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

// The divisors the kernels use, from the extents (every launch path).
inline GemmParams gemm_params_finalize(GemmParams p) {
  auto pos = [](int v) { return v > 0 ? v : 1; };
  p.fd_splits = FastDiv::make(pos(p.splits));
  p.fd_ta = FastDiv::make(pos(p.tiles_a));
  p.fd_tb = FastDiv::make(pos(p.tiles_b));
  p.fd_cWo = FastDiv::make(pos(p.cWo));
  p.fd_cHo = FastDiv::make(pos(p.cHo));
  p.fd_cCg = FastDiv::make(pos(p.cCg));
  p.fd_cK = FastDiv::make(pos(p.cK));
  return p;
}

NF_DEVICE UnitCoord decode_unit(const GemmParams& p, int u, bool swap) {
  UnitCoord c;
  c.tile = p.fd_splits.div(u);
  c.s = u - c.tile * p.splits;
  // swapped: B (tokens) fastest; normal: A (token tiles) fastest, so CTAs
  // running concurrently share one weight tile in L2.
  if (swap) {
    const int q = p.fd_tb.div(c.tile);
    c.tb = c.tile - q * p.tiles_b;
    c.g = p.fd_ta.div(q);
    c.ta = q - c.g * p.tiles_a;
  } else {
    const int q = p.fd_ta.div(c.tile);
    c.ta = c.tile - q * p.tiles_a;
    c.g = p.fd_tb.div(q);
    c.tb = q - c.g * p.tiles_b;
  }
  c.kb0 = c.s * p.kb_per_split;
  c.kb1 = min(p.kb_total, c.kb0 + p.kb_per_split);
  return c;
}

// cp.async with zero-fill: copies `src_bytes` (0 or the chunk size) and
// fills the rest of the chunk with zeros.
template <int BYTES>
NF_DEVICE void cp_async_zfill(uint32_t dst, const void* src, int src_bytes) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
NF_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
NF_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int BN, bool SWAP, bool HAS_RES, int GATHER, bool PAIR, int KPT = 1>
__global__ void __launch_bounds__(gemm_threads<BN, GATHER>(), 1)
    k_grouped_gemm_tc(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_y,
                      const __grid_constant__ CUtensorMap map_r, GemmParams p) {
  using C = GemmCfg<BN, SWAP, PAIR, GATHER, KPT>;
  constexpr int kStages = C::kStages;
  static_assert(KPT == 1 || (KPT == 2 && SWAP && !PAIR && !GATHER), "multi-k-block stages");
  static_assert(!(PAIR && GATHER), "CTA pairs take TMA operands only");
  constexpr int kRowsA = PAIR ? 2 * kGemmBM : kGemmBM;  // A rows per unit
  constexpr int kEpiWarps = epi_warps<BN>();
  constexpr int kEpiThreads = 32 * kEpiWarps;
  constexpr int kColsPerThread = BN * 4 / kEpiWarps;  // columns each epilogue thread drains
  // Residual tiles arrive by TMA into the output staging buffer (same
  // swizzled layout as the result), so the epilogue adds them from smem.
  constexpr bool kResTma = HAS_RES && C::kStaged;
  // the residual tile is requested at the top of the unit, ahead of the
  // accumulator
  constexpr int EC = BN < 32 ? BN : 32;  // epilogue column chunk
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
  uint64_t* rbar = tempty + 2;  // [2] residual tile (per epilogue half on token-row tiles)
  uint64_t* hbar = rbar + 2;  // [2] halo buffers (GATHER == 1)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hbar + 2);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
  float* sNorm = reinterpret_cast<float*>(sOut + C::kOutBytes + 512);  // C::kNormBytes
  constexpr bool kFold = C::kNormBytes > 0;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) NF_TRACE(0);
  // A pair walks the unit list together: cluster index / cluster count.
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int ubase = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int ustride = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (C::kStaged) tma_prefetch_desc(&map_y);
    if (kResTma) tma_prefetch_desc(&map_r);
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    mbar_init(&hbar[0], 1);
    mbar_init(&hbar[1], 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], GATHER ? 1 + kGatherThreads : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 : kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_slot, C::kTmemCols);
    else tmem_alloc(tmem_slot, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the peer signals our barriers after this
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) NF_TRACE(1);
  // Let the next kernel in the stream get scheduled as SMs free up; it waits
  // on griddepcontrol.wait for this grid's results before reading them.
  grid_dependents_launch();

  if (warp == 0) {
    if (lane == 0) {
      // Weights stream once: evict-first. Activations are re-read by sibling
      // CTAs: evict-last keeps them in L2.
      const uint64_t hint_a = SWAP ? kEvictFirst : kEvictLast;
      const uint64_t hint_b = SWAP ? kEvictLast : kEvictFirst;
      // Pair: the leader's full barrier counts both CTAs' bytes.
      constexpr uint32_t kTx = GATHER ? (SWAP ? C::kABytes : C::kBBytes)
                                      : (PAIR ? 2 : 1) * C::kStageBytes;
      auto tload = [&](uint8_t* dst, const CUtensorMap* map, int stage, int c0, int c1, int c2,
                       uint64_t hint) {
        if constexpr (PAIR) tma_load_3d_pair(dst, map, &full[stage], c0, c1, c2, hint);
        else tma_load_3d(dst, map, &full[stage], c0, c1, c2, hint);
      };
      auto arm = [&](int stage) {
        if (leader) mbar_arrive_expect_tx(&full[stage], kTx);
      };
      auto a_row = [&](const UnitCoord& c) { return c.ta * kRowsA + int(rank) * kGemmBM; };
      auto b_row = [&](const UnitCoord& c) { return c.tb * BN + (PAIR ? int(rank) * (BN / 2) : 0); };
      auto load_w = [&](int stage, const UnitCoord& c, int kb) {
        if constexpr (KPT > 1) {  // 4-D maps (64, rows, K/64, G): KPT k-blocks per box
          tma_load_4d(sA + stage * C::kABytes, &map_a, &full[stage], 0, a_row(c), kb, c.g,
                      hint_a);
          return;
        }
        if (SWAP)
          tload(sA + stage * C::kABytes, &map_a, stage, kb * kGemmBK, a_row(c), c.g, hint_a);
        else
          tload(sB + stage * C::kBBytes, &map_b, stage, kb * kGemmBK, b_row(c), c.g, hint_b);
      };
      auto load_x = [&](int stage, const UnitCoord& c, int kb) {
        if (GATHER) return;  // gathered by warps 6..9
        if constexpr (KPT > 1) {
          tma_load_4d(sB + stage * C::kBBytes, &map_b, &full[stage], 0, b_row(c), kb, c.g,
                      hint_b);
          return;
        }
        if (SWAP)
          tload(sB + stage * C::kBBytes, &map_b, stage, kb * kGemmBK, b_row(c), c.g, hint_b);
        else
          tload(sA + stage * C::kABytes, &map_a, stage, kb * kGemmBK, a_row(c), c.g, hint_a);
      };
      int it = 0;
      int u = ubase;
      int pre = 0;
      int ready_x = -1;  // linked launches: last instance whose inputs were acquired
      auto wait_x = [&](const UnitCoord& c) {
        const int inst = c.g / p.link_gpi;
        if (inst != ready_x) {
          wait_counter(p.dep_x + inst, p.dep_x_target);
          ready_x = inst;
        }
      };
      if (u < p.units) {
        // Under programmatic dependent launch the weights do not depend on
        // the previous kernel but the activations do: request the first
        // ring's worth of weight tiles before the dependency wait.
        const UnitCoord c = decode_unit(p, u, SWAP);
        pre = min(kStages, (c.kb1 - c.kb0 + KPT - 1) / KPT);
        for (int i = 0; i < pre; ++i) {
          arm(i);
          load_w(i, c, c.kb0 + i * KPT);
        }
        if (!GATHER) {
          if (p.dep_x) wait_x(c);
          else grid_dependency_wait();
        }
        for (int i = 0; i < pre; ++i) load_x(i, c, c.kb0 + i * KPT);
        it = pre;
      } else if (!GATHER && !p.dep_x) {
        grid_dependency_wait();
      }
      for (; u < p.units; u += ustride) {
        const UnitCoord c = decode_unit(p, u, SWAP);
        if (!GATHER && p.dep_x && pre == 0) wait_x(c);
        for (int kb = c.kb0 + pre * KPT; kb < c.kb1; kb += KPT, ++it) {
          const int stage = it % kStages;
          {
            NF_WAIT_BEGIN();
            mbar_wait(&empty[stage], ((it / kStages) & 1) ^ 1);
            NF_WAIT_END(0);
          }
          arm(stage);
          load_w(stage, c, kb);
          load_x(stage, c, kb);
        }
        pre = 0;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16_f32(kRowsA, BN);
    int it = 0, local = 0;
    // Pair: only the leader issues (M=256 over both CTAs' smem / TMEM).
    for (int u = leader ? ubase : p.units; u < p.units; u += ustride, ++local) {
      const UnitCoord c = decode_unit(p, u, SWAP);
      const int acc = local & 1;
      {
        NF_WAIT_BEGIN();
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        if (lane == 0) NF_WAIT_END(2);
      }
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
      for (int kb = c.kb0; kb < c.kb1; kb += KPT, ++it) {
        const int stage = it % kStages;
        {
          NF_WAIT_BEGIN();
          mbar_wait(&full[stage], (it / kStages) & 1);
          if (lane == 0) NF_WAIT_END(1);
        }
        tc_fence_after();
        if (lane == 0 && it == 0) NF_TRACE(2);
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < KPT; ++h) {
            if (kb + h >= c.kb1) break;  // a split's range ends mid-stage
            const uint32_t a_base = smem_u32(sA + stage * C::kABytes) + h * (C::kABytes / KPT);
            const uint32_t b_base = smem_u32(sB + stage * C::kBBytes) + h * (C::kBBytes / KPT);
#pragma unroll
            for (int kk = 0; kk < kGemmBK / 16; ++kk) {
              if constexpr (PAIR)
                umma_f16_ss_pair(d_tmem, make_sw128_kmajor_desc(a_base + kk * 32),
                                 make_sw128_kmajor_desc(b_base + kk * 32), idesc,
                                 (kb + h != c.kb0 || kk != 0) ? 1u : 0u);
              else
                umma_f16_ss(d_tmem, make_sw128_kmajor_desc(a_base + kk * 32),
                            make_sw128_kmajor_desc(b_base + kk * 32), idesc,
                            (kb + h != c.kb0 || kk != 0) ? 1u : 0u);
            }
          }
          // frees the smem slot (both CTAs' halves) once these MMAs retire
          if constexpr (PAIR) umma_commit_pair(&empty[stage]);
          else umma_commit(&empty[stage]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if constexpr (PAIR) umma_commit_pair(&tfull[acc]);
        else umma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
    if (lane == 0) NF_TRACE(3);
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;         // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;  // accumulator row == TMEM lane
    const int etid = threadIdx.x - 64;    // 0 .. kEpiThreads-1
    const int col0 = ((warp - 2) >> 2) * kColsPerThread;  // this thread's column range
    // The residual tile and folded-LN statistics are fetched by these
    // threads ahead of the accumulator: order them after the previous launch
    // like the producer's operand loads.
    if ((kResTma || (kFold && (p.nin_stats || p.nres_stats))) && !p.dep_x)
      grid_dependency_wait();
    int ready_r = -1;  // linked launches: last instance whose residual was acquired
    // linked launches: this unit's output tile is stored (the caller made the
    // writes complete and ordered them before this thread): count it
    auto publish = [&](int g) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      publish_count(p.done + g / p.link_gpi);
    };
    const uint32_t stage_base = smem_u32(sOut);
    // Token-row staged tiles store progressively: each half of the epilogue
    // warps (4 warps = 128 rows x kColsPerThread columns) TMA-stores every
    // 64-column block as soon as its rows are staged, so the stores stream
    // out while the next block's math runs, and the staging of the next unit
    // waits only for this half's own stores (no whole-tile read-out between
    // units: that serialisation cost ~35% of the short-K GEMMs at large T).
    constexpr bool kProg = !SWAP && C::kStaged;
    constexpr int kHalfBlocks = kColsPerThread / kOutBlock;
    static_assert(!kProg || kColsPerThread % kOutBlock == 0, "half = whole 64-column blocks");
    const int half = (warp - 2) >> 2;
    const bool issuer = (etid & 127) == 0;
    uint64_t* my_rbar = kProg ? &rbar[half] : &rbar[0];
    uint32_t res_phase = 0;
    int local = 0;
    // Hand an accumulator buffer back to the MMA issuer (the leader's barrier
    // collects one arrival per CTA in pair mode).
    auto release_acc = [&](int acc) {
      tc_fence_before();
      if constexpr (PAIR) {
        named_bar_sync(1, kEpiThreads);
        if (etid == 0) mbar_arrive_leader(&tempty[acc]);
      } else {
        mbar_arrive(&tempty[acc]);
      }
    };
    const bool fold_in = kFold && p.nin_stats != nullptr;
    const bool fold_res = kFold && kResTma && p.nres_stats != nullptr;
    for (int u = ubase; u < p.units; u += ustride, ++local) {
      const UnitCoord c = decode_unit(p, u, SWAP);
      const int acc = local & 1;
      // Epilogue operands that do not depend on the accumulator are fetched
      // while the main loop runs: the residual tile (the previous unit's
      // store has finished reading the staging buffer: bulk_wait_read0 +
      // barrier at the end of the unit) and the folded-LN statistics.
      auto issue_residual = [&]() {
        if constexpr (kProg) {
          if (issuer) {  // this half's blocks (its previous stores were read)
            const int m0r = c.ta * kRowsA + int(rank) * kGemmBM, n0r = c.tb * BN;
            mbar_arrive_expect_tx(my_rbar, kHalfBlocks * kGemmBM * 128);
#pragma unroll
            for (int i = 0; i < kHalfBlocks; ++i) {
              const int b = half * kHalfBlocks + i;
              tma_load_3d(sOut + b * kGemmBM * 128, &map_r, my_rbar, n0r + b * kOutBlock, m0r,
                          c.g, kEvictFirst);
            }
          }
        } else if (etid == 0) {
          const int m0r = c.ta * kRowsA + int(rank) * kGemmBM, n0r = c.tb * BN;
          mbar_arrive_expect_tx(rbar, C::kOutBytes);
          if constexpr (KPT > 1) {
            // 4-D map (64, T, N/64, G): the tile's two 64-feature blocks in one box
            tma_load_4d(sOut, &map_r, rbar, 0, n0r, m0r / kOutBlock, c.g, kEvictFirst);
          } else {
#pragma unroll
            for (int b = 0; b < kGemmBM / kOutBlock; ++b)
              tma_load_3d(sOut + b * BN * 128, &map_r, rbar, m0r + b * kOutBlock, n0r, c.g,
                          kEvictFirst);
          }
        }
      };
      if constexpr (kProg) {
        // this half's staging blocks are free once its previous stores read them
        if (issuer) bulk_wait_read0();
        if constexpr (!kResTma) named_bar_sync(3 + half, 128);
      }
      if (HAS_RES && p.dep_r && c.g / p.link_gpi != ready_r) {
        // linked: the residual's producer stored this instance's tiles
        if (etid == 0) wait_counter(p.dep_r + c.g / p.link_gpi, p.dep_r_target);
        named_bar_sync(1, kEpiThreads);
        ready_r = c.g / p.link_gpi;
      }
      if constexpr (kResTma) issue_residual();
      if constexpr (kFold) {
        if (fold_in || fold_res) {
          // (mean, rstd) of this tile's BN tokens, once per unit
          const int n0s = c.tb * BN;
          for (int t = etid; t < BN; t += kEpiThreads) {
            const int tok = n0s + t < p.rows_b ? n0s + t : p.rows_b - 1;
            if (fold_in) {
              const float2 m = fold_stats(p.nin_stats, p.nin_parts, p.rows_b, c.g, tok,
                                          p.nin_inv_d, p.nin_eps);
              sNorm[t] = m.x;
              sNorm[BN + t] = m.y;
            }
            if (fold_res) {
              const float2 m = fold_stats(p.nres_stats, p.nres_parts, p.rows_b, c.g, tok,
                                          p.nres_inv_d, p.nres_eps);
              sNorm[C::kResNormOff + t] = m.x;
              sNorm[C::kResNormOff + BN + t] = m.y;
            }
          }
          named_bar_sync(1, kEpiThreads);
        }
      }
      // token-row tiles: the bias of the next 32 columns, one value per lane
      // (broadcast to the row threads by shuffles), loaded a chunk ahead --
      // the first during the main loop: a bias load issued right before its
      // use was the epilogue's top stall (long scoreboard), and a register
      // per lane fits where a float4 x 8 per thread would spill.
      constexpr bool kBiasAhead = !SWAP && EC == 32;
      float bpre = 0.f;
      // an unconditional load (clamped index, a zero word when there is no
      // bias): a select on the loaded value made the prefetch wait for it
      // right away (the FF1 epilogue's top stall in ncu)
      const float* bsrc = p.bias ? p.bias + int64_t(c.g) * p.features : g_zero_bias;
      const int blast = p.bias ? p.rows_b - 1 : 0;
      auto bias_chunk = [&](int cc_) {
        const int f = c.tb * BN + cc_ + lane;
        bpre = __ldg(bsrc + (f < blast ? f : blast));  // columns past N are not stored
      };
      if constexpr (kBiasAhead) bias_chunk(((warp - 2) >> 2) * kColsPerThread);
      // swapped tiles: this thread's feature row constants, loaded ahead too
      float hb = 0.f, hcs = 0.f, hgm = 0.f, hbt = 0.f;
      if constexpr (SWAP) {
        const int feat = c.ta * kRowsA + int(rank) * kGemmBM + row;
        if (feat < p.rows_a) {
          const int64_t fi = int64_t(c.g) * p.features + feat;
          if (p.bias) hb = __ldg(p.bias + fi);
          if (fold_in) hcs = __ldg(p.nin_colsum + fi);
          if (fold_res) {
            hgm = __ldg(p.nres_gamma + fi);
            hbt = __ldg(p.nres_beta + fi);
          }
        }
      }
      {
        NF_WAIT_BEGIN();
        mbar_wait(&tfull[acc], (local >> 1) & 1);
        if (etid == 0) NF_WAIT_END(3);
      }
      NF_WAIT_BEGIN();  // epilogue busy: accumulator ready -> buffer released
      tc_fence_after();
      if (etid == 0 && local == 0) NF_TRACE(4);
      const uint32_t t_row = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      const int m0 = c.ta * kRowsA + int(rank) * kGemmBM, n0 = c.tb * BN;
      const int wtile = PAIR ? c.tile * 2 + int(rank) : c.tile;  // this CTA's 128-row tile
      float* part = nullptr;
      if (p.splits > 1) {
        // Publish this split's fp32 partial; the last arriver reduces.
        // Partials are stored column-major over TMEM lanes ([col][row]):
        // each warp store covers one contiguous 128-byte line.
        part = p.ws + (int64_t(wtile) * p.splits) * kGemmBM * BN;
        float* mine = part + int64_t(c.s) * kGemmBM * BN + row;
#pragma unroll 1
        for (int cc = col0; cc < col0 + kColsPerThread; cc += EC) {
          uint32_t r[EC];
          tmem_ld_cols<EC>(t_row + uint32_t(cc), r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < EC; ++j) __stcg(mine + (cc + j) * kGemmBM, __uint_as_float(r[j]));
        }
        named_bar_sync(1, kEpiThreads);
        if (etid == 0) *last_flag = (arrive_acq_rel(p.counters + wtile) == unsigned(p.splits - 1));
        named_bar_sync(1, kEpiThreads);
        if (!*last_flag) {
          release_acc(acc);
          if constexpr (kResTma) {
            mbar_wait(my_rbar, res_phase);  // its residual tile landed unused
            res_phase ^= 1u;
          }
          continue;
        }
      }
      const __nv_bfloat16* res =
          HAS_RES ? reinterpret_cast<const __nv_bfloat16*>(p.residual) +
                        int64_t(c.g) * p.out_gstride
                  : nullptr;
      if constexpr (kResTma) {
        mbar_wait(my_rbar, res_phase);  // issued before the accumulator wait
        res_phase ^= 1u;
      }
      const float* bias = p.bias ? p.bias + int64_t(c.g) * p.features : nullptr;
      // TMEM loads run one chunk ahead: chunk cc+EC is requested before
      // chunk cc is processed, so its latency hides behind the epilogue math
      // (the consumer of a just-issued tcgen05.ld was the top stall).
      // (Not in the 448-thread gather kernels: their 128-register budget
      // would spill the second chunk.)
      // Token-row tiles only: on swapped batch-1 tiles the prefetch measured
      // slower (BERT-base N=8 B=1 0.653 -> 0.697 ms).
      constexpr bool kLdAhead = GATHER == 0 && !SWAP;
      uint32_t rnext[EC];
      if constexpr (kLdAhead) {
        tmem_ld_cols<EC>(t_row + uint32_t(col0), rnext);
        tmem_ld_wait();
      }
#pragma unroll 1
      for (int cc = col0; cc < col0 + kColsPerThread; cc += EC) {
        if constexpr (!kLdAhead) {
          tmem_ld_cols<EC>(t_row + uint32_t(cc), rnext);
          tmem_ld_wait();
        }
        float v[EC];
#pragma unroll
        for (int j = 0; j < EC; ++j) v[j] = __uint_as_float(rnext[j]);
        if (kLdAhead && cc + EC < col0 + kColsPerThread)
          tmem_ld_cols<EC>(t_row + uint32_t(cc + EC), rnext);
        float bcur = 0.f;
        if constexpr (kBiasAhead) {
          bcur = bpre;
          if (cc + EC < col0 + kColsPerThread) bias_chunk(cc + EC);
        }
        if (p.splits > 1) {
          // Deterministic reduction: splits summed in index order.
          float sum[EC];
#pragma unroll
          for (int j = 0; j < EC; ++j) sum[j] = 0.f;
          for (int s2 = 0; s2 < p.splits; ++s2) {
            if (s2 == c.s) {
#pragma unroll
              for (int j = 0; j < EC; ++j) sum[j] += v[j];
            } else {
              const float* src = part + int64_t(s2) * kGemmBM * BN + row + cc * kGemmBM;
#pragma unroll
              for (int j = 0; j < EC; ++j) sum[j] += __ldcg(src + j * kGemmBM);
            }
          }
#pragma unroll
          for (int j = 0; j < EC; ++j) v[j] = sum[j];
        }
        if (!SWAP) {
          // Thread = token row; EC consecutive features n0+cc ...
          const int tok = m0 + row;
          const int f0 = n0 + cc;
          if (kBiasAhead && bias) {
#pragma unroll
            for (int j = 0; j < EC; ++j) v[j] += __shfl_sync(0xffffffffu, bcur, j);
          } else if (bias) {
            if (f0 + EC <= p.rows_b) {
#pragma unroll
              for (int j = 0; j < EC; j += 4) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + f0 + j));
                v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < EC; ++j)
                if (f0 + j < p.rows_b) v[j] += __ldg(bias + f0 + j);
            }
          }
          if constexpr (kResTma) {
#pragma unroll
            for (int q = 0; q < EC / 8; ++q) {
              uint32_t w4[4];
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(w4[0]), "=r"(w4[1]), "=r"(w4[2]), "=r"(w4[3])
                           : "r"(stage_base + stage_offset(row, cc + 8 * q, kGemmBM)));
              float r8[8];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                r8[2 * e] = __uint_as_float(w4[e] << 16);
                r8[2 * e + 1] = __uint_as_float(w4[e] & 0xffff0000u);
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) v[8 * q + e] += r8[e];
            }
          } else if (HAS_RES && tok < p.rows_a) {
            const __nv_bfloat16* rp = res + int64_t(tok) * p.out_ld + f0;
#pragma unroll
            for (int q = 0; q < EC / 4; ++q)
              if (f0 + 4 * q + 4 <= p.rows_b) {
                const uint2 u2 = *reinterpret_cast<const uint2*>(rp + 4 * q);
                v[4 * q] += __uint_as_float(u2.x << 16);
                v[4 * q + 1] += __uint_as_float(u2.x & 0xffff0000u);
                v[4 * q + 2] += __uint_as_float(u2.y << 16);
                v[4 * q + 3] += __uint_as_float(u2.y & 0xffff0000u);
              }
          }
          apply_act<GATHER != 0>(p.act, v);
          if constexpr (C::kStaged) {
#pragma unroll
            for (int q = 0; q < EC / 8; ++q) {
              const uint32_t w0 = pack_bf16x2(v[8 * q], v[8 * q + 1]);
              const uint32_t w1 = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
              const uint32_t w2 = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
              const uint32_t w3 = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
              st_shared_v4(stage_base + stage_offset(row, cc + 8 * q, kGemmBM), w0, w1, w2, w3);
            }
          } else if (tok < p.rows_a) {
            // Narrow tiles (grouped convs with 4..32 channels per group):
            // each thread writes its row's features straight to HBM.
            __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(p.y_direct) +
                                int64_t(c.g) * p.out_gstride + int64_t(tok) * p.out_ld + f0;
#pragma unroll
            for (int q = 0; q < EC / 4; ++q)
              if (f0 + 4 * q + 4 <= p.rows_b) {
                uint2 u2;
                u2.x = pack_bf16x2(v[4 * q], v[4 * q + 1]);
                u2.y = pack_bf16x2(v[4 * q + 2], v[4 * q + 3]);
                *reinterpret_cast<uint2*>(yp + 4 * q) = u2;
              }
          }
        } else {
          // Thread = feature row; 32 consecutive tokens. Neighbouring lanes
          // (features f, f^1) swap one value so each lane stores a packed
          // bf16 pair of adjacent features: 16 32-bit smem stores per chunk.
          const int feat = m0 + row;
          const float b = hb, cs = hcs, gm = hgm, bt = hbt;
          if constexpr (kFold) {
            if (fold_in) {
#pragma unroll
              for (int j = 0; j < EC; j += 4) {
                const float4 mu = *reinterpret_cast<const float4*>(sNorm + cc + j);
                const float4 rs = *reinterpret_cast<const float4*>(sNorm + BN + cc + j);
                v[j] = rs.x * fmaf(-mu.x, cs, v[j]);
                v[j + 1] = rs.y * fmaf(-mu.y, cs, v[j + 1]);
                v[j + 2] = rs.z * fmaf(-mu.z, cs, v[j + 2]);
                v[j + 3] = rs.w * fmaf(-mu.w, cs, v[j + 3]);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < EC; ++j) {
            v[j] += b;
            if constexpr (HAS_RES && !C::kStaged) {
              // lanes = consecutive features of one token: coalesced
              const int tok = n0 + cc + j;
              if (feat < p.rows_a && tok < p.rows_b)
                v[j] += __bfloat162float(res[int64_t(tok) * p.out_ld + feat]);
            }
            if constexpr (kResTma) {
              uint16_t h;
              asm volatile("ld.shared.u16 %0, [%1];"
                           : "=h"(h)
                           : "r"(stage_base + stage_offset(cc + j, row, BN)));
              float r = __uint_as_float(uint32_t(h) << 16);
              if constexpr (kFold) {
                if (fold_res)
                  r = fmaf((r - sNorm[C::kResNormOff + cc + j]) * sNorm[C::kResNormOff + BN + cc + j],
                           gm, bt);
              }
              v[j] += r;
            }
          }
          apply_act<GATHER != 0>(p.act, v);
          if constexpr (kResTma) __syncwarp();  // partner lanes read before the pair stores
          const bool odd = lane & 1;
          const int feven = row & ~1;
#pragma unroll
          for (int j = 0; j < EC; j += 2) {
            const float send = odd ? v[j] : v[j + 1];
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const uint32_t packed = odd ? pack_bf16x2(recv, v[j + 1]) : pack_bf16x2(v[j], recv);
            const int t = cc + j + (odd ? 1 : 0);
            if constexpr (C::kStaged) {
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(stage_base +
                                                             stage_offset(t, feven, BN)),
                           "r"(packed)
                           : "memory");
            } else {
              // even lanes: token t, odd lanes: token t+1; each half-warp
              // writes 64 contiguous bytes of one token row.
              const int tok = n0 + t;
              const int f = m0 + feven;
              if (tok < p.rows_b && f < p.rows_a)
                *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(p.y_direct) +
                                             int64_t(c.g) * p.out_gstride +
                                             int64_t(tok) * p.out_ld + f) = packed;
            }
          }
        }
        if constexpr (kProg) {
          if ((cc + EC - col0) % kOutBlock == 0) {
            // this half finished a 64-column block: store it now
            fence_proxy_async_smem();
            named_bar_sync(3 + half, 128);
            if (issuer) {
              const int b = (cc + EC) / kOutBlock - 1;
              tma_store_3d(&map_y, sOut + b * kGemmBM * 128, n0 + b * kOutBlock, m0, c.g);
              bulk_commit();
            }
          }
        }
        if constexpr (kLdAhead) tmem_ld_wait();  // the next chunk's columns have landed
      }
      // All TMEM reads of this buffer are done: hand it back to the MMA warp.
      if (etid == 0) NF_WAIT_END(4);
      release_acc(acc);
      if constexpr (kProg) {
        if (p.splits > 1 && etid == 0) p.counters[wtile] = 0u;  // re-arm for the next launch
        if (p.done) {
          // both halves' stores complete, then one count for the tile
          if (issuer) bulk_wait0();
          named_bar_sync(1, kEpiThreads);
          if (etid == 0) publish(c.g);
        }
      } else if constexpr (C::kStaged) {
        fence_proxy_async_smem();
        named_bar_sync(1, kEpiThreads);
        if (etid == 0) {
          if (!SWAP) {
#pragma unroll
            for (int b = 0; b < BN / kOutBlock; ++b)
              tma_store_3d(&map_y, sOut + b * kGemmBM * 128, n0 + b * kOutBlock, m0, c.g);
          } else if constexpr (KPT > 1) {
            tma_store_4d(&map_y, sOut, 0, n0, m0 / kOutBlock, c.g);
          } else {
#pragma unroll
            for (int b = 0; b < kGemmBM / kOutBlock; ++b)
              tma_store_3d(&map_y, sOut + b * BN * 128, m0 + b * kOutBlock, n0, c.g);
          }
          bulk_commit();
          if (p.splits > 1) p.counters[wtile] = 0u;  // re-arm for the next launch
        }
        if constexpr (kFold) {
          if (p.nout_stats) {
            // LN statistics of token t over this tile's 128 features, from the
            // bf16 values just staged (what the consumer will read), in one
            // pass of shifted sums: with the shift c = the token's first
            // feature, S1 = sum(x - c), S2 = sum((x - c)^2), the part's sum is
            // S1 + 128 c and its centred M2 = S2 - S1^2 / 128. |x - c| is on
            // the scale of the spread, not of the mean, so the subtraction
            // does not cancel when |mean| >> std (no E[x^2] - mean^2).
            // Lane pair (2t, 2t+1) takes token t's two 64-feature blocks; the
            // swizzle spreads each 16-byte chunk read over all banks.
            constexpr int kBlocks = kGemmBM / kOutBlock;  // 2
            constexpr int kPerTok = kEpiThreads / BN;      // threads per token
            static_assert(kPerTok == 1 || kPerTok == kBlocks, "stats split");
            const int t = kPerTok == 1 ? etid : etid >> 1;
            float s1 = 0.f, s2 = 0.f, shift = 0.f;
            if (t < BN) {
              uint16_t h0;
              asm volatile("ld.shared.u16 %0, [%1];"
                           : "=h"(h0)
                           : "r"(stage_base + uint32_t(t * 128) + (uint32_t(t & 7) << 4)));
              shift = __uint_as_float(uint32_t(h0) << 16);  // feature 0 of token t
#pragma unroll
              for (int bb = 0; bb < kBlocks / kPerTok; ++bb) {
                const int b = kPerTok == 1 ? bb : (etid & 1);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  uint32_t w4[4];
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(w4[0]), "=r"(w4[1]), "=r"(w4[2]), "=r"(w4[3])
                               : "r"(stage_base + uint32_t(b * BN * 128 + t * 128) +
                                     (uint32_t(q ^ (t & 7)) << 4)));
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float lo = __uint_as_float(w4[e] << 16) - shift;
                    const float hi = __uint_as_float(w4[e] & 0xffff0000u) - shift;
                    s1 += lo + hi;
                    s2 = fmaf(lo, lo, fmaf(hi, hi, s2));
                  }
                }
              }
            }
            if constexpr (kPerTok > 1) {
              s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
              s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
            }
            const float s = fmaf(float(kGemmBM), shift, s1);
            const float m2 = fmaxf(s2 - s1 * s1 * (1.0f / float(kGemmBM)), 0.f);
            if (t < BN && (kPerTok == 1 || (etid & 1) == 0) && n0 + t < p.rows_b)
              __stcg(p.nout_stats + (int64_t(c.g) * p.tiles_a + c.ta) * p.rows_b + n0 + t,
                     make_float2(s, m2));
          }
        }
        if (etid == 0) {
          if (p.done) {
            bulk_wait0();  // the tile is in global memory (and the staging free)
            publish(c.g);
          } else {
            bulk_wait_read0();  // staging reusable
          }
        }
        named_bar_sync(1, kEpiThreads);
      } else {
        if (p.splits > 1 || p.done) {
          named_bar_sync(1, kEpiThreads);  // every thread's direct stores issued
          if (etid == 0 && p.splits > 1) p.counters[wtile] = 0u;
          if (etid == 0 && p.done) publish(c.g);
        }
      }
    }
    if constexpr (kProg) {
      if (issuer) bulk_wait_read0();  // the staging must outlive this half's last stores
    }
    if (etid == 0) NF_TRACE(5);
  } else if constexpr (GATHER == 1) {
    // --------------------- halo im2col (conv, pixels on M) ---------------------
    // One TMA box per 128-pixel tile: cg channels x halo_w columns x the
    // input rows the tile's taps touch (zero-filled outside the image), double
    // buffered across units; each k-block's im2col rows are then built with
    // 16-byte shared-memory copies (every input pixel leaves HBM / L2 once
    // per tile instead of once per tap).
    const int gt = threadIdx.x - (64 + kEpiThreads);
    const int j = gt & 7;   // 16-byte chunk of the 128-byte operand row
    const int rb = gt >> 3; // rows rb + 16 * i
    uint8_t* halo = sOut + C::kOutBytes + 1024;
    const int taps = p.cK * p.cK;
    const int rows = p.rows_a;
    const int hw = p.halo_w;
    auto issue_halo = [&](int u, int hb) {
      const UnitCoord c = decode_unit(p, u, false);
      const int oh_lo = p.fd_cWo.div(c.ta * kGemmBM);
      mbar_arrive_expect_tx(&hbar[hb], p.halo_tx);
      // the box's first channel must sit on a 16-byte boundary: 4-channel
      // groups start at the even-group boundary and index +4 inside the pixel
      tma_load_4d(halo + hb * p.halo_bytes, &map_a, &hbar[hb], (c.g * p.cCg) & ~7, -p.cP,
                  oh_lo * p.cS - p.cP, 0, kEvictNormal);
    };
    // Linked launches: a halo is requested once its instance's input tiles
    // are stored. The next unit's halo is prefetched only if that instance
    // is already complete (non-blocking check); otherwise it is requested
    // (blocking) when its unit starts, so a late instance never stalls the
    // current unit's gather.
    auto inst_ready = [&](int u, bool block) {
      const int inst = decode_unit(p, u, false).g / p.link_gpi;
      if (block) {
        wait_counter(p.dep_x + inst, p.dep_x_target);
        return true;
      }
      return counter_ready(p.dep_x + inst, p.dep_x_target);
    };
    bool halo_issued = true;  // the current unit's halo was requested (gt == 0)
    if (!p.dep_x) grid_dependency_wait();
    if (gt == 0 && int(blockIdx.x) < p.units) {
      if (p.dep_x) inst_ready(blockIdx.x, true);
      issue_halo(blockIdx.x, 0);
    }
    int it = 0, local = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++local) {
      const int hb = local & 1;
      if (gt == 0 && !halo_issued) {  // its prefetch was skipped: request it now
        inst_ready(u, true);
        fence_proxy_async_smem();  // generic reads of that buffer (two units ago) done
        issue_halo(u, hb);
      }
      if (gt == 0) {
        halo_issued = false;
        if (u + int(gridDim.x) < p.units && (!p.dep_x || inst_ready(u + gridDim.x, false))) {
          fence_proxy_async_smem();  // generic reads of that buffer (previous unit) done
          issue_halo(u + gridDim.x, hb ^ 1);
          halo_issued = true;
        }
      }
      const UnitCoord c = decode_unit(p, u, false);
      const int p0 = c.ta * kGemmBM;
      const int oh_lo = p.fd_cWo.div(p0);
      int hoff[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int pix = p0 + rb + 16 * i;
        const int oh = p.fd_cWo.div(pix), ow = pix - oh * p.cWo;
        hoff[i] = pix < rows ? ((oh - oh_lo) * p.cS * hw + ow * p.cS) : -1;
      }
      const uint32_t hsrc = smem_u32(halo + hb * p.halo_bytes) + uint32_t(((c.g * p.cCg) & 7) * 2);
      mbar_wait(&hbar[hb], uint32_t(local >> 1) & 1u);
      for (int kb = c.kb0; kb < c.kb1; ++kb, ++it) {
        const int stage = it % kStages;
        mbar_wait(&empty[stage], ((it / kStages) & 1) ^ 1);
        const int k0 = kb * kGemmBK + j * 8;
        const uint32_t sbase = smem_u32(sA + stage * C::kABytes);
        if (p.cCg >= 8) {
          // chunk j = K elements [k0, k0+8) of one tap: one 16-byte copy per row
          const int tap = p.fd_cCg.div(k0);
          const int ch = k0 - tap * p.cCg;
          const int kh = p.fd_cK.div(tap);
          const int tap_off = (kh * hw + (tap - kh * p.cK)) * p.halo_cpp + ch;
          const bool tap_ok = tap < taps;
          // all eight 16-byte reads first, then the eight writes: one
          // shared-memory latency per k-block instead of eight in series
          uint32_t v[8][4];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0;
            if (tap_ok && hoff[i] >= 0)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3])
                           : "r"(hsrc + uint32_t((hoff[i] * p.halo_cpp + tap_off) * 2)));
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = rb + 16 * i;
            st_shared_v4(sbase + uint32_t(r * 128) + (uint32_t(j ^ (r & 7)) << 4), v[i][0],
                         v[i][1], v[i][2], v[i][3]);
          }
        } else {
          // 4-channel groups (padded stem): two taps per 16-byte chunk
          int off[2];
          bool okh[2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int tap = p.fd_cCg.div(k0 + hh * 4);
            const int kh = p.fd_cK.div(tap);
            off[hh] = (kh * hw + (tap - kh * p.cK)) * p.halo_cpp;
            okh[hh] = tap < taps;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = rb + 16 * i;
            uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
            if (hoff[i] >= 0) {
              const uint32_t pix = hsrc + uint32_t(hoff[i] * p.halo_cpp * 2);
              if (okh[0])
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                             : "=r"(v0), "=r"(v1)
                             : "r"(pix + uint32_t(off[0] * 2)));
              if (okh[1])
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                             : "=r"(v2), "=r"(v3)
                             : "r"(pix + uint32_t(off[1] * 2)));
            }
            st_shared_v4(sbase + uint32_t(r * 128) + (uint32_t(j ^ (r & 7)) << 4), v0, v1, v2, v3);
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&full[stage]);
      }
      named_bar_sync(2, kGatherThreads);  // everyone is done with halo buffer hb
    }
  } else if constexpr (GATHER != 0) {
    // ------------------------ im2col gather (conv) ------------------------
    constexpr int R = SWAP ? BN : kGemmBM;  // activation rows per tile
    constexpr int CPR = 128 / GATHER;       // chunks per 128-byte row
    constexpr int RPP = kGatherThreads / CPR;
    constexpr int PASSES = R / RPP;
    constexpr int CE = GATHER / 2;           // channels per chunk
    // Arrivals trail the issue by LAG iterations; LAG < kStages or the
    // producer would wait on a slot whose fill it has not yet published.
    constexpr int LAG = kGatherLag < kStages - 1 ? kGatherLag : kStages - 1;
    const int gt = threadIdx.x - (64 + kEpiThreads);
    const int j = gt % CPR;
    const int r0 = gt / CPR;
    const uint32_t act_smem = smem_u32(SWAP ? sB : sA);
    constexpr uint32_t kActBytes = SWAP ? C::kBBytes : C::kABytes;
    // swizzled byte offset of chunk j within a row r (SWIZZLE_128B)
    const uint32_t jb = uint32_t(j * GATHER);
    const int taps = p.cK * p.cK;
    const int rows = SWAP ? p.rows_b : p.rows_a;
    if (!p.dep_x) grid_dependency_wait();
    int it = 0, ready = -1;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const UnitCoord c = decode_unit(p, u, SWAP);
      if (p.dep_x && c.g / p.link_gpi != ready) {
        // linked: this instance's input tiles are stored
        if (gt == 0) wait_counter(p.dep_x + c.g / p.link_gpi, p.dep_x_target);
        named_bar_sync(2, kGatherThreads);
        ready = c.g / p.link_gpi;
      }
      const int row0 = SWAP ? c.tb * BN : c.ta * kGemmBM;
      const __nv_bfloat16* xg = p.cx + int64_t(c.g) * p.cCg;
      int pix_off[PASSES], ih0[PASSES], iw0[PASSES];
#pragma unroll
      for (int i = 0; i < PASSES; ++i) {
        const int pix = row0 + r0 + RPP * i;
        const int t2 = p.fd_cWo.div(pix);
        const int ow = pix - t2 * p.cWo;
        const int n = p.fd_cHo.div(t2);
        const int oh = t2 - n * p.cHo;
        ih0[i] = pix < rows ? oh * p.cS - p.cP : -(1 << 20);
        iw0[i] = ow * p.cS - p.cP;
        pix_off[i] = n * p.cH * p.cW;
      }
      for (int kb = c.kb0; kb < c.kb1; ++kb, ++it) {
        const int stage = it % kStages;
        mbar_wait(&empty[stage], ((it / kStages) & 1) ^ 1);
        const int k0 = kb * kGemmBK + j * CE;
        const int tap = p.fd_cCg.div(k0);
        const int ch = k0 - tap * p.cCg;
        const int kh = p.fd_cK.div(tap);
        const int kw = tap - kh * p.cK;
        const bool tap_ok = tap < taps;
        const uint32_t sbase = act_smem + uint32_t(stage) * kActBytes;
#pragma unroll
        for (int i = 0; i < PASSES; ++i) {
          const int r = r0 + RPP * i;
          const int ih = ih0[i] + kh, iw = iw0[i] + kw;
          const bool ok = tap_ok && ih >= 0 && ih < p.cH && iw >= 0 && iw < p.cW;
          const __nv_bfloat16* src =
              ok ? xg + (int64_t(pix_off[i]) + ih * p.cW + iw) * p.cC + ch : p.cx;
          const uint32_t dst =
              sbase + uint32_t(r * 128) + ((((jb >> 4) ^ uint32_t(r & 7)) << 4) | (jb & 15));
          cp_async_zfill<GATHER>(dst, src, ok ? GATHER : 0);
        }
        cp_async_commit();
        if (it >= LAG) {
          cp_async_wait<LAG>();
          fence_proxy_async_smem();
          mbar_arrive(&full[(it - LAG) % kStages]);
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int back = it - LAG < 0 ? 0 : it - LAG; back < it; ++back)
      mbar_arrive(&full[back % kStages]);
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the leader's MMAs into the peer's TMEM are done
  if (threadIdx.x == 0) NF_TRACE(6);
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, C::kTmemCols);
    else tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
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
                   int box_inner, int box_rows, int64_t row_stride, int64_t g_stride);

template <int BN, bool SWAP, bool HAS_RES, int GATHER = 0, bool PAIR = false, int KPT = 1>
static int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& my,
                     const CUtensorMap& mr, const GemmParams& p, int grid, cudaStream_t stream) {
  using C = GemmCfg<BN, SWAP, PAIR, GATHER, KPT>;
  auto kern = k_grouped_gemm_tc<BN, SWAP, HAS_RES, GATHER, PAIR, KPT>;
  const GemmParams pf = gemm_params_finalize(p);
  static SmemAttrOnce smem_attr;  // one per kernel instantiation, a bit per device
  smem_attr.set(kern, GATHER == 1 ? 232448 : int(C::kBytes));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm_threads<BN, GATHER>());
  cfg.dynamicSmemBytes = C::kBytes + (GATHER == 1 ? 1024 + 2 * size_t(p.halo_bytes) : 0);
  cfg.stream = stream;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  if (PAIR) {
    la[1].id = cudaLaunchAttributeClusterDimension;
    la[1].val.clusterDim.x = 2;
    la[1].val.clusterDim.y = 1;
    la[1].val.clusterDim.z = 1;
  }
  cfg.attrs = la;
  cfg.numAttrs = PAIR ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, my, mr, pf);
  return e == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

// Residual / no-residual instantiation (the activation is a kernel argument).
template <int BN, bool SWAP, int GATHER = 0, bool PAIR = false, int KPT = 1>
static int launch_tc_res(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& my,
                         const CUtensorMap& mr, const GemmParams& p, int grid,
                         cudaStream_t stream) {
  if (p.residual)
    return launch_tc<BN, SWAP, true, GATHER, PAIR, KPT>(ma, mb, my, mr, p, grid, stream);
  return launch_tc<BN, SWAP, false, GATHER, PAIR, KPT>(ma, mb, my, mr, p, grid, stream);
}

}  // namespace nf
