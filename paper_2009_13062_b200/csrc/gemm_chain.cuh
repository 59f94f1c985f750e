// Chained batch-1 merged Linears in ONE persistent launch (e.g. a BERT
// layer's attention projection -> FF1+GELU -> FF2). Each op is a swapped
// weight-streaming GEMM (the `k_grouped_gemm_tc<128, SWAP, *, 0, false, 2>`
// tile: weights fill the MMA's 128-row side, 128 tokens, two 64-wide k-blocks
// per TMA transaction). The ops' work units are concatenated (op-major,
// instance-major inside an op) and walked round-robin by one CTA per SM.
//
// Why: at batch 1 every launch pays ~5-8 us of fixed cost (launch, first
// cold TMA, epilogue tail; profiles/r01_bert8_timeline.txt) around a 2-6 us
// weight stream. Here the operand ring runs across op boundaries: a unit's
// WEIGHT tiles (independent of any activation) are requested as soon as ring
// slots free up, and only its ACTIVATION tiles wait for the producing op.
// Dependencies are per instance: op j's activation tiles of instance g wait
// until op j-1 has stored all of g's output tiles (a release counter per
// (op, g), bumped after each tile's TMA store completed); the epilogue waits
// likewise for the chain op its residual / LayerNorm statistics come from.
// Instances never read each other's rows.
//
// Forward progress: dependencies point to lower unit indices only and every
// CTA walks its units in increasing order with its producer at most one unit
// ahead of its MMA/epilogue, so the lowest unfinished unit is always
// runnable. All CTAs are co-resident (grid <= #SMs, one CTA per SM).
//
// Counters are zero at launch; the last CTA to exit re-arms them (every CTA
// has finished waiting by then), so the launch is CUDA-graph replayable --
// unless a later kernel waits on them (the next layer's fused QKV+attention
// starts instance g once FF2 has stored g's tiles): then the caller zeroes
// them before each forward.
//
// Replaces the reference's per-node `batch_matmul` calls
// (pkg/src/modelmerge/engine.py:215-235) for a run of consecutive merged
// Linear nodes of one instance-packed model; results are identical to
// launching the ops one by one (same tiles, same split order).
#pragma once
#include "gemm_sm100.cuh"

namespace nf {

constexpr int kChainMaxOps = 3;


struct alignas(64) ChainOp {
  CUtensorMap ma, mb, my, mr;  // 4-D (64, rows, K/64 | N/64, G) maps, two blocks per box
  GemmParams p;
  int unit0;      // first global unit index of this op
  int epi_dep;    // chain op whose results the epilogue reads (residual / LN
                  // statistics), -1: only earlier kernels
};

struct ChainParams {
  ChainOp ops[kChainMaxOps];
  int nops, units, groups;
  unsigned* done_tiles;  // [op][g] output tiles published
  unsigned* exit_count;  // CTAs finished (re-arm barrier)
  int rearm;             // 1: the last CTA zeroes the counters; 0: a later
                         // kernel still reads them (the caller zeroes them)
  const unsigned* ext_dep;  // [g] completion counter of the kernel producing
  unsigned ext_target;      // op 0's inputs (e.g. attention heads), or null
};

NF_DEVICE void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

#ifdef NF_CHAIN_TRACE
// Per-CTA, per-unit timestamps (globaltimer ns) of the last chained launch:
// [cta][local unit < 4][slot]: 0 producer starts unit, 1 its dependency
// satisfied, 2 MMA: first stage landed, 3 MMA: accumulator committed,
// 4 epilogue: accumulator ready, 5 epilogue: tile published, 6 op index,
// 7 CTA entry (unit 0 only), epilogue: 8 residual landed, 9 tile staged,
// 10 statistics written, 11 store complete. Read with nf_debug_chain_trace (tools/chain_trace.py).
__device__ unsigned long long g_chain_trace[148 * 4 * 16];
// per epilogue warp: [cta][unit][warp - 2][0 chunk loop start, 1 end]
__device__ unsigned long long g_chain_wtrace[148 * 4 * 8 * 8];
NF_DEVICE unsigned long long chain_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define NF_WT(slot)                                                               \
  do {                                                                            \
    if (lane == 0 && blockIdx.x < 148 && local < 4)                               \
      g_chain_wtrace[((blockIdx.x * 4 + local) * 8 + (warp - 2)) * 8 + (slot)] =  \
          chain_clock();                                                          \
  } while (0)
#define NF_CT(local, slot, val)                                                   \
  do {                                                                            \
    if (blockIdx.x < 148 && (local) < 4)                                          \
      g_chain_trace[(blockIdx.x * 4 + (local)) * 16 + (slot)] = (val);             \
  } while (0)
#else
#define NF_CT(local, slot, val) \
  do {                          \
  } while (0)
#define NF_WT(slot) \
  do {              \
  } while (0)
#endif

NF_DEVICE int chain_op_of(const ChainParams& cp, int u) {
  int op = 0;
#pragma unroll
  for (int j = 1; j < kChainMaxOps; ++j)
    if (j < cp.nops && u >= cp.ops[j].unit0) op = j;
  return op;
}

__global__ void __launch_bounds__(64 + 32 * epi_warps<128>(), 1)
    k_linear_chain_tc(const __grid_constant__ ChainParams cp) {
  constexpr int BN = 128, KPT = 2;
  using C = GemmCfg<BN, true, false, 0, KPT>;
  static_assert(C::kStaged && C::kNormBytes > 0, "staged swapped tiles with fold space");
  constexpr int kStages = C::kStages;
  constexpr int kEpiWarps = epi_warps<BN>();
  constexpr int kEpiThreads = 32 * kEpiWarps;
  constexpr int kColsPerThread = BN * 4 / kEpiWarps;
  constexpr int EC = 32;
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
  uint64_t* rbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 4);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
  float* sNorm = reinterpret_cast<float*>(sOut + C::kOutBytes + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#ifdef NF_CHAIN_TRACE
  if (threadIdx.x == 0) NF_CT(0, 7, chain_clock());
#endif
  if (warp == 0 && lane == 0) {
    for (int j = 0; j < cp.nops; ++j) {
      tma_prefetch_desc(&cp.ops[j].ma);
      tma_prefetch_desc(&cp.ops[j].mb);
      tma_prefetch_desc(&cp.ops[j].my);
      if (cp.ops[j].p.residual) tma_prefetch_desc(&cp.ops[j].mr);
    }
    mbar_init(&rbar[0], 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_dependents_launch();

  if (warp == 0) {
    if (lane == 0) {
      // --------------------------- TMA producer ---------------------------
      int it = 0, local = 0;
      bool first = true;
      for (int u = blockIdx.x; u < cp.units; u += gridDim.x, ++local) {
        const int op = chain_op_of(cp, u);
        const ChainOp& o = cp.ops[op];
        const UnitCoord c = decode_unit(o.p, u - o.unit0, true);
#ifdef NF_CHAIN_TRACE
        NF_CT(local, 0, chain_clock());
        NF_CT(local, 6, op);
#endif
        const int a_row = c.ta * kGemmBM, b_row = c.tb * BN;
        const int nst = (c.kb1 - c.kb0 + KPT - 1) / KPT;
        const int pre = nst < kStages ? nst : kStages;
        // Weights first: they depend on nothing, so they stream while the
        // producing op (or the previous kernel) finishes.
        for (int i = 0; i < pre; ++i) {
          const int stage = (it + i) % kStages;
          mbar_wait(&empty[stage], (((it + i) / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          tma_load_4d(sA + stage * C::kABytes, &o.ma, &full[stage], 0, a_row, c.kb0 + i * KPT,
                      c.g, kEvictFirst);
        }
        if (op == 0 && cp.ext_dep) {
          // op 0's activations come from a launch that counts instance g's
          // finished work: start as soon as g is done, not the whole launch
          wait_counter(cp.ext_dep + c.g, cp.ext_target);
        } else if (first && !cp.ext_dep) {
          // (with ext_dep, ops > 0 depend on earlier kernels only through op 0)
          grid_dependency_wait();
          first = false;
        }
        // Activations of op > 0 are the previous op's output: wait until it
        // has stored all of this instance's tiles. (Per-tile flags checked
        // per stage measured slower: a blocking L2 round trip per stage.)
        if (op > 0) {
          const ChainOp& d = cp.ops[op - 1];
          wait_counter(cp.done_tiles + (op - 1) * cp.groups + c.g,
                       unsigned(d.p.tiles_a * d.p.tiles_b));
        }
#ifdef NF_CHAIN_TRACE
        NF_CT(local, 1, chain_clock());
#endif
        for (int i = 0; i < pre; ++i) {
          const int stage = (it + i) % kStages;
          tma_load_4d(sB + stage * C::kBBytes, &o.mb, &full[stage], 0, b_row, c.kb0 + i * KPT,
                      c.g, kEvictLast);
        }
        for (int i = pre; i < nst; ++i) {
          const int stage = (it + i) % kStages;
          mbar_wait(&empty[stage], (((it + i) / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          tma_load_4d(sA + stage * C::kABytes, &o.ma, &full[stage], 0, a_row, c.kb0 + i * KPT,
                      c.g, kEvictFirst);
          tma_load_4d(sB + stage * C::kBBytes, &o.mb, &full[stage], 0, b_row, c.kb0 + i * KPT,
                      c.g, kEvictLast);
        }
        it += nst;
      }
    }
  } else if (warp == 1) {
    // ---------------------- MMA issuer (one lane) ----------------------
    constexpr uint32_t idesc = make_idesc_bf16_f32(kGemmBM, BN);
    int it = 0, local = 0;
    for (int u = blockIdx.x; u < cp.units; u += gridDim.x, ++local) {
      const int op = chain_op_of(cp, u);
      const UnitCoord c = decode_unit(cp.ops[op].p, u - cp.ops[op].unit0, true);
      const int acc = local & 1;
      mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
      for (int kb = c.kb0; kb < c.kb1; kb += KPT, ++it) {
        const int stage = it % kStages;
        mbar_wait(&full[stage], (it / kStages) & 1);
        tc_fence_after();
#ifdef NF_CHAIN_TRACE
        if (lane == 0 && kb == c.kb0) NF_CT(local, 2, chain_clock());
#endif
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < KPT; ++h) {
            if (kb + h >= c.kb1) break;
            const uint32_t a_base = smem_u32(sA + stage * C::kABytes) + h * (C::kABytes / KPT);
            const uint32_t b_base = smem_u32(sB + stage * C::kBBytes) + h * (C::kBBytes / KPT);
#pragma unroll
            for (int kk = 0; kk < kGemmBK / 16; ++kk)
              umma_f16_ss(d_tmem, make_sw128_kmajor_desc(a_base + kk * 32),
                          make_sw128_kmajor_desc(b_base + kk * 32), idesc,
                          (kb + h != c.kb0 || kk != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&tfull[acc]);
#ifdef NF_CHAIN_TRACE
      if (lane == 0) NF_CT(local, 3, chain_clock());
#endif
      __syncwarp();
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // feature row within the tile == TMEM lane
    const int etid = threadIdx.x - 64;
    const int col0 = ((warp - 2) >> 2) * kColsPerThread;  // token columns
    const uint32_t stage_base = smem_u32(sOut);
    uint32_t res_phase = 0;
    int local = 0;
    // residual tiles / statistics of earlier kernels: behind the grid
    // dependency, or per instance behind ext_dep for op 0 (whose producer
    // acquired what op 0 reads, transitively)
    if (!cp.ext_dep) grid_dependency_wait();
    for (int u = blockIdx.x; u < cp.units; u += gridDim.x, ++local) {
      const int op = chain_op_of(cp, u);
      const ChainOp& o = cp.ops[op];
      const GemmParams& p = o.p;
      const UnitCoord c = decode_unit(p, u - o.unit0, true);
      const int acc = local & 1;
      const bool has_res = p.residual != nullptr;
      const bool fold_in = p.nin_stats != nullptr;
      const bool fold_res = has_res && p.nres_stats != nullptr;
      const int m0 = c.ta * kGemmBM, n0 = c.tb * BN;
      // this thread's feature-row constants (weights-side, no dependency):
      // requested before the waits below
      float hb = 0.f, hcs = 0.f, hgm = 0.f, hbt = 0.f;
      {
        const int feat = m0 + row;
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
      // Everything below reads the producing op's results (residual tile,
      // LN statistics): one thread acquires, the barrier orders the rest.
      if (o.epi_dep >= 0) {
        if (etid == 0) {
          const ChainOp& d = cp.ops[o.epi_dep];
          wait_counter(cp.done_tiles + o.epi_dep * cp.groups + c.g,
                       unsigned(d.p.tiles_a * d.p.tiles_b));
        }
        named_bar_sync(1, kEpiThreads);
      } else if (cp.ext_dep) {
        // op reading only earlier kernels' results: behind ext_dep for g
        if (etid == 0) wait_counter(cp.ext_dep + c.g, cp.ext_target);
        named_bar_sync(1, kEpiThreads);
      }
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 12, chain_clock());
#endif
      if (has_res && etid == 0) {
        mbar_arrive_expect_tx(rbar, C::kOutBytes);
        tma_load_4d(sOut, &o.mr, rbar, 0, n0, m0 / kOutBlock, c.g, kEvictFirst);
      }
      if (fold_in || fold_res) {
        for (int t = etid; t < BN; t += kEpiThreads) {
          const int tok = n0 + t < p.rows_b ? n0 + t : p.rows_b - 1;
          const float2 m = fold_in ? fold_stats(p.nin_stats, p.nin_parts, p.rows_b, c.g, tok,
                                                p.nin_inv_d, p.nin_eps)
                                   : fold_stats(p.nres_stats, p.nres_parts, p.rows_b, c.g, tok,
                                                p.nres_inv_d, p.nres_eps);
          sNorm[t] = m.x;
          sNorm[BN + t] = m.y;
        }
        named_bar_sync(1, kEpiThreads);
      }
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 13, chain_clock());
#endif
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 4, chain_clock());
#endif
      const uint32_t t_row = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      float* part = nullptr;
      if (p.splits > 1) {
        // split-K: publish this split's fp32 partial, the last arriver reduces
        part = p.ws + (int64_t(c.tile) * p.splits) * kGemmBM * BN;
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
        if (etid == 0) *last_flag = (arrive_acq_rel(p.counters + c.tile) == unsigned(p.splits - 1));
        named_bar_sync(1, kEpiThreads);
        if (!*last_flag) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          if (has_res) {
            mbar_wait(rbar, res_phase);  // its residual tile landed unused
            res_phase ^= 1u;
          }
          continue;
        }
      }
      if (has_res) {
        mbar_wait(rbar, res_phase);
        res_phase ^= 1u;
      }
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 8, chain_clock());
      if (lane == 0 && blockIdx.x < 148 && local < 4)
        g_chain_wtrace[((blockIdx.x * 4 + local) * 8 + (warp - 2)) * 8] = chain_clock();
#endif
#pragma unroll 1
      for (int cc = col0; cc < col0 + kColsPerThread; cc += EC) {
        uint32_t rr[EC];
        tmem_ld_cols<EC>(t_row + uint32_t(cc), rr);
        tmem_ld_wait();
        if (cc == col0) NF_WT(1); else NF_WT(4);
        float v[EC];
#pragma unroll
        for (int j = 0; j < EC; ++j) v[j] = __uint_as_float(rr[j]);
        if (p.splits > 1) {
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
        if (fold_in) {
#pragma unroll
          for (int j = 0; j < EC; j += 4) {
            const float4 mu = *reinterpret_cast<const float4*>(sNorm + cc + j);
            const float4 rs = *reinterpret_cast<const float4*>(sNorm + BN + cc + j);
            v[j] = rs.x * fmaf(-mu.x, hcs, v[j]);
            v[j + 1] = rs.y * fmaf(-mu.y, hcs, v[j + 1]);
            v[j + 2] = rs.z * fmaf(-mu.z, hcs, v[j + 2]);
            v[j + 3] = rs.w * fmaf(-mu.w, hcs, v[j + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < EC; ++j) v[j] += hb;
        if (has_res) {
#pragma unroll
          for (int j = 0; j < EC; j += 4) {
            float r4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint16_t h;
              asm volatile("ld.shared.u16 %0, [%1];"
                           : "=h"(h)
                           : "r"(stage_base + stage_offset(cc + j + e, row, BN)));
              r4[e] = __uint_as_float(uint32_t(h) << 16);
            }
            if (fold_res) {  // (mean, rstd) of 4 tokens per 128-bit broadcast read
              const float4 mu = *reinterpret_cast<const float4*>(sNorm + cc + j);
              const float4 rs = *reinterpret_cast<const float4*>(sNorm + BN + cc + j);
              r4[0] = fmaf((r4[0] - mu.x) * rs.x, hgm, hbt);
              r4[1] = fmaf((r4[1] - mu.y) * rs.y, hgm, hbt);
              r4[2] = fmaf((r4[2] - mu.z) * rs.z, hgm, hbt);
              r4[3] = fmaf((r4[3] - mu.w) * rs.w, hgm, hbt);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) v[j + e] += r4[e];
          }
        }
        if (cc == col0) NF_WT(2); else NF_WT(5);
        apply_act<false>(p.act, v);
        __syncwarp();  // partner lanes read their residual before the pair stores
        const bool odd = lane & 1;
        const int feven = row & ~1;
#pragma unroll
        for (int j = 0; j < EC; j += 2) {
          const float send = odd ? v[j] : v[j + 1];
          const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
          const uint32_t packed = odd ? pack_bf16x2(recv, v[j + 1]) : pack_bf16x2(v[j], recv);
          const int t = cc + j + (odd ? 1 : 0);
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(stage_base + stage_offset(t, feven, BN)),
                       "r"(packed)
                       : "memory");
        }
        if (cc == col0) NF_WT(3); else NF_WT(6);
      }
#ifdef NF_CHAIN_TRACE
      if (lane == 0 && blockIdx.x < 148 && local < 4)
        g_chain_wtrace[((blockIdx.x * 4 + local) * 8 + (warp - 2)) * 8 + 7] = chain_clock();
#endif
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // TMEM buffer back to the MMA warp
      fence_proxy_async_smem();
      named_bar_sync(1, kEpiThreads);
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 9, chain_clock());
#endif
      if (etid == 0) {
        tma_store_4d(&o.my, sOut, 0, n0, m0 / kOutBlock, c.g);
        bulk_commit();
        if (p.splits > 1) p.counters[c.tile] = 0u;  // re-arm for the next launch
      }
      if (p.nout_stats) {
        // per-token (shifted sum, centred M2) over this tile's 128 features,
        // from the staged bf16 values (as gemm_sm100.cuh's swapped epilogue)
        constexpr int kBlocks = kGemmBM / kOutBlock;
        constexpr int kPerTok = kEpiThreads / BN;
        static_assert(kPerTok == kBlocks, "two threads per token");
        const int t = etid >> 1;
        float s1 = 0.f, s2 = 0.f;
        uint16_t h0;
        asm volatile("ld.shared.u16 %0, [%1];"
                     : "=h"(h0)
                     : "r"(stage_base + uint32_t(t * 128) + (uint32_t(t & 7) << 4)));
        const float shift = __uint_as_float(uint32_t(h0) << 16);
        const int b = etid & 1;
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
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        const float s = fmaf(float(kGemmBM), shift, s1);
        const float m2 = fmaxf(s2 - s1 * s1 * (1.0f / float(kGemmBM)), 0.f);
        if ((etid & 1) == 0 && n0 + t < p.rows_b)
          __stcg(p.nout_stats + (int64_t(c.g) * p.tiles_a + c.ta) * p.rows_b + n0 + t,
                 make_float2(s, m2));
      }
      named_bar_sync(1, kEpiThreads);
#ifdef NF_CHAIN_TRACE
      if (etid == 0) NF_CT(local, 10, chain_clock());
#endif
      if (etid == 0) {
        // the tile (TMA store) and its statistics are in global memory:
        // publish them to the consuming op's units
        bulk_wait0();
#ifdef NF_CHAIN_TRACE
        NF_CT(local, 11, chain_clock());
#endif
        fence_proxy_async_global();
        publish_count(cp.done_tiles + op * cp.groups + c.g);
#ifdef NF_CHAIN_TRACE
        NF_CT(local, 5, chain_clock());
#endif
      }
      named_bar_sync(1, kEpiThreads);  // staging reusable
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && cp.rearm) {
    __threadfence();
    if (atomicAdd(cp.exit_count, 1u) == gridDim.x - 1) {
      // every CTA is past its last wait: re-arm for the next launch
      for (int i = 0; i < cp.nops * cp.groups; ++i) cp.done_tiles[i] = 0u;
      *cp.exit_count = 0u;
      __threadfence();
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

}  // namespace nf
