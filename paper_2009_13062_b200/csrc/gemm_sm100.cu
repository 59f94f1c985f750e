// Merged Linear host entry (tcgen05 grouped GEMM; kernel in gemm_sm100.cuh).
// Replaces the reference's `batch_matmul` (pkg/src/modelmerge/engine.py:215-235).
#include "gemm_chain.cuh"

namespace nf {

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

// 4-D view (64, rows, K/64, G) of a K-major bf16 operand with a
// (64, box_rows, 2, 1) SWIZZLE_128B box: one TMA transaction delivers two
// consecutive 64-wide k-blocks ([kb][row][128 B] in shared memory).
bool make_bf16_map_kpt2(CUtensorMap* map, const void* base, int64_t G, int64_t rows, int64_t K,
                        int box_rows, int64_t row_stride, int64_t g_stride, int kpt) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || K % 64) return false;
  if (row_stride <= 0) row_stride = K;
  if (g_stride <= 0) g_stride = rows * row_stride;
  if ((row_stride * 2) % 16 || (g_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(base) & 15))
    return false;
  cuuint64_t dims[4] = {64, cuuint64_t(rows), cuuint64_t(K / 64), cuuint64_t(G)};
  cuuint64_t strides[3] = {cuuint64_t(row_stride * 2), 128, cuuint64_t(g_stride * 2)};
  cuuint32_t box[4] = {64, cuuint32_t(box_rows), cuuint32_t(kpt), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int pick_bn(int64_t T, int64_t N) {
  if (T <= 256) return T <= 64 ? 64 : (T <= 128 ? 128 : 256);
  return N >= 256 ? 256 : (N > 64 ? 128 : 64);
}

// Split-K: a split adds a partial write + reduction to the critical path, so
// each one must still stream at least this many 64-wide K blocks.
constexpr int kSplitMinKB = 16;

// Split-K factor: enough units to cover the SMs when the tile count is low,
// with long K ranges per split and a workspace that fits.
static int choose_splits(int64_t tiles, int kb_total, int bn, int64_t ws_bytes) {
  if (ws_bytes <= kCounterBytes || tiles >= 100 || tiles > kCounterBytes / 4) return 1;
  int s = int(kNumSMs / tiles);
  s = s < kMaxSplits ? s : kMaxSplits;
  const int cap = kb_total / kSplitMinKB;
  s = s < cap ? s : cap;
  while (s > 1 && tiles * s * int64_t(kGemmBM) * bn * 4 > ws_bytes - kCounterBytes) --s;
  return s < 1 ? 1 : s;
}

struct LinearPlan {
  bool swap, pair;
  int bn;
  int64_t tiles_a, tiles_b, tiles;  // tiles_a counts pair tiles (256 rows) when pair
  int splits;
};

static LinearPlan plan_linear(int64_t G, int64_t T, int64_t K, int64_t N, int64_t ws_bytes) {
  LinearPlan L;
  L.swap = T <= 256;
  L.bn = pick_bn(T, N);
  // Measured (tools/gemm_trace.cu): pairs cut the MMA's operand stalls on
  // 128x256 tensor-bound tiles (4-5 stages of 32 KB per CTA instead of 3 of
  // 48 KB); on batch-1 weight-streaming tiles they only add cluster-launch
  // latency, so swapped tiles stay single-CTA.
  L.pair = !L.swap && L.bn == 256;
  const int64_t rows_a = L.swap ? N : T, rows_b = L.swap ? T : N;
  const int rows_per_a = L.pair ? 2 * kGemmBM : kGemmBM;
  L.tiles_a = (rows_a + rows_per_a - 1) / rows_per_a;
  L.tiles_b = (rows_b + L.bn - 1) / L.bn;
  L.tiles = G * L.tiles_a * L.tiles_b;
  const int kb_total = int((K + kGemmBK - 1) / kGemmBK);
  // split-K sizing works on per-CTA tiles (a pair unit occupies two SMs)
  L.splits = choose_splits(L.pair ? 2 * L.tiles : L.tiles, kb_total, L.bn, ws_bytes);
  return L;
}

// Folded LayerNorms are implemented for swapped, staged 128-token tiles
// (batch-1 encoders): the plan asks before folding.
bool linear_fold_supported(int64_t G, int64_t T, int64_t K, int64_t N) {
  if (G < 1 || K % 8 || N % 8 || G > 65535) return false;
  const LinearPlan L = plan_linear(G, T, K, N, 0);
  // Swapped 128-token tiles only (batch 1). Token-row tiles at large T were
  // built and measured twice (per-row statistics from the epilogue
  // registers): the extra epilogue work outweighs the saved norm launches
  // there (BERT N=32 B=8 7.21 -> 8.06 ms, XLNet N=32 B=4 4.28 -> 4.93 ms).
  return L.swap && L.bn == 128 && GemmOut<128, true>::kStaged && N % 128 == 0;
}

int64_t linear_link_units(int64_t G, int64_t T, int64_t K, int64_t N) {
  const LinearPlan L = plan_linear(G, T, K, N, 0);
  return (L.pair ? 2 : 1) * L.tiles_a * L.tiles_b;
}

int64_t linear_workspace_bytes(int64_t G, int64_t T, int64_t K, int64_t N) {
  const LinearPlan L = plan_linear(G, T, K, N, INT64_MAX);
  if (L.splits <= 1) return 0;
  const int64_t cta_tiles = L.pair ? 2 * L.tiles : L.tiles;
  return kCounterBytes + cta_tiles * L.splits * int64_t(kGemmBM) * L.bn * 4;
}

// Validation and kernel parameters of one merged Linear (shared by the
// single-op entry and the chained launch).
static int linear_setup(const void* ws, int64_t ws_bytes, int64_t G, int64_t T, int64_t K,
                        int64_t N, int out_dtype, int act, const float* bias,
                        const void* residual, void* y, int64_t y_ld, int64_t y_gs,
                        const NormFold* fold, GemmParams& p, LinearPlan& L) {
  // TMA needs 16-byte aligned row strides for x, w and y.
  if (out_dtype != NF_BF16 || K % 8 != 0 || N % 8 != 0) return NF_ERR_UNSUPPORTED;
  if (G > 65535 || T > (int64_t(1) << 30) || N > (int64_t(1) << 30)) return NF_ERR_UNSUPPORTED;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255)) return NF_ERR_SHAPE;
  p = GemmParams{};
  p.act = act;
  p.bias = bias;
  p.residual = residual;
  p.out_gstride = y_gs;
  p.out_ld = y_ld;
  p.features = int(N);
  p.groups = int(G);
  p.y_direct = y;
  p.kb_total = int((K + kGemmBK - 1) / kGemmBK);
  L = plan_linear(G, T, K, N, ws ? ws_bytes : 0);
  if (fold) {
    if (!linear_fold_supported(G, T, K, N)) return NF_ERR_UNSUPPORTED;
    if ((fold->in_stats && (!fold->in_colsum || fold->in_parts < 1)) ||
        (fold->res_stats && (!residual || !fold->res_gamma || !fold->res_beta ||
                             fold->res_parts < 1)))
      return NF_ERR_SHAPE;
    p.nin_stats = reinterpret_cast<const float2*>(fold->in_stats);
    p.nin_colsum = fold->in_colsum;
    p.nin_parts = fold->in_parts;
    p.nin_inv_d = 1.0f / float(K);
    p.nin_eps = fold->in_eps;
    p.nres_stats = reinterpret_cast<const float2*>(fold->res_stats);
    p.nres_gamma = fold->res_gamma;
    p.nres_beta = fold->res_beta;
    p.nres_parts = fold->res_parts;
    p.nres_inv_d = 1.0f / float(N);
    p.nres_eps = fold->res_eps;
    p.nout_stats = reinterpret_cast<float2*>(fold->out_stats);
  }
  p.rows_a = int(L.swap ? N : T);
  p.rows_b = int(L.swap ? T : N);
  p.tiles_a = int(L.tiles_a);
  p.tiles_b = int(L.tiles_b);
  p.splits = L.splits;
  p.kb_per_split = (p.kb_total + p.splits - 1) / p.splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  if (L.tiles * p.splits * 2 > (int64_t(1) << 31) - 1) return NF_ERR_UNSUPPORTED;
  p.units = int(L.tiles * p.splits);
  p.counters = static_cast<unsigned*>(const_cast<void*>(ws));
  p.ws = ws ? reinterpret_cast<float*>(static_cast<uint8_t*>(const_cast<void*>(ws)) + kCounterBytes)
            : nullptr;
  return NF_OK;
}

// Entry used by the C ABI. x rows at x + g*x_gs + t*x_ld (bf16); w (G, N, K)
// K-major bf16; bias fp32 (G, N) or null; y / residual rows at
// y + g*y_gs + t*y_ld (bf16). `ws` (zero-initialised once; the kernel
// restores its semaphores) enables split-K; null disables it.
int grouped_linear_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                      const float* bias, const void* residual, void* y, int64_t y_ld,
                      int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int out_dtype,
                      int act, void* ws, int64_t ws_bytes, cudaStream_t stream,
                      const NormFold* fold, const LinkSpec* link) {
  GemmParams p;
  LinearPlan L;
  const int st = linear_setup(ws, ws_bytes, G, T, K, N, out_dtype, act, bias, residual, y, y_ld,
                              y_gs, fold, p, L);
  if (st != NF_OK) return st;
  if (link) {
    if (link->gpi < 1 || (link->dep_x && residual && !link->dep_r)) return NF_ERR_SHAPE;
    p.dep_x = link->dep_x;
    p.dep_x_target = link->dep_x_target;
    p.dep_r = link->dep_r;
    p.dep_r_target = link->dep_r_target;
    p.done = link->done;
    p.link_gpi = link->gpi;
  }
  const bool swap = L.swap;
  const int bn = L.bn;
  const int bbox = L.pair ? bn / 2 : bn;  // B rows each CTA loads
  CUtensorMap ma, mb, my, mr;
  if (swap) {
    if (!make_bf16_map(&ma, w, G, N, K, kGemmBK, kGemmBM, 0, 0) ||
        !make_bf16_map(&mb, x, G, T, K, kGemmBK, bbox, x_ld, x_gs) ||
        !make_bf16_map(&my, y, G, T, N, kOutBlock, bn, y_ld, y_gs))
      return NF_ERR_UNSUPPORTED;
  } else {
    if (!make_bf16_map(&ma, x, G, T, K, kGemmBK, kGemmBM, x_ld, x_gs) ||
        !make_bf16_map(&mb, w, G, N, K, kGemmBK, bbox, 0, 0) ||
        !make_bf16_map(&my, y, G, T, N, kOutBlock, kGemmBM, y_ld, y_gs))
      return NF_ERR_UNSUPPORTED;
  }
  mr = my;
  if (residual &&
      !(swap ? make_bf16_map(&mr, residual, G, T, N, kOutBlock, bn, y_ld, y_gs)
             : make_bf16_map(&mr, residual, G, T, N, kOutBlock, kGemmBM, y_ld, y_gs)))
    return NF_ERR_UNSUPPORTED;
  if (L.pair) {
    const int clusters = p.units < kNumSMs / 2 ? p.units : kNumSMs / 2;
    const int grid = 2 * clusters;
    return launch_tc_res<256, false, 0, true>(ma, mb, my, mr, p, grid, stream);
  }
  int grid = p.units < kNumSMs ? p.units : kNumSMs;
  // Swapped launches: a balanced persistent grid, as many waves as one CTA
  // per SM needs but the same unit count per CTA (192 units: 96 CTAs x 2
  // instead of 44 x 2 + 104 x 1; BERT-base N=8 B=1 0.641 -> 0.636 ms).
  if (swap) grid = balanced_grid(p.units, kNumSMs);
#define NF_TC(BNV, SW) return launch_tc_res<BNV, SW>(ma, mb, my, mr, p, grid, stream)
  // Swapped 128-token tiles move two 64-wide k-blocks per TMA transaction:
  // the batch-1 main loop is bound by a per-stage cost, not bytes
  // (tools/gemm_trace.cu: 768->768 main loop 3.7 -> 2.9 us, 3072->768 split
  // 5.1 -> 3.9 us). Three per stage measured slower (0.620 -> 0.639 ms).
  if (swap && bn == 128 && K % 64 == 0 && N % 128 == 0 &&
      !(fold && fold->in_stats && fold->res_stats)) {
    CUtensorMap ma2, mb2, my2, mr2;
    constexpr int kpt = 2;
    // output / residual tiles (128 tokens x 128 features) as one 4-D box:
    // (64, T, N/64, G) with a (64, 128, 2, 1) box, the staging buffer's layout
    if (make_bf16_map_kpt2(&ma2, w, G, N, K, kGemmBM, 0, 0, kpt) &&
        make_bf16_map_kpt2(&mb2, x, G, T, K, bn, x_ld, x_gs, kpt) &&
        make_bf16_map_kpt2(&my2, y, G, T, N, bn, y_ld, y_gs, 2) &&
        (!residual || make_bf16_map_kpt2(&mr2, residual, G, T, N, bn, y_ld, y_gs, 2))) {
      if (!residual) mr2 = my2;
      return launch_tc_res<128, true, 0, false, 2>(ma2, mb2, my2, mr2, p, grid, stream);
    }
  }
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

// Ops the chained launch implements: the swapped 128-token tile with two
// k-blocks per stage (batch-1 weight-streaming shapes).
bool linear_chain_supported(int64_t G, int64_t T, int64_t K, int64_t N) {
  if (G < 1 || G > 65535 || K % 64 || N % 128) return false;
  const LinearPlan L = plan_linear(G, T, K, N, 0);
  return L.swap && L.bn == 128;
}

// Consecutive merged Linears of one instance-packed model in one persistent
// launch (gemm_chain.cuh). ops[j] reads only what ops[< j] or earlier
// kernels wrote, instance by instance. `counters` holds n_ops * G + 1 zeroed
// words; the kernel leaves them zeroed.
int grouped_linear_chain_tc(int nops, const LinearOpDesc* ops, unsigned* counters,
                            cudaStream_t stream, bool rearm, const unsigned* ext_dep,
                            unsigned ext_target) {
  if (nops < 1 || nops > kChainMaxOps || !ops || !counters) return NF_ERR_SHAPE;
  ChainParams cp{};
  cp.nops = nops;
  cp.groups = int(ops[0].G);
  int units = 0;
  for (int j = 0; j < nops; ++j) {
    const LinearOpDesc& d = ops[j];
    if (!d.x || !d.w || !d.y || d.G != ops[0].G) return NF_ERR_SHAPE;
    if (!linear_chain_supported(d.G, d.T, d.K, d.N)) return NF_ERR_UNSUPPORTED;
    const NormFold* fold = d.has_fold ? &d.fold : nullptr;
    if (fold && fold->in_stats && fold->res_stats) return NF_ERR_UNSUPPORTED;
    ChainOp& o = cp.ops[j];
    LinearPlan L;
    const int st = linear_setup(d.ws, d.ws_bytes, d.G, d.T, d.K, d.N, NF_BF16, d.act, d.bias,
                                d.residual, d.y, d.y_ld, d.y_gs, fold, o.p, L);
    if (st != NF_OK) return st;
    o.p = gemm_params_finalize(o.p);
    if (!make_bf16_map_kpt2(&o.ma, d.w, d.G, d.N, d.K, kGemmBM, 0, 0, 2) ||
        !make_bf16_map_kpt2(&o.mb, d.x, d.G, d.T, d.K, 128, d.x_ld, d.x_gs, 2) ||
        !make_bf16_map_kpt2(&o.my, d.y, d.G, d.T, d.N, 128, d.y_ld, d.y_gs, 2))
      return NF_ERR_UNSUPPORTED;
    o.mr = o.my;
    if (d.residual &&
        !make_bf16_map_kpt2(&o.mr, d.residual, d.G, d.T, d.N, 128, d.y_ld, d.y_gs, 2))
      return NF_ERR_UNSUPPORTED;
    o.unit0 = units;
    if (o.p.tiles_b != 1) return NF_ERR_UNSUPPORTED;
    // the epilogue's inputs: a residual or LN statistics written by an
    // earlier op of this chain (else by earlier kernels)
    o.epi_dep = -1;
    for (int i = 0; i < j; ++i) {
      const void* out_stats = ops[i].has_fold ? ops[i].fold.out_stats : nullptr;
      const bool reads = (d.residual && d.residual == ops[i].y) ||
                         (fold && out_stats &&
                          (fold->in_stats == out_stats || fold->res_stats == out_stats));
      if (reads) o.epi_dep = i;
    }
    if (j && d.x != ops[j - 1].y) return NF_ERR_UNSUPPORTED;  // activations = previous output
    if (int64_t(units) + o.p.units > (int64_t(1) << 30)) return NF_ERR_UNSUPPORTED;
    units += o.p.units;
  }
  cp.units = units;
  cp.done_tiles = counters;
  cp.exit_count = counters + int64_t(nops) * cp.groups;
  cp.rearm = rearm ? 1 : 0;
  cp.ext_dep = ext_dep;
  cp.ext_target = ext_target;
  using C = GemmCfg<128, true, false, 0, 2>;
  static SmemAttrOnce smem_attr;
  smem_attr.set(k_linear_chain_tc, int(C::kBytes));
  const int grid = units < kNumSMs ? units : kNumSMs;
  return launch_pdl(k_linear_chain_tc, dim3(grid), dim3(64 + 32 * epi_warps<128>()), C::kBytes,
                    stream, cp) == cudaSuccess
             ? NF_OK
             : NF_ERR_LAUNCH;
}

}  // namespace nf

#ifdef NF_CHAIN_TRACE
extern "C" int nf_debug_chain_trace(void* host, int bytes) {
  return int(cudaMemcpyFromSymbol(host, nf::g_chain_trace, size_t(bytes)));
}
extern "C" int nf_debug_chain_wtrace(void* host, int bytes) {
  return int(cudaMemcpyFromSymbol(host, nf::g_chain_wtrace, size_t(bytes)));
}
#endif
