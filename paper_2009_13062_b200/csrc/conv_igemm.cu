// Merged / grouped convolution as an implicit GEMM on the tensor cores.
//
// Replaces the reference's `grouped_conv2d` / `conv2d`
// (pkg/src/modelmerge/engine.py:122-191) for NHWC bf16 activations: group g
// is the GEMM  y[p, g*coutg + o] = sum_{kh,kw,c} x[pix(p)+(kh,kw), g*cg + c]
// * W[g][o][(kh*k + kw)*cg + c]  with folded BatchNorm bias, optional
// residual and ReLU in the epilogue. The kernel is k_grouped_gemm_tc
// (gemm_sm100.cuh) with GATHER warps: im2col rows are gathered from HBM/L2
// into shared memory by cp.async, never written to HBM.
//
// Orientation: pixels on the 128-row MMA side (normal) with a narrow N tile
// (16 / 32 / 64 / 128 / 256 output channels of one group: ResNeXt's 4..32
// channel groups waste at most 4x of a tiny MMA), or, for few pixels and
// wide groups (ResNet layer3/4 at batch 1), weights on the 128-row side
// (swapped) plus split-K so the weight stream covers every SM.
#include <algorithm>

#include "gemm_sm100.cuh"

namespace nf {

namespace {

// The 4-channel (padded RGB stem) halo gather: two taps per 16-byte chunk.
// Measured slower than the per-tap 8-byte cp.async gather for the ResNet
// stem, so the stem keeps the per-tap gather (kernel path kept and tested).
constexpr bool kHaloStem = false;

// 4-D NHWC box for the halo gather: (cg channels, halo_w columns, halo_h rows, 1 image).
bool make_halo_map(CUtensorMap* map, const void* x, int N, int H, int W, int C, int cg,
                   int halo_w, int halo_h) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
  cuuint64_t strides[3] = {cuuint64_t(C) * 2, cuuint64_t(W) * C * 2, cuuint64_t(H) * W * C * 2};
  cuuint32_t box[4] = {cuuint32_t(cg), cuuint32_t(halo_w), cuuint32_t(halo_h), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int conv_pick(int64_t pix, int64_t coutg, bool* swap) {
  *swap = pix <= 256 && coutg >= 128;
  if (*swap) return pix <= 64 ? 64 : (pix <= 128 ? 128 : 256);
  if (coutg <= 16) return 16;
  if (coutg <= 32) return 32;
  if (coutg <= 64) return 64;
  if (coutg <= 128 || pix < 4096) return 128;
  return 256;
}

// Max split-K factor for convs: the last arriving split reduces every
// partial of its tile alone, so deep splits trade HBM streaming parallelism
// for a serial fix-up.
constexpr int kConvMaxSplits = 4;

int conv_splits(int64_t tiles, int kb_total, int bn, int64_t ws_bytes) {
  if (ws_bytes <= kCounterBytes || tiles >= 96 || tiles > kCounterBytes / 4) return 1;
  int s = int(kNumSMs / tiles);
  s = s < kConvMaxSplits ? s : kConvMaxSplits;
  s = s < kb_total / 4 ? s : kb_total / 4;  // >= 4 K blocks per split
  while (s > 1 && tiles * s * int64_t(kGemmBM) * bn * 4 > ws_bytes - kCounterBytes) --s;
  return s < 1 ? 1 : s;
}


}  // namespace

int64_t conv_workspace_bytes(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t G,
                             int64_t k, int64_t stride, int64_t pad, int64_t Kpad) {
  if (G < 1 || C % G || Cout % G || stride < 1) return 0;
  const int64_t Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const int64_t pix = N * Ho * Wo, coutg = Cout / G;
  bool swap;
  const int bn = conv_pick(pix, coutg, &swap);
  const int64_t ta = swap ? (coutg + kGemmBM - 1) / kGemmBM : (pix + kGemmBM - 1) / kGemmBM;
  const int64_t tb = swap ? (pix + bn - 1) / bn : (coutg + bn - 1) / bn;
  const int64_t tiles = G * ta * tb;
  const int s = conv_splits(tiles, int((Kpad + kGemmBK - 1) / kGemmBK), bn, INT64_MAX);
  if (s <= 1) return 0;
  return kCounterBytes + tiles * s * int64_t(kGemmBM) * bn * 4;
}

int64_t conv_link_units(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t G,
                        int64_t k, int64_t stride, int64_t pad) {
  if (G < 1 || C % G || Cout % G || stride < 1) return 0;
  const int64_t Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const int64_t pix = N * Ho * Wo, coutg = Cout / G;
  bool swap;
  const int bn = conv_pick(pix, coutg, &swap);
  const int64_t ta = swap ? (coutg + kGemmBM - 1) / kGemmBM : (pix + kGemmBM - 1) / kGemmBM;
  const int64_t tb = swap ? (pix + bn - 1) / bn : (coutg + bn - 1) / bn;
  return ta * tb;
}

int grouped_conv_tc(const void* x, const void* w, const float* bias, const void* residual,
                    void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                    int pad, int Kpad, int relu, void* ws, int64_t ws_bytes, cudaStream_t stream,
                    const LinkSpec* link) {
  if (G < 1 || C % G || Cout % G || k < 1 || stride < 1 || pad < 0) return NF_ERR_SHAPE;
  const int cg = C / G, coutg = Cout / G;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1 || Kpad < k * k * cg || Kpad % 8) return NF_ERR_SHAPE;
  const int gather = cg % 8 == 0 ? 16 : (cg % 4 == 0 ? 8 : 0);
  if (!gather || coutg % 4 || G > 65535) return NF_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) return NF_ERR_UNSUPPORTED;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255)) return NF_ERR_SHAPE;
  const int64_t pix = int64_t(N) * Ho * Wo;
  if (pix > (int64_t(1) << 30) || int64_t(N) * H * W > (int64_t(1) << 30)) return NF_ERR_UNSUPPORTED;
  bool swap;
  const int bn = conv_pick(pix, coutg, &swap);
  if (gather == 8 && (swap || bn > 64)) return NF_ERR_UNSUPPORTED;
  // Halo gather: one image, pixels on M, 16..64-channel groups, a halo that
  // fits two buffers next to the operand ring.
  const int rows_out = std::min(Ho, (kGemmBM - 1 + Wo - 1) / Wo + 1);
  const int halo_h = (rows_out - 1) * stride + k;
  const int halo_w = (Wo - 1) * stride + k;
  const int halo_cpp = cg < 8 ? 8 : cg;  // TMA boxes need 16-byte rows
  const int64_t halo_raw = int64_t(halo_cpp) * 2 * halo_w * halo_h;
  const int64_t halo_bytes = (halo_raw + 1023) / 1024 * 1024;
  // (4-channel groups work too — the padded stem — but measured slower than
  // the 8-byte cp.async gather: a 7x7/s2 halo is barely smaller than 49 taps.)
  bool halo = !swap && N == 1 && (cg == 16 || cg == 32 || cg == 64 || (cg == 4 && kHaloStem)) &&
              bn <= 64 && halo_h <= 256 && halo_w <= 256 && halo_bytes <= 48 * 1024;

  GemmParams p{};
  if (link) {
    if (link->gpi < 1 || (link->dep_x && residual && !link->dep_r)) return NF_ERR_SHAPE;
    p.dep_x = link->dep_x;
    p.dep_x_target = link->dep_x_target;
    p.dep_r = link->dep_r;
    p.dep_r_target = link->dep_r_target;
    p.done = link->done;
    p.link_gpi = link->gpi;
  }
  p.act = relu ? NF_ACT_RELU : NF_ACT_NONE;
  p.bias = bias;
  p.residual = residual;
  p.out_gstride = coutg;
  p.out_ld = Cout;
  p.features = coutg;
  p.groups = G;
  p.kb_total = (Kpad + kGemmBK - 1) / kGemmBK;
  p.y_direct = y;
  p.cx = static_cast<const __nv_bfloat16*>(x);
  p.cH = H; p.cW = W; p.cC = C; p.cCg = cg; p.cK = k; p.cS = stride; p.cP = pad;
  p.cHo = Ho; p.cWo = Wo;
  CUtensorMap mw, my, mr, mh;
  if (halo && !make_halo_map(&mh, x, N, H, W, C, halo_cpp, halo_w, halo_h))
    halo = false;  // e.g. pixel rows not 16-byte multiples: per-tap gather instead
  if (halo) {
    p.halo_w = halo_w;
    p.halo_cpp = halo_cpp;
    p.halo_bytes = int(halo_bytes);
    p.halo_tx = uint32_t(halo_raw);
  }
  if (swap) {
    if (!make_bf16_map(&mw, w, G, coutg, Kpad, kGemmBK, kGemmBM, 0, 0) ||
        !make_bf16_map(&my, y, G, pix, coutg, kOutBlock, bn, Cout, coutg))
      return NF_ERR_UNSUPPORTED;
    p.rows_a = coutg;
    p.rows_b = int(pix);
  } else {
    if (!make_bf16_map(&mw, w, G, coutg, Kpad, kGemmBK, bn, 0, 0)) return NF_ERR_UNSUPPORTED;
    if (bn >= 64 && !make_bf16_map(&my, y, G, pix, coutg, kOutBlock, kGemmBM, Cout, coutg))
      return NF_ERR_UNSUPPORTED;
    if (bn < 64) my = mw;  // unused: narrow tiles store from registers
    p.rows_a = int(pix);
    p.rows_b = coutg;
  }
  mr = my;
  if (residual && bn >= 64 &&
      !(swap ? make_bf16_map(&mr, residual, G, pix, coutg, kOutBlock, bn, Cout, coutg)
             : make_bf16_map(&mr, residual, G, pix, coutg, kOutBlock, kGemmBM, Cout, coutg)))
    return NF_ERR_UNSUPPORTED;
  p.tiles_a = (p.rows_a + kGemmBM - 1) / kGemmBM;
  p.tiles_b = (p.rows_b + bn - 1) / bn;
  const int64_t tiles = int64_t(G) * p.tiles_a * p.tiles_b;
  p.splits = conv_splits(tiles, p.kb_total, bn, ws ? ws_bytes : 0);
  p.kb_per_split = (p.kb_total + p.splits - 1) / p.splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  if (tiles * p.splits > (int64_t(1) << 31) - 1) return NF_ERR_UNSUPPORTED;
  p.units = int(tiles * p.splits);
  p.counters = static_cast<unsigned*>(ws);
  p.ws = ws ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes) : nullptr;
  const int grid = p.units < kNumSMs ? p.units : kNumSMs;
  // The weights map is the only TMA operand; it sits in the slot its
  // orientation reads (A when swapped, B otherwise).
#define NF_CV(BNV, SW, GA) return launch_tc_res<BNV, SW, GA>(mw, mw, my, mr, p, grid, stream)
#define NF_CH(BNV) return launch_tc_res<BNV, false, 1>(mh, mw, my, mr, p, grid, stream)
  if (halo) {
    if (bn == 16) NF_CH(16);
    if (bn == 32) NF_CH(32);
    NF_CH(64);
  }
#undef NF_CH
  if (swap) {
    if (bn == 64) NF_CV(64, true, 16);
    if (bn == 128) NF_CV(128, true, 16);
    NF_CV(256, true, 16);
  }
  if (gather == 8) {
    if (bn == 16) NF_CV(16, false, 8);
    if (bn == 32) NF_CV(32, false, 8);
    NF_CV(64, false, 8);
  }
  if (bn == 16) NF_CV(16, false, 16);
  if (bn == 32) NF_CV(32, false, 16);
  if (bn == 64) NF_CV(64, false, 16);
  if (bn == 128) NF_CV(128, false, 16);
  NF_CV(256, false, 16);
#undef NF_CV
}

}  // namespace nf
