// Grouped 2-D convolution on the CUDA cores, NCHW.
//
// EXACT mode restates the reference `grouped_conv2d` / `conv2d`
// (pkg/src/modelmerge/engine.py:122-191) bit for bit: output channel c reads
// input channels (c / (C_out/G)) * C_in/G + [0, C_in/G); the sum runs input
// channel outermost, then kernel row, then kernel column, with each product
// and each sum rounded separately (no FMA), and the bias added once after.
// Zero-padding taps are skipped: adding a signed zero to the running sum
// (which starts at +0 and can never become -0) leaves it unchanged, so this
// is identical to the reference's explicit zero-padded operand.
// FAST mode is the same loop with FFMA, plus optional fused epilogue
// (folded-BN scale/shift, residual, ReLU) for the CNN plans.
#include "common.cuh"
#include "kernels.h"

namespace nf {

struct ConvGeom {
  int N, Cin, H, W, Cout, Ho, Wo, k, stride, pad, groups;
};

template <typename T, bool EXACT>
__global__ void __launch_bounds__(256)
    k_conv_simt(const T* __restrict__ x, const T* __restrict__ w, const float* __restrict__ bias,
                const float* __restrict__ scale, const T* __restrict__ residual,
                T* __restrict__ y, ConvGeom g, int relu) {
  pdl_enter();
  const int64_t total = int64_t(g.N) * g.Cout * g.Ho * g.Wo;
  const int cin_g = g.Cin / g.groups;
  const int cout_g = g.Cout / g.groups;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int wo = int(i % g.Wo);
    const int ho = int((i / g.Wo) % g.Ho);
    const int co = int((i / (int64_t(g.Wo) * g.Ho)) % g.Cout);
    const int n = int(i / (int64_t(g.Wo) * g.Ho * g.Cout));
    const int cbase = (co / cout_g) * cin_g;
    const T* wp = w + int64_t(co) * cin_g * g.k * g.k;
    float acc = 0.0f;
    for (int ci = 0; ci < cin_g; ++ci) {
      const T* xp = x + (int64_t(n) * g.Cin + cbase + ci) * g.H * g.W;
      for (int r = 0; r < g.k; ++r) {
        const int h = ho * g.stride - g.pad + r;
        if (h < 0 || h >= g.H) continue;
        for (int s = 0; s < g.k; ++s) {
          const int ww = wo * g.stride - g.pad + s;
          if (ww < 0 || ww >= g.W) continue;
          const float a = to_f32(wp[(ci * g.k + r) * g.k + s]);
          const float b = to_f32(xp[h * g.W + ww]);
          acc = EXACT ? __fadd_rn(acc, __fmul_rn(a, b)) : fmaf(a, b, acc);
        }
      }
    }
    if (scale) acc = __fmul_rn(acc, scale[co]);
    if (bias) acc = __fadd_rn(acc, bias[co]);
    if (residual) acc = __fadd_rn(acc, to_f32(residual[i]));
    if (relu) acc = fmaxf(acc, 0.0f);
    y[i] = from_f32<T>(acc);
  }
}

int conv2d_simt(const void* x, const void* w, const float* bias, const float* scale,
                const void* residual, void* y, int N, int Cin, int H, int W, int Cout, int k,
                int stride, int pad, int groups, int relu, int dtype, int exact,
                cudaStream_t s) {
  if (groups < 1 || Cin % groups || Cout % groups || k < 1 || stride < 1 || pad < 0)
    return NF_ERR_SHAPE;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1) return NF_ERR_SHAPE;
  ConvGeom g{N, Cin, H, W, Cout, Ho, Wo, k, stride, pad, groups};
  const int64_t total = int64_t(N) * Cout * Ho * Wo;
  int64_t blocks = (total + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 64) blocks = int64_t(kNumSMs) * 64;
#define NF_CONV(T, E)                                                                      \
  launch_pdl(k_conv_simt<T, E>, dim3(unsigned(blocks)), dim3(256), 0, s,                                       \
      static_cast<const T*>(x), static_cast<const T*>(w), bias, scale,                     \
      static_cast<const T*>(residual), static_cast<T*>(y), g, relu)
  if (dtype == NF_F32) {
    if (exact) NF_CONV(float, true); else NF_CONV(float, false);
  } else if (dtype == NF_BF16) {
    if (exact) NF_CONV(__nv_bfloat16, true); else NF_CONV(__nv_bfloat16, false);
  } else {
    return NF_ERR_UNSUPPORTED;
  }
#undef NF_CONV
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

}  // namespace nf
