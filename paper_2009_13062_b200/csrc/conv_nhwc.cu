// NHWC convolution helpers for the merged CNN plans (ResNet-50 / ResNeXt-50).
//
// A merged conv is a grouped conv (reference `grouped_conv2d`,
// pkg/src/modelmerge/engine.py:155-191) with G = M * groups. In NHWC the
// channels of one pixel are contiguous, so group g's input is a strided
// column block of the pixel matrix and the conv is a grouped GEMM:
//   * 1x1 stride-1 convs feed k_grouped_gemm_tc directly (row stride C,
//     group stride C/G) — no copy;
//   * other convs with tensor-core-sized groups go through k_im2col_nhwc,
//     which writes rows [pixel][group][(kh, kw, c) padded to K_pad];
//   * small groups (ResNeXt's 4..32 channels per group, where a 128-wide
//     MMA tile would be mostly padding) run k_conv_nhwc_direct: one thread
//     per (pixel, out channel), fused folded-BN bias + residual + ReLU.
// Plus NHWC max / mean pooling (with padding).
#include "common.cuh"
#include "kernels.h"

namespace nf {

struct Im2colGeom {
  int N, H, W, C, G, Cg, k, stride, pad, Ho, Wo, Kpad;
};

// Row (n, ho, wo), group g, column kk = (kh*k + kw)*Cg + c  (kk >= k*k*Cg: 0).
template <typename T>
__global__ void k_im2col_nhwc(const T* __restrict__ x, T* __restrict__ y, Im2colGeom g) {
  pdl_enter();
  const int64_t total = int64_t(g.N) * g.Ho * g.Wo * g.G * g.Kpad;
  const int kk_valid = g.k * g.k * g.Cg;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int kk = int(i % g.Kpad);
    const int64_t rg = i / g.Kpad;
    const int grp = int(rg % g.G);
    const int64_t pix = rg / g.G;
    const int wo = int(pix % g.Wo);
    const int ho = int((pix / g.Wo) % g.Ho);
    const int n = int(pix / (int64_t(g.Wo) * g.Ho));
    T v = from_f32<T>(0.0f);
    if (kk < kk_valid) {
      const int c = kk % g.Cg;
      const int tap = kk / g.Cg;
      const int kh = tap / g.k, kw = tap % g.k;
      const int h = ho * g.stride - g.pad + kh, w = wo * g.stride - g.pad + kw;
      if (h >= 0 && h < g.H && w >= 0 && w < g.W)
        v = x[((int64_t(n) * g.H + h) * g.W + w) * g.C + int64_t(grp) * g.Cg + c];
    }
    y[i] = v;
  }
}

int im2col_nhwc(const void* x, void* y, int N, int H, int W, int C, int G, int k, int stride,
                int pad, int Kpad, int dtype, cudaStream_t s) {
  if (G < 1 || C % G || k < 1 || stride < 1 || pad < 0) return NF_ERR_SHAPE;
  const int Cg = C / G;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1 || Kpad < k * k * Cg) return NF_ERR_SHAPE;
  Im2colGeom g{N, H, W, C, G, Cg, k, stride, pad, Ho, Wo, Kpad};
  const int64_t total = int64_t(N) * Ho * Wo * G * Kpad;
  int64_t blocks = (total + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 32) blocks = int64_t(kNumSMs) * 32;
  if (dtype == NF_BF16)
    launch_pdl(k_im2col_nhwc<__nv_bfloat16>, dim3(unsigned(blocks)), dim3(256), 0, s,
               static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), g);
  else if (dtype == NF_F32)
    launch_pdl(k_im2col_nhwc<float>, dim3(unsigned(blocks)), dim3(256), 0, s,
               static_cast<const float*>(x), static_cast<float*>(y), g);
  else
    return NF_ERR_UNSUPPORTED;
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

// Direct grouped conv, NHWC in / out, weights (Cout, kh, kw, Cg) fp32-folded
// as T. One thread per output element; consecutive threads take consecutive
// output channels of one pixel, so stores and the channel-contiguous input
// reads coalesce. Epilogue: relu?(acc + bias[c] + residual).
struct DirectGeom {
  int N, H, W, C, Ho, Wo, Cout, G, Cg, k, stride, pad;
};

template <typename T>
__global__ void __launch_bounds__(256)
    k_conv_nhwc_direct(const T* __restrict__ x, const T* __restrict__ w,
                       const float* __restrict__ bias, const T* __restrict__ res,
                       T* __restrict__ y, DirectGeom g, int relu) {
  pdl_enter();
  const int64_t total = int64_t(g.N) * g.Ho * g.Wo * g.Cout;
  const int cout_g = g.Cout / g.G;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int co = int(i % g.Cout);
    const int64_t pix = i / g.Cout;
    const int wo = int(pix % g.Wo);
    const int ho = int((pix / g.Wo) % g.Ho);
    const int n = int(pix / (int64_t(g.Wo) * g.Ho));
    const int grp = co / cout_g;
    const T* wp = w + int64_t(co) * g.k * g.k * g.Cg;
    float acc = 0.f;
    for (int kh = 0; kh < g.k; ++kh) {
      const int h = ho * g.stride - g.pad + kh;
      if (h < 0 || h >= g.H) continue;
      for (int kw = 0; kw < g.k; ++kw) {
        const int ww = wo * g.stride - g.pad + kw;
        if (ww < 0 || ww >= g.W) continue;
        const T* xp = x + ((int64_t(n) * g.H + h) * g.W + ww) * g.C + int64_t(grp) * g.Cg;
        const T* wt = wp + (kh * g.k + kw) * g.Cg;
        for (int c = 0; c < g.Cg; ++c) acc = fmaf(to_f32(xp[c]), to_f32(wt[c]), acc);
      }
    }
    if (bias) acc += bias[co];
    if (res) acc += to_f32(res[i]);
    if (relu) acc = fmaxf(acc, 0.f);
    y[i] = from_f32<T>(acc);
  }
}

int conv_nhwc_direct(const void* x, const void* w, const float* bias, const void* residual,
                     void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                     int pad, int relu, int dtype, cudaStream_t s) {
  if (G < 1 || C % G || Cout % G || k < 1 || stride < 1 || pad < 0) return NF_ERR_SHAPE;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1) return NF_ERR_SHAPE;
  DirectGeom g{N, H, W, C, Ho, Wo, Cout, G, C / G, k, stride, pad};
  const int64_t total = int64_t(N) * Ho * Wo * Cout;
  int64_t blocks = (total + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 32) blocks = int64_t(kNumSMs) * 32;
  if (dtype == NF_BF16)
    launch_pdl(k_conv_nhwc_direct<__nv_bfloat16>, dim3(unsigned(blocks)), dim3(256), 0, s,
               static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w), bias,
               static_cast<const __nv_bfloat16*>(residual), static_cast<__nv_bfloat16*>(y), g,
               relu);
  else if (dtype == NF_F32)
    launch_pdl(k_conv_nhwc_direct<float>, dim3(unsigned(blocks)), dim3(256), 0, s,
               static_cast<const float*>(x), static_cast<const float*>(w), bias,
               static_cast<const float*>(residual), static_cast<float*>(y), g, relu);
  else
    return NF_ERR_UNSUPPORTED;
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

// NHWC pooling: thread per (n, ho, wo, c), channels fastest. Max pads with
// -inf; mean divides the window sum (row-major window order) by k^2.
template <typename T, bool MAXP>
__global__ void k_pool_nhwc(const T* __restrict__ x, T* __restrict__ y, int N, int H, int W,
                            int C, int Ho, int Wo, int k, int stride, int pad) {
  pdl_enter();
  const int64_t total = int64_t(N) * Ho * Wo * C;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(i % C);
    const int64_t pix = i / C;
    const int wo = int(pix % Wo);
    const int ho = int((pix / Wo) % Ho);
    const int n = int(pix / (int64_t(Wo) * Ho));
    float acc = MAXP ? -INFINITY : 0.f;
    for (int r = 0; r < k; ++r) {
      const int h = ho * stride - pad + r;
      for (int q = 0; q < k; ++q) {
        const int w = wo * stride - pad + q;
        const bool in = h >= 0 && h < H && w >= 0 && w < W;
        const float v = in ? to_f32(x[((int64_t(n) * H + h) * W + w) * C + c])
                           : (MAXP ? -INFINITY : 0.f);
        acc = MAXP ? fmaxf(acc, v) : __fadd_rn(acc, v);
      }
    }
    y[i] = from_f32<T>(MAXP ? acc : __fdiv_rn(acc, float(k * k)));
  }
}

// bf16, C % 8 == 0: one thread per (pixel, 8-channel group) with 16-byte
// loads / stores and 32-bit indexing (HBM-bound). Max is order-free; the mean
// sums in the same row-major window order as the scalar kernel.
template <bool MAXP>
__global__ void k_pool_nhwc_v8(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                               int N, int H, int W, int C8, int Ho, int Wo, int k, int stride,
                               int pad) {
  pdl_enter();
  const int total = N * Ho * Wo * C8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = i % C8;
    const int pix = i / C8;
    const int wo = pix % Wo;
    const int t = pix / Wo;
    const int ho = t % Ho;
    const int n = t / Ho;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = MAXP ? -INFINITY : 0.f;
    for (int r = 0; r < k; ++r) {
      const int h = ho * stride - pad + r;
      for (int q = 0; q < k; ++q) {
        const int w = wo * stride - pad + q;
        if (h >= 0 && h < H && w >= 0 && w < W) {
          const uint4 u = *reinterpret_cast<const uint4*>(
              x + ((int64_t(n) * H + h) * W + w) * (C8 * 8) + c8 * 8);
          const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(p2[e]);
            acc[2 * e] = MAXP ? fmaxf(acc[2 * e], f.x) : __fadd_rn(acc[2 * e], f.x);
            acc[2 * e + 1] = MAXP ? fmaxf(acc[2 * e + 1], f.y) : __fadd_rn(acc[2 * e + 1], f.y);
          }
        } else if (!MAXP) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], 0.f);
        }
      }
    }
    uint4 o;
    uint32_t* po = reinterpret_cast<uint32_t*>(&o);
    const float inv_den = float(k * k);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      po[e] = MAXP ? pack_bf16x2(acc[2 * e], acc[2 * e + 1])
                   : pack_bf16x2(__fdiv_rn(acc[2 * e], inv_den), __fdiv_rn(acc[2 * e + 1], inv_den));
    *reinterpret_cast<uint4*>(y + int64_t(pix) * (C8 * 8) + c8 * 8) = o;
  }
}

// fp32, C % 4 == 0: one thread per (pixel, 4-channel group), 16-byte loads /
// stores, 32-bit indexing; per element the same window order and arithmetic
// as k_pool_nhwc (bit-identical), without its per-element 64-bit divisions.
template <bool MAXP>
__global__ void k_pool_nhwc_v4f(const float* __restrict__ x, float* __restrict__ y, int N, int H,
                                int W, int C4, int Ho, int Wo, int k, int stride, int pad) {
  pdl_enter();
  const int total = N * Ho * Wo * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int pix = i / C4;
    const int c4 = i - pix * C4;
    const int t = pix / Wo;
    const int wo = pix - t * Wo;
    const int n = t / Ho;
    const int ho = t - n * Ho;
    float4 acc = MAXP ? make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < k; ++r) {
      const int h = ho * stride - pad + r;
      for (int q = 0; q < k; ++q) {
        const int w = wo * stride - pad + q;
        float4 v = MAXP ? make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        if (h >= 0 && h < H && w >= 0 && w < W)
          v = *reinterpret_cast<const float4*>(x + ((n * H + h) * W + w) * (C4 * 4) + c4 * 4);
        if (MAXP) {
          acc.x = fmaxf(acc.x, v.x); acc.y = fmaxf(acc.y, v.y);
          acc.z = fmaxf(acc.z, v.z); acc.w = fmaxf(acc.w, v.w);
        } else {
          acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
          acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
        }
      }
    }
    if (!MAXP) {
      const float den = float(k * k);
      acc.x = __fdiv_rn(acc.x, den); acc.y = __fdiv_rn(acc.y, den);
      acc.z = __fdiv_rn(acc.z, den); acc.w = __fdiv_rn(acc.w, den);
    }
    *reinterpret_cast<float4*>(y + pix * (C4 * 4) + c4 * 4) = acc;
  }
}

int pool_nhwc(const void* x, void* y, int N, int H, int W, int C, int kind, int k, int stride,
              int pad, int dtype, cudaStream_t s) {
  if (k < 1 || stride < 1 || pad < 0 || 2 * pad > k) return NF_ERR_SHAPE;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1) return NF_ERR_SHAPE;
  const int64_t total = int64_t(N) * Ho * Wo * C;
  int64_t blocks = (total + 255) / 256;
  if (blocks > int64_t(kNumSMs) * 32) blocks = int64_t(kNumSMs) * 32;
#define NF_PN(T)                                                                                   \
  do {                                                                                             \
    auto* px = static_cast<const T*>(x);                                                           \
    auto* py = static_cast<T*>(y);                                                                 \
    if (kind == NF_POOL_MAX)                                                                       \
      launch_pdl(k_pool_nhwc<T, true>, dim3(unsigned(blocks)), dim3(256), 0, s, px, py, N, H, W, \
                 C, Ho, Wo, k, stride, pad);                                                       \
    else                                                                                           \
      launch_pdl(k_pool_nhwc<T, false>, dim3(unsigned(blocks)), dim3(256), 0, s, px, py, N, H,   \
                 W, C, Ho, Wo, k, stride, pad);                                                    \
  } while (0)
  const bool v8 = dtype == NF_BF16 && C % 8 == 0 && int64_t(N) * H * W * C < (int64_t(1) << 31) &&
                  ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  const bool v4f = dtype == NF_F32 && C % 4 == 0 && int64_t(N) * H * W * C < (int64_t(1) << 31) &&
                   int64_t(N) * Ho * Wo * C < (int64_t(1) << 31) &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  if (v4f) {
    const int64_t work = int64_t(N) * Ho * Wo * (C / 4);
    int64_t b4 = (work + 255) / 256;
    if (b4 > int64_t(kNumSMs) * 16) b4 = int64_t(kNumSMs) * 16;
    auto* px = static_cast<const float*>(x);
    auto* py = static_cast<float*>(y);
    if (kind == NF_POOL_MAX)
      launch_pdl(k_pool_nhwc_v4f<true>, dim3(unsigned(b4)), dim3(256), 0, s, px, py, N, H, W,
                 C / 4, Ho, Wo, k, stride, pad);
    else
      launch_pdl(k_pool_nhwc_v4f<false>, dim3(unsigned(b4)), dim3(256), 0, s, px, py, N, H, W,
                 C / 4, Ho, Wo, k, stride, pad);
    return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
  }
  if (v8) {
    const int64_t work = int64_t(N) * Ho * Wo * (C / 8);
    int64_t b8 = (work + 255) / 256;
    if (b8 > int64_t(kNumSMs) * 16) b8 = int64_t(kNumSMs) * 16;
    auto* px = static_cast<const __nv_bfloat16*>(x);
    auto* py = static_cast<__nv_bfloat16*>(y);
    if (kind == NF_POOL_MAX)
      launch_pdl(k_pool_nhwc_v8<true>, dim3(unsigned(b8)), dim3(256), 0, s, px, py, N, H, W,
                 C / 8, Ho, Wo, k, stride, pad);
    else
      launch_pdl(k_pool_nhwc_v8<false>, dim3(unsigned(b8)), dim3(256), 0, s, px, py, N, H, W,
                 C / 8, Ho, Wo, k, stride, pad);
  } else if (dtype == NF_BF16) NF_PN(__nv_bfloat16);
  else if (dtype == NF_F32) NF_PN(float);
  else return NF_ERR_UNSUPPORTED;
#undef NF_PN
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

}  // namespace nf
