// Grouped linear on the CUDA cores.
//
// EXACT mode is the bit-exact restatement of the reference kernels
// `matmul` / `batch_matmul` (pkg/src/modelmerge/engine.py:194-235): for each
// output element the contraction runs k = 0, 1, ... in ascending order with
// the product and the sum each rounded to fp32 (numpy evaluates
// `y += x[..., k] * w[k]` as a rounded multiply then a rounded add, never a
// fused FMA), and the bias is added once after the loop. `__fmul_rn` /
// `__fadd_rn` forbid FMA contraction, so the result is byte-identical to the
// numpy kernel. FAST mode uses FFMA with the same loop (used for fp32 shapes
// the tensor-core path does not take, and for ragged bf16 shapes).
#include "common.cuh"
#include "kernels.h"

namespace nf {

constexpr int kSimtRows = 8;      // token rows per thread (weight reuse)
constexpr int kSimtThreads = 256;  // output features per block
constexpr int kSimtChunk = 512;    // K elements staged per pass

template <typename T, bool EXACT, bool WKN>
__global__ void __launch_bounds__(kSimtThreads)
    k_linear_simt(const T* __restrict__ x, const T* __restrict__ w, const float* __restrict__ bias,
                  const T* __restrict__ residual, T* __restrict__ y, int T_rows, int K, int N,
                  int act, int64_t x_ld, int64_t x_gs, int64_t y_ld, int64_t y_gs) {
  pdl_enter();
  __shared__ float xs[kSimtRows][kSimtChunk];
  const int g = blockIdx.z;
  const int t0 = blockIdx.y * kSimtRows;
  const int n = blockIdx.x * kSimtThreads + threadIdx.x;
  const T* xg = x + int64_t(g) * x_gs;
  const T* wg = w + int64_t(g) * K * N;
  float acc[kSimtRows];
#pragma unroll
  for (int r = 0; r < kSimtRows; ++r) acc[r] = 0.0f;

  for (int k0 = 0; k0 < K; k0 += kSimtChunk) {
    const int kc = min(kSimtChunk, K - k0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtRows * kc; idx += kSimtThreads) {
      const int r = idx / kc, kk = idx % kc;
      const int t = t0 + r;
      xs[r][kk] = t < T_rows ? to_f32(xg[int64_t(t) * x_ld + k0 + kk]) : 0.0f;
    }
    __syncthreads();
    if (n < N) {
      for (int kk = 0; kk < kc; ++kk) {
        const int k = k0 + kk;
        const float wv = to_f32(WKN ? wg[int64_t(k) * N + n] : wg[int64_t(n) * K + k]);
#pragma unroll
        for (int r = 0; r < kSimtRows; ++r) {
          if (EXACT)
            acc[r] = __fadd_rn(acc[r], __fmul_rn(xs[r][kk], wv));
          else
            acc[r] = fmaf(xs[r][kk], wv, acc[r]);
        }
      }
    }
  }
  if (n >= N) return;
  const float b = bias ? bias[int64_t(g) * N + n] : 0.0f;
#pragma unroll
  for (int r = 0; r < kSimtRows; ++r) {
    const int t = t0 + r;
    if (t >= T_rows) break;
    float v = acc[r];
    if (bias) v = __fadd_rn(v, b);
    const int64_t off = int64_t(g) * y_gs + int64_t(t) * y_ld + n;
    if (residual) v = __fadd_rn(v, to_f32(residual[off]));
    y[off] = from_f32<T>(apply_act(v, act));
  }
}

// FAST-mode few-row GEMV (T <= 8 rows, weights (K, N) row-major): the
// per-task classifier heads of the fp32 configs (FC 2048 -> 1000 at batch
// 1). A CTA owns 32 output columns and splits K over its 16 warps; each lane
// streams one column (consecutive lanes = consecutive 4-byte words, one
// 128-byte line per k), the rows of x are warp-uniform broadcasts, and the
// warps' partial sums are added in warp order through shared memory
// (deterministic). Weight-streaming: one pass over W at HBM rate instead of
// the 8-rows-per-thread kernel's N/256 CTAs.
constexpr int kGemvCols = 32;
constexpr int kGemvWarps = 16;

template <typename T>
__global__ void __launch_bounds__(kGemvCols * kGemvWarps)
    k_linear_gemv(const T* __restrict__ x, const T* __restrict__ w, const float* __restrict__ bias,
                  const T* __restrict__ residual, T* __restrict__ y, int T_rows, int K, int N,
                  int act, int64_t x_ld, int64_t x_gs, int64_t y_ld, int64_t y_gs) {
  pdl_enter();
  __shared__ float part[kGemvWarps][kSimtRows][kGemvCols];
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = blockIdx.x * kGemvCols + lane;
  const T* xg = x + int64_t(g) * x_gs;
  const T* wg = w + int64_t(g) * K * N;
  const int per = (K + kGemvWarps - 1) / kGemvWarps;
  const int k0 = warp * per, k1 = min(K, k0 + per);
  float acc[kSimtRows];
#pragma unroll
  for (int r = 0; r < kSimtRows; ++r) acc[r] = 0.0f;
  if (n < N) {
    // 16 independent weight loads in flight per lane: the kernel is bound by
    // bytes in flight (32 CTAs for N = 1000), not by the FMAs
#pragma unroll 16
    for (int k = k0; k < k1; ++k) {
      const float wv = to_f32(__ldg(wg + int64_t(k) * N + n));
#pragma unroll
      for (int r = 0; r < kSimtRows; ++r)
        if (r < T_rows) acc[r] = fmaf(to_f32(__ldg(xg + int64_t(r) * x_ld + k)), wv, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < kSimtRows; ++r) part[warp][r][lane] = acc[r];
  __syncthreads();
  if (warp != 0 || n >= N) return;
  const float b = bias ? bias[int64_t(g) * N + n] : 0.0f;
  for (int r = 0; r < T_rows; ++r) {
    float v = 0.0f;
#pragma unroll
    for (int q = 0; q < kGemvWarps; ++q) v += part[q][r][lane];
    v += b;
    const int64_t off = int64_t(g) * y_gs + int64_t(r) * y_ld + n;
    if (residual) v += to_f32(residual[off]);
    y[off] = from_f32<T>(apply_act(v, act));
  }
}

template <typename T>
static int launch_simt(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                       const float* bias, const void* residual, void* y, int64_t y_ld,
                       int64_t y_gs, int64_t G, int64_t Tr, int64_t K, int64_t N, int w_layout,
                       int act, int exact, cudaStream_t stream) {
  dim3 grid((N + kSimtThreads - 1) / kSimtThreads, (Tr + kSimtRows - 1) / kSimtRows, G);
  const T* xp = static_cast<const T*>(x);
  const T* wp = static_cast<const T*>(w);
  const T* rp = static_cast<const T*>(residual);
  T* yp = static_cast<T*>(y);
#define NF_SIMT(E, L)                                                                       \
  launch_pdl(k_linear_simt<T, E, L>, dim3(grid), dim3(kSimtThreads), 0, stream, xp, wp, bias, rp, yp, int(Tr), \
                                                            int(K), int(N), act, x_ld, x_gs, \
                                                            y_ld, y_gs)
  if (!exact && w_layout == NF_W_KN && Tr <= kSimtRows && G <= 65535) {
    launch_pdl(k_linear_gemv<T>, dim3((N + kGemvCols - 1) / kGemvCols, G),
               dim3(kGemvCols * kGemvWarps), 0, stream, xp, wp, bias, rp, yp, int(Tr), int(K),
               int(N), act, x_ld, x_gs, y_ld, y_gs);
  } else if (exact) {
    if (w_layout == NF_W_KN) NF_SIMT(true, true); else NF_SIMT(true, false);
  } else {
    if (w_layout == NF_W_KN) NF_SIMT(false, true); else NF_SIMT(false, false);
  }
#undef NF_SIMT
  return cudaGetLastError() == cudaSuccess ? NF_OK : NF_ERR_LAUNCH;
}

int grouped_linear_simt(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                        const float* bias, const void* residual, void* y, int64_t y_ld,
                        int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int dtype,
                        int w_layout, int act, int exact, cudaStream_t stream) {
  if (G > 65535 || (T + kSimtRows - 1) / kSimtRows > 65535) return NF_ERR_UNSUPPORTED;
  if (dtype == NF_F32)
    return launch_simt<float>(x, x_ld, x_gs, w, bias, residual, y, y_ld, y_gs, G, T, K, N,
                              w_layout, act, exact, stream);
  if (dtype == NF_BF16)
    return launch_simt<__nv_bfloat16>(x, x_ld, x_gs, w, bias, residual, y, y_ld, y_gs, G, T, K,
                                      N, w_layout, act, exact, stream);
  return NF_ERR_UNSUPPORTED;
}

}  // namespace nf
