// Internal (C++) launcher declarations shared between the kernel translation
// units and the C ABI in capi.cu. Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

// Folded LayerNorm operands of a batch-1 GEMM (see GemmParams::nin_*):
// stats are [g][part][token] (sum, centred sum of squares M2) float pairs
// over the part's 128 features.
struct NormFold {
  const float* in_stats;
  const float* in_colsum;
  int in_parts;
  float in_eps;
  const float* res_stats;
  const float* res_gamma;
  const float* res_beta;
  int res_parts;
  float res_eps;
  float* out_stats;
};

// Per-instance launch linking (see GemmParams::dep_x): counters are
// [instance] tile counts; instance of group g = g / gpi.
struct LinkSpec {
  const unsigned* dep_x;
  unsigned dep_x_target;
  const unsigned* dep_r;
  unsigned dep_r_target;
  unsigned* done;
  int gpi;
};

// gemm_sm100.cu — tcgen05 grouped GEMM (bf16 in, fp32 accumulate).
bool linear_fold_supported(int64_t G, int64_t T, int64_t K, int64_t N);
int grouped_linear_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                      const float* bias, const void* residual, void* y, int64_t y_ld,
                      int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int out_dtype,
                      int act, void* ws, int64_t ws_bytes, cudaStream_t stream,
                      const NormFold* fold = nullptr, const LinkSpec* link = nullptr);
int64_t linear_workspace_bytes(int64_t G, int64_t T, int64_t K, int64_t N);
// output tiles one group publishes (a CTA pair's two halves count apart)
int64_t linear_link_units(int64_t G, int64_t T, int64_t K, int64_t N);
// One op of a chained launch (same operands as grouped_linear_tc).
struct LinearOpDesc {
  const void* x;
  int64_t x_ld, x_gs;
  const void* w;
  const float* bias;
  const void* residual;
  void* y;
  int64_t y_ld, y_gs, G, T, K, N;
  int act;
  void* ws;
  int64_t ws_bytes;
  int has_fold;
  NormFold fold;
};
bool linear_chain_supported(int64_t G, int64_t T, int64_t K, int64_t N);
int grouped_linear_chain_tc(int nops, const LinearOpDesc* ops, unsigned* counters,
                            cudaStream_t stream, bool rearm = true,
                            const unsigned* ext_dep = nullptr, unsigned ext_target = 0);

// linear_simt.cu — CUDA-core grouped linear (exact reference order or FMA).
int grouped_linear_simt(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                        const float* bias, const void* residual, void* y, int64_t y_ld,
                        int64_t y_gs, int64_t G, int64_t T, int64_t K, int64_t N, int dtype,
                        int w_layout, int act, int exact, cudaStream_t stream);

// pointwise.cu
struct NormGeomC {
  int64_t R1, R2, s1, s2, G, Cg, sg, sc, rows_per_affine;
  float eps;
};
int elementwise(int op, const void* a, const void* b, void* y, int64_t n, int dtype,
                cudaStream_t s);
int s2d_stem(const void* x, void* y, int N, int G, int cg, int H, int W, cudaStream_t s);
int copy_strided(const void* src, void* dst, int rank, const int64_t* dims,
                 const int64_t* src_strides, const int64_t* dst_strides, int elem_bytes,
                 cudaStream_t s);
int group_norm(const void* x, const void* residual, const float* gamma, const float* beta,
               void* y, const NormGeomC& g, int dtype, cudaStream_t s);
int softmax(const void* x, void* y, int64_t outer, int64_t L, int64_t inner, int64_t so,
            int64_t sl, int64_t si, int dtype, cudaStream_t s);
int batch_norm(const void* x, const float* gamma, const float* beta, const float* mean,
               const float* var, void* y, int64_t N, int64_t C, int64_t inner, float eps,
               int dtype, cudaStream_t s);
int pool2d(const void* x, void* y, int64_t N, int64_t C, int H, int W, int kind, int k,
           int stride, int pad, int dtype, cudaStream_t s);

// conv_simt.cu
int conv2d_simt(const void* x, const void* w, const float* bias, const float* scale,
                const void* residual, void* y, int N, int Cin, int H, int W, int Cout, int k,
                int stride, int pad, int groups, int relu, int dtype, int exact,
                cudaStream_t s);

// conv_igemm.cu — implicit-GEMM conv (tcgen05, cp.async im2col gather).
int grouped_conv_tc(const void* x, const void* w, const float* bias, const void* residual,
                    void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                    int pad, int Kpad, int relu, void* ws, int64_t ws_bytes, cudaStream_t stream,
                    const LinkSpec* link = nullptr);
int64_t conv_link_units(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t G,
                        int64_t k, int64_t stride, int64_t pad);
int64_t conv_workspace_bytes(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t G,
                             int64_t k, int64_t stride, int64_t pad, int64_t Kpad);

// conv_tf32.cu — fp32 implicit-GEMM conv, 3xTF32 on tcgen05.
int grouped_conv_tf32(const void* x, const void* w, const float* bias, const void* residual,
                      void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                      int pad, int Kpad, int relu, void* ws, int64_t ws_bytes,
                      cudaStream_t stream);
int64_t conv_tf32_workspace_bytes(int64_t N, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                  int64_t G, int64_t k, int64_t stride, int64_t pad,
                                  int64_t Kpad);

// conv_nhwc.cu
int im2col_nhwc(const void* x, void* y, int N, int H, int W, int C, int G, int k, int stride,
                int pad, int Kpad, int dtype, cudaStream_t s);
int conv_nhwc_direct(const void* x, const void* w, const float* bias, const void* residual,
                     void* y, int N, int H, int W, int C, int Cout, int G, int k, int stride,
                     int pad, int relu, int dtype, cudaStream_t s);
int pool_nhwc(const void* x, void* y, int N, int H, int W, int C, int kind, int k, int stride,
              int pad, int dtype, cudaStream_t s);

// qkv_attention.cu — fused QKV projection + attention, batch 1, S = 128.
int qkv_attention_tc(const void* x, int64_t x_ld, int64_t x_gs, const void* w, const float* bias,
                     void* out, int64_t G, int64_t S, int64_t D, int64_t heads, float scale,
                     cudaStream_t stream, const NormFold* fold = nullptr,
                     const unsigned* dep = nullptr, unsigned dep_target = 0,
                     unsigned* done = nullptr);

// attention.cu
int attention(const void* qkv, void* out, int64_t Bt, int64_t S, int64_t H, int64_t dh,
              float scale, int dtype, int mode, cudaStream_t stream);
int rel_attention(const void* qkv, const void* r, const float* rwb, const float* rrb, void* out,
                  int64_t Bt, int64_t S, int64_t H, int64_t dh, int64_t seqs_per_bias,
                  int64_t seqs_per_r, float scale, int dtype, int mode, cudaStream_t stream);

}  // namespace nf
