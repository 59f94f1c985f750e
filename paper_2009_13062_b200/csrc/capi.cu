// extern "C" entry points: argument validation, dispatch to the kernel
// launchers, status mapping. See include/netfuse_b200.h for the contract.
#include "common.cuh"
#include "kernels.h"

extern "C" {

int nf_abi_version(void) { return 2; }

const char* nf_status_string(int status) {
  switch (status) {
    case NF_OK: return "ok";
    case NF_ERR_SHAPE: return "bad shape or argument";
    case NF_ERR_UNSUPPORTED: return "unsupported dtype or configuration";
    case NF_ERR_LAUNCH: return "CUDA launch failure";
    default: return "unknown status";
  }
}

int64_t nf_linear_workspace_bytes(int64_t groups, int64_t rows, int64_t k, int64_t n) {
  if (groups < 1 || rows < 1 || k < 1 || n < 1) return 0;
  return nf::linear_workspace_bytes(groups, rows, k, n);
}

int nf_grouped_linear_ws(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                         const void* bias, const void* residual, void* y, int64_t y_ld,
                         int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                         int dtype, int w_layout, int act, int mode, void* workspace,
                         int64_t workspace_bytes, void* stream) {
  if (!x || !w || !y || groups < 1 || rows < 1 || k < 1 || n < 1) return NF_ERR_SHAPE;
  if (x_ld < k || y_ld < n || (groups > 1 && (x_gs < 1 || y_gs < 1))) return NF_ERR_SHAPE;
  if (dtype != NF_F32 && dtype != NF_BF16) return NF_ERR_UNSUPPORTED;
  if (w_layout != NF_W_NK && w_layout != NF_W_KN) return NF_ERR_UNSUPPORTED;
  if (act < NF_ACT_NONE || act > NF_ACT_TANH) return NF_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float* b = static_cast<const float*>(bias);
  if (mode == NF_MODE_FAST && dtype == NF_BF16 && w_layout == NF_W_NK) {
    int st = nf::grouped_linear_tc(x, x_ld, x_gs, w, b, residual, y, y_ld, y_gs, groups, rows, k,
                                   n, dtype, act, workspace, workspace_bytes, s);
    if (st != NF_ERR_UNSUPPORTED) return st;
  }
  return nf::grouped_linear_simt(x, x_ld, x_gs, w, b, residual, y, y_ld, y_gs, groups, rows, k,
                                 n, dtype, w_layout, act, mode == NF_MODE_EXACT, s);
}

int nf_grouped_linear_strided(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                              const void* bias, const void* residual, void* y, int64_t y_ld,
                              int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                              int dtype, int w_layout, int act, int mode, void* stream) {
  return nf_grouped_linear_ws(x, x_ld, x_gs, w, bias, residual, y, y_ld, y_gs, groups, rows, k, n,
                              dtype, w_layout, act, mode, nullptr, 0, stream);
}

int nf_grouped_linear(const void* x, const void* w, const void* bias, const void* residual,
                      void* y, int64_t groups, int64_t rows, int64_t k, int64_t n, int dtype,
                      int w_layout, int act, int mode, void* stream) {
  return nf_grouped_linear_strided(x, k, rows * k, w, bias, residual, y, n, rows * n, groups,
                                   rows, k, n, dtype, w_layout, act, mode, stream);
}

int nf_grouped_conv2d(const void* x, const void* w, const float* bias, const float* scale,
                      const void* residual, void* y, int64_t N, int64_t Cin, int64_t H,
                      int64_t W, int64_t Cout, int kernel, int stride, int pad, int groups,
                      int relu, int dtype, int mode, void* stream) {
  if (!x || !w || !y || N < 1 || Cin < 1 || H < 1 || W < 1 || Cout < 1) return NF_ERR_SHAPE;
  if (mode == NF_MODE_EXACT && (scale || residual || relu)) return NF_ERR_UNSUPPORTED;
  return nf::conv2d_simt(x, w, bias, scale, residual, y, int(N), int(Cin), int(H), int(W),
                         int(Cout), kernel, stride, pad, groups, relu, dtype,
                         mode == NF_MODE_EXACT, static_cast<cudaStream_t>(stream));
}

int nf_elementwise(int op, const void* a, const void* b, void* y, int64_t n, int dtype,
                   void* stream) {
  if (!a || !y || n < 0) return NF_ERR_SHAPE;
  if (n == 0) return NF_OK;
  return nf::elementwise(op, a, b, y, n, dtype, static_cast<cudaStream_t>(stream));
}

int nf_counters_rearm(void* counters, int64_t bytes, void* stream) {
  if (!counters || bytes < 0) return NF_ERR_SHAPE;
  return cudaMemsetAsync(counters, 0, size_t(bytes), static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? NF_OK
             : NF_ERR_LAUNCH;
}

int nf_copy_strided(const void* x, void* y, int rank, const int64_t* dims,
                    const int64_t* x_strides, const int64_t* y_strides, int elem_bytes,
                    void* stream) {
  if (!x || !y || !dims || !x_strides || !y_strides) return NF_ERR_SHAPE;
  return nf::copy_strided(x, y, rank, dims, x_strides, y_strides, elem_bytes,
                          static_cast<cudaStream_t>(stream));
}

int nf_group_norm(const void* x, const void* residual, const float* gamma, const float* beta,
                  void* y, int64_t R1, int64_t R2, int64_t s1, int64_t s2, int64_t G,
                  int64_t Cg, int64_t sg, int64_t sc, int64_t rows_per_affine, float eps,
                  int dtype, void* stream) {
  if (!x || !y || !gamma || !beta) return NF_ERR_SHAPE;
  nf::NormGeomC g{R1, R2, s1, s2, G, Cg, sg, sc, rows_per_affine, eps};
  return nf::group_norm(x, residual, gamma, beta, y, g, dtype, static_cast<cudaStream_t>(stream));
}

int nf_softmax(const void* x, void* y, int64_t outer, int64_t L, int64_t inner, int64_t so,
               int64_t sl, int64_t si, int dtype, void* stream) {
  if (!x || !y) return NF_ERR_SHAPE;
  return nf::softmax(x, y, outer, L, inner, so, sl, si, dtype, static_cast<cudaStream_t>(stream));
}

int nf_attention(const void* qkv, void* out, int64_t Bt, int64_t S, int64_t H, int64_t dh,
                 float scale, int dtype, int mode, void* stream) {
  if (!qkv || !out) return NF_ERR_SHAPE;
  return nf::attention(qkv, out, Bt, S, H, dh, scale, dtype, mode,
                       static_cast<cudaStream_t>(stream));
}

int nf_rel_attention(const void* qkv, const void* r, const float* r_w_bias,
                     const float* r_r_bias, void* out, int64_t Bt, int64_t S, int64_t H,
                     int64_t dh, int64_t seqs_per_bias, int64_t seqs_per_r, float scale,
                     int dtype, int mode, void* stream) {
  if (!qkv || !r || !r_w_bias || !r_r_bias || !out) return NF_ERR_SHAPE;
  return nf::rel_attention(qkv, r, r_w_bias, r_r_bias, out, Bt, S, H, dh, seqs_per_bias,
                           seqs_per_r, scale, dtype, mode, static_cast<cudaStream_t>(stream));
}

int nf_batch_norm(const void* x, const float* gamma, const float* beta, const float* mean,
                  const float* var, void* y, int64_t N, int64_t C, int64_t inner, float eps,
                  int dtype, void* stream) {
  if (!x || !y || !gamma || !beta || !mean || !var) return NF_ERR_SHAPE;
  return nf::batch_norm(x, gamma, beta, mean, var, y, N, C, inner, eps, dtype,
                        static_cast<cudaStream_t>(stream));
}

int nf_pool2d(const void* x, void* y, int64_t N, int64_t C, int H, int W, int kind, int kernel,
              int stride, int pad, int dtype, void* stream) {
  if (!x || !y || N < 1 || C < 1 || H < 1 || W < 1) return NF_ERR_SHAPE;
  if (kind != NF_POOL_MAX && kind != NF_POOL_MEAN) return NF_ERR_UNSUPPORTED;
  return nf::pool2d(x, y, N, C, H, W, kind, kernel, stride, pad, dtype,
                    static_cast<cudaStream_t>(stream));
}

int nf_im2col_nhwc(const void* x, void* y, int N, int H, int W, int C, int groups, int kernel,
                   int stride, int pad, int kpad, int dtype, void* stream) {
  if (!x || !y || N < 1 || H < 1 || W < 1 || C < 1) return NF_ERR_SHAPE;
  return nf::im2col_nhwc(x, y, N, H, W, C, groups, kernel, stride, pad, kpad, dtype,
                         static_cast<cudaStream_t>(stream));
}

int nf_conv_nhwc_direct(const void* x, const void* w, const float* bias, const void* residual,
                        void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                        int stride, int pad, int relu, int dtype, void* stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || Cout < 1) return NF_ERR_SHAPE;
  return nf::conv_nhwc_direct(x, w, bias, residual, y, N, H, W, C, Cout, groups, kernel, stride,
                              pad, relu, dtype, static_cast<cudaStream_t>(stream));
}

int nf_grouped_conv_tc(const void* x, const void* w, const float* bias, const void* residual,
                       void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                       int stride, int pad, int kpad, int relu, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || Cout < 1) return NF_ERR_SHAPE;
  return nf::grouped_conv_tc(x, w, bias, residual, y, N, H, W, C, Cout, groups, kernel, stride,
                             pad, kpad, relu, workspace, workspace_bytes,
                             static_cast<cudaStream_t>(stream));
}

int nf_linear_link_units(int64_t groups, int64_t rows, int64_t k, int64_t n) {
  if (groups < 1 || rows < 1 || k < 1 || n < 1) return 0;
  return int(nf::linear_link_units(groups, rows, k, n));
}

int nf_conv_link_units(int N, int H, int W, int C, int Cout, int groups, int kernel, int stride,
                       int pad) {
  return int(nf::conv_link_units(N, H, W, C, Cout, groups, kernel, stride, pad));
}

static bool link_args(const void* dep_x, uint32_t tx, const void* dep_r, uint32_t tr,
                      void* done, int gpi, nf::LinkSpec* l) {
  if (gpi < 1 || (dep_x && tx < 1) || (dep_r && tr < 1)) return false;
  *l = nf::LinkSpec{static_cast<const unsigned*>(dep_x), tx, static_cast<const unsigned*>(dep_r),
                    tr, static_cast<unsigned*>(done), gpi};
  return true;
}

int nf_grouped_linear_linked(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                             const void* bias, const void* residual, void* y, int64_t y_ld,
                             int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                             int act, void* workspace, int64_t workspace_bytes,
                             const void* dep_x, uint32_t dep_x_target, const void* dep_r,
                             uint32_t dep_r_target, void* done, int groups_per_instance,
                             void* stream) {
  if (!x || !w || !y || groups < 1 || rows < 1 || k < 1 || n < 1) return NF_ERR_SHAPE;
  if (x_ld < k || y_ld < n || (groups > 1 && (x_gs < 1 || y_gs < 1))) return NF_ERR_SHAPE;
  if (act < NF_ACT_NONE || act > NF_ACT_TANH) return NF_ERR_UNSUPPORTED;
  nf::LinkSpec l;
  if (!link_args(dep_x, dep_x_target, dep_r, dep_r_target, done, groups_per_instance, &l))
    return NF_ERR_SHAPE;
  return nf::grouped_linear_tc(x, x_ld, x_gs, w, static_cast<const float*>(bias), residual, y,
                               y_ld, y_gs, groups, rows, k, n, NF_BF16, act, workspace,
                               workspace_bytes, static_cast<cudaStream_t>(stream), nullptr, &l);
}

int nf_grouped_conv_tc_linked(const void* x, const void* w, const float* bias,
                              const void* residual, void* y, int N, int H, int W, int C, int Cout,
                              int groups, int kernel, int stride, int pad, int kpad, int relu,
                              void* workspace, int64_t workspace_bytes, const void* dep_x,
                              uint32_t dep_x_target, const void* dep_r, uint32_t dep_r_target,
                              void* done, int groups_per_instance, void* stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || Cout < 1) return NF_ERR_SHAPE;
  nf::LinkSpec l;
  if (!link_args(dep_x, dep_x_target, dep_r, dep_r_target, done, groups_per_instance, &l))
    return NF_ERR_SHAPE;
  return nf::grouped_conv_tc(x, w, bias, residual, y, N, H, W, C, Cout, groups, kernel, stride,
                             pad, kpad, relu, workspace, workspace_bytes,
                             static_cast<cudaStream_t>(stream), &l);
}

int nf_grouped_conv_tf32(const void* x, const void* w, const float* bias, const void* residual,
                         void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                         int stride, int pad, int kpad, int relu, void* workspace,
                         int64_t workspace_bytes, void* stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || Cout < 1) return NF_ERR_SHAPE;
  return nf::grouped_conv_tf32(x, w, bias, residual, y, N, H, W, C, Cout, groups, kernel, stride,
                               pad, kpad, relu, workspace, workspace_bytes,
                               static_cast<cudaStream_t>(stream));
}

int64_t nf_conv_tf32_workspace_bytes(int N, int H, int W, int C, int Cout, int groups, int kernel,
                                     int stride, int pad, int kpad) {
  return nf::conv_tf32_workspace_bytes(N, H, W, C, Cout, groups, kernel, stride, pad, kpad);
}

int64_t nf_conv_workspace_bytes(int N, int H, int W, int C, int Cout, int groups, int kernel,
                                int stride, int pad, int kpad) {
  return nf::conv_workspace_bytes(N, H, W, C, Cout, groups, kernel, stride, pad, kpad);
}

int nf_qkv_attention(const void* x, int64_t x_ld, int64_t x_gs, const void* w, const float* bias,
                     void* out, int64_t groups, int64_t seq, int64_t d_model, int64_t heads,
                     float scale, void* stream) {
  if (!x || !w || !out) return NF_ERR_SHAPE;
  return nf::qkv_attention_tc(x, x_ld, x_gs, w, bias, out, groups, seq, d_model, heads, scale,
                              static_cast<cudaStream_t>(stream));
}

int nf_linear_fold_supported(int64_t groups, int64_t rows, int64_t k, int64_t n) {
  return nf::linear_fold_supported(groups, rows, k, n) ? 1 : 0;
}

int nf_grouped_linear_fold(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                           const void* bias, const void* residual, void* y, int64_t y_ld,
                           int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                           int act, void* workspace, int64_t workspace_bytes,
                           const float* in_stats, int in_parts, const float* in_colsum,
                           float in_eps, const float* res_stats, int res_parts,
                           const float* res_gamma, const float* res_beta, float res_eps,
                           float* out_stats, void* stream) {
  if (!x || !w || !y || groups < 1 || rows < 1 || k < 1 || n < 1) return NF_ERR_SHAPE;
  if (x_ld < k || y_ld < n || (groups > 1 && (x_gs < 1 || y_gs < 1))) return NF_ERR_SHAPE;
  if (act < NF_ACT_NONE || act > NF_ACT_TANH) return NF_ERR_UNSUPPORTED;
  const nf::NormFold fold{in_stats, in_colsum, in_parts, in_eps, res_stats,
                          res_gamma, res_beta, res_parts, res_eps, out_stats};
  return nf::grouped_linear_tc(x, x_ld, x_gs, w, static_cast<const float*>(bias), residual, y,
                               y_ld, y_gs, groups, rows, k, n, NF_BF16, act, workspace,
                               workspace_bytes, static_cast<cudaStream_t>(stream), &fold);
}

int nf_qkv_attention_fold(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                          const float* bias, void* out, int64_t groups, int64_t seq,
                          int64_t d_model, int64_t heads, float scale, const float* in_stats,
                          int in_parts, const float* in_colsum, float in_eps, void* stream) {
  if (!x || !w || !out) return NF_ERR_SHAPE;
  const nf::NormFold fold{in_stats, in_colsum, in_parts, in_eps, nullptr,
                          nullptr, nullptr, 0, 0.f, nullptr};
  return nf::qkv_attention_tc(x, x_ld, x_gs, w, bias, out, groups, seq, d_model, heads, scale,
                              static_cast<cudaStream_t>(stream), &fold);
}

int nf_space_to_depth_stem(const void* x, void* y, int N, int groups, int cg, int H, int W,
                           void* stream) {
  if (!x || !y) return NF_ERR_SHAPE;
  return nf::s2d_stem(x, y, N, groups, cg, H, W, static_cast<cudaStream_t>(stream));
}

int nf_linear_chain_supported(int64_t groups, int64_t rows, int64_t k, int64_t n) {
  return nf::linear_chain_supported(groups, rows, k, n) ? 1 : 0;
}

int64_t nf_linear_chain_counter_bytes(int n_ops, int64_t groups) {
  if (n_ops < 1 || groups < 1) return 0;
  // per-(op, instance) tile counters and the exit counter
  return (int64_t(n_ops) * groups + 1) * int64_t(sizeof(unsigned));
}

static int chain_entry(int n_ops, const nf_linear_op* ops, int64_t groups, void* counters,
                       void* stream, bool rearm, const unsigned* ext_dep = nullptr,
                       unsigned ext_target = 0) {
  if (!ops || !counters || n_ops < 1 || n_ops > 3 || groups < 1) return NF_ERR_SHAPE;
  nf::LinearOpDesc d[3];
  for (int j = 0; j < n_ops; ++j) {
    const nf_linear_op& o = ops[j];
    if (o.rows < 1 || o.k < 1 || o.n < 1 || o.x_ld < o.k || o.y_ld < o.n) return NF_ERR_SHAPE;
    if (groups > 1 && (o.x_gs < 1 || o.y_gs < 1)) return NF_ERR_SHAPE;
    if (o.act < NF_ACT_NONE || o.act > NF_ACT_TANH) return NF_ERR_UNSUPPORTED;
    d[j] = nf::LinearOpDesc{o.x, o.x_ld, o.x_gs, o.w, o.bias, o.residual, o.y, o.y_ld, o.y_gs,
                            groups, o.rows, o.k, o.n, o.act, o.workspace, o.workspace_bytes,
                            (o.in_stats || o.res_stats || o.out_stats) ? 1 : 0,
                            nf::NormFold{o.in_stats, o.in_colsum, o.in_parts, o.in_eps,
                                         o.res_stats, o.res_gamma, o.res_beta, o.res_parts,
                                         o.res_eps, o.out_stats}};
  }
  return nf::grouped_linear_chain_tc(n_ops, d, static_cast<unsigned*>(counters),
                                     static_cast<cudaStream_t>(stream), rearm, ext_dep,
                                     ext_target);
}

int nf_grouped_linear_chain(int n_ops, const nf_linear_op* ops, int64_t groups, void* counters,
                            void* stream) {
  return chain_entry(n_ops, ops, groups, counters, stream, true);
}

int nf_qkv_attention_after(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                           const float* bias, void* out, int64_t groups, int64_t seq,
                           int64_t d_model, int64_t heads, float scale, const float* in_stats,
                           int in_parts, const float* in_colsum, float in_eps,
                           const void* dep_counters, uint32_t dep_target,
                           void* done_counters, void* stream) {
  if (!x || !w || !out || (dep_counters && dep_target < 1)) return NF_ERR_SHAPE;
  const nf::NormFold fold{in_stats, in_colsum, in_parts, in_eps, nullptr,
                          nullptr, nullptr, 0, 0.f, nullptr};
  return nf::qkv_attention_tc(x, x_ld, x_gs, w, bias, out, groups, seq, d_model, heads, scale,
                              static_cast<cudaStream_t>(stream), in_stats ? &fold : nullptr,
                              static_cast<const unsigned*>(dep_counters), dep_target,
                              static_cast<unsigned*>(done_counters));
}

int nf_grouped_linear_chain_ex(int n_ops, const nf_linear_op* ops, int64_t groups,
                               void* counters, int flags, const void* dep_counters,
                               uint32_t dep_target, void* stream) {
  if (flags & ~NF_CHAIN_KEEP_COUNTERS) return NF_ERR_UNSUPPORTED;
  if (dep_counters && dep_target < 1) return NF_ERR_SHAPE;
  return chain_entry(n_ops, ops, groups, counters, stream, !(flags & NF_CHAIN_KEEP_COUNTERS),
                     static_cast<const unsigned*>(dep_counters), dep_target);
}

int nf_pool2d_nhwc(const void* x, void* y, int N, int H, int W, int C, int kind, int kernel,
                   int stride, int pad, int dtype, void* stream) {
  if (!x || !y || N < 1 || H < 1 || W < 1 || C < 1) return NF_ERR_SHAPE;
  if (kind != NF_POOL_MAX && kind != NF_POOL_MEAN) return NF_ERR_UNSUPPORTED;
  return nf::pool_nhwc(x, y, N, H, W, C, kind, kernel, stride, pad, dtype,
                       static_cast<cudaStream_t>(stream));
}

}  // extern "C"
