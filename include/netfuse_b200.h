/*
 * netfuse_b200.h — C ABI of the B200 (sm_100a) merged-operator kernels.
 *
 * This is the drop-in boundary for the NetFuse hot path. The reference
 * (`modelmerge`, pure Python + numpy) has no native code; its "operator API"
 * is the set of kernel functions in pkg/src/modelmerge/engine.py dispatched by
 * the if-chain in `_run_node` (engine.py:456-510). Each entry point below
 * replaces one of those kernels (cited per function) for the merged
 * (instance-packed) shapes the merger emits.
 *
 * Conventions (all entry points):
 *   - Plain device pointers and sizes; the caller allocates every output and
 *     workspace. Kernels never allocate, never synchronise, never touch host
 *     memory, so every call is CUDA-graph capturable.
 *   - `stream` is a cudaStream_t passed as void*; work is stream-ordered.
 *   - Return value: NF_OK, or NF_ERR_SHAPE (the reference's ShapeError,
 *     errors.py:34), NF_ERR_UNSUPPORTED (UnsupportedOpError, errors.py:38),
 *     NF_ERR_LAUNCH (a CUDA launch failure; surfaced as ExecutionError,
 *     errors.py:54). The Python shim adds the node id, as engine.py:549 does.
 *   - No mutable global state: TMA descriptors are built per call and passed
 *     as __grid_constant__ kernel parameters.
 */
#ifndef NETFUSE_B200_H
#define NETFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define NF_OK 0
#define NF_ERR_SHAPE 1
#define NF_ERR_UNSUPPORTED 2
#define NF_ERR_LAUNCH 3

/* element types */
#define NF_F32 0
#define NF_BF16 1

/* fused epilogue activations */
#define NF_ACT_NONE 0
#define NF_ACT_RELU 1
#define NF_ACT_GELU 2
#define NF_ACT_TANH 3

/* arithmetic mode: FAST = tensor-core / reordered FMA paths;
 * EXACT = the reference's accumulation order with separately rounded
 * multiply and add (engine.py:1-21), bit-identical to the numpy kernels. */
#define NF_MODE_FAST 0
#define NF_MODE_EXACT 1

/* elementwise ops (nf_elementwise) */
#define NF_EW_ADD 0
#define NF_EW_MUL 1
#define NF_EW_RELU 2
#define NF_EW_TANH 3
#define NF_EW_GELU 4

/* pooling kinds (nf_pool2d) */
#define NF_POOL_MAX 0
#define NF_POOL_MEAN 1

/* max rank handled by nf_copy_strided */
#define NF_MAX_RANK 8

/* weight layouts for nf_grouped_linear */
#define NF_W_NK 0 /* (G, N, K): K-major, the kernel-native merged layout   */
#define NF_W_KN 1 /* (G, K, N): the reference layout (rules.py:180-184)    */

/* ABI version, bumped on any signature change. */
int nf_abi_version(void);

/* Human-readable name for a status code (static storage). */
const char* nf_status_string(int status);

/*
 * Merged Linear == reference `batch_matmul` (engine.py:215-235), and with
 * groups=1 the unmerged `matmul` (engine.py:194-212):
 *   y[g, t, :] = act(x[g, t, :] @ W[g] + bias[g] + residual[g, t, :])
 * x: (groups, rows, k) row-major; W per `w_layout`; bias: (groups, n) or NULL;
 * residual: (groups, rows, n) or NULL; y: (groups, rows, n).
 * FAST bf16 runs a tcgen05/TMEM/TMA tile kernel (weights streamed once per
 * instance); EXACT f32 reproduces the reference accumulation order bit for
 * bit (k ascending, mul and add each rounded, bias added after).
 */
int nf_grouped_linear(const void* x, const void* w, const void* bias, const void* residual,
                      void* y, int64_t groups, int64_t rows, int64_t k, int64_t n, int dtype,
                      int w_layout, int act, int mode, void* stream);

/*
 * nf_grouped_linear with explicit element strides: x row r of group g at
 * x + g*x_gs + r*x_ld (x_ld >= k), y (and residual) at y + g*y_gs + r*y_ld.
 * Lets the executor feed the GEMM strided views (e.g. the first-token rows of
 * every instance's encoder output, or a padded output width) without copies.
 * Strides must keep 16-byte row alignment for the tensor-core path.
 */
int nf_grouped_linear_strided(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                              const void* bias, const void* residual, void* y, int64_t y_ld,
                              int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                              int dtype, int w_layout, int act, int mode, void* stream);

/*
 * NHWC helpers for merged convs lowered to grouped GEMMs (reference
 * `grouped_conv2d`, engine.py:155-191): im2col rows [pixel][group][Kpad]
 * with column (kh*k + kw)*Cg + c (zeros beyond k*k*Cg), x NHWC (N,H,W,C).
 */
int nf_im2col_nhwc(const void* x, void* y, int N, int H, int W, int C, int groups, int kernel,
                   int stride, int pad, int kpad, int dtype, void* stream);

/*
 * Direct NHWC grouped conv for small groups (ResNeXt 4..32 channels / group):
 * w (Cout, kh, kw, Cin/groups), y = relu?(conv + bias[c] + residual), fp32
 * bias (folded BN shift) or NULL, residual NHWC like y or NULL.
 */
int nf_conv_nhwc_direct(const void* x, const void* w, const float* bias, const void* residual,
                        void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                        int stride, int pad, int relu, int dtype, void* stream);

/*
 * Merged / grouped Conv2d as an implicit GEMM on the tensor cores (replaces
 * reference `grouped_conv2d` / `conv2d`, engine.py:122-191, for the
 * BN-folded bf16 CNN plans). x NHWC (N, H, W, C) bf16, w (groups, Cout/groups,
 * kpad) bf16 K-major with K = (kh*k + kw)*(C/groups) + c zero-padded to kpad,
 * bias fp32 (Cout) or NULL, residual NHWC like y or NULL, y NHWC
 * (N, Ho, Wo, Cout) = relu?(conv + bias + residual). Needs C/groups % 4 == 0
 * and Cout/groups % 4 == 0. workspace (from nf_conv_workspace_bytes, zeroed
 * once) enables split-K; NULL disables it.
 */
int nf_grouped_conv_tc(const void* x, const void* w, const float* bias, const void* residual,
                       void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                       int stride, int pad, int kpad, int relu, void* workspace,
                       int64_t workspace_bytes, void* stream);
int64_t nf_conv_workspace_bytes(int N, int H, int W, int C, int Cout, int groups, int kernel,
                                int stride, int pad, int kpad);

/*
 * fp32 merged Conv2d on the tensor cores (3xTF32): reference `grouped_conv2d`
 * (engine.py:155-191) / `conv2d` (122-152) at fp32 accuracy for the fp32
 * configuration. x NHWC fp32 (N, H, W, C), C = groups * cg with cg % 4 == 0;
 * w (2 * groups, Cout/groups, kpad) fp32 K-major with K = (kh, kw, c) zero
 * padded to kpad (a multiple of 32): groups [0, G) hold hi = w with the low
 * 13 mantissa bits cleared, [G, 2G) lo = w - hi; bias (Cout) fp32 or NULL
 * (BatchNorm folded); residual / y NHWC fp32 (N, Ho, Wo, Cout); y =
 * relu?(conv + bias + residual). The activation operand is split the same
 * way on chip; each K step issues lo*hi + hi*lo + hi*hi (fp32 accumulate in
 * TMEM): ~2^-20 relative per product. Split-K workspace as
 * nf_grouped_conv_tc (nf_conv_tf32_workspace_bytes; zeroed once).
 */
int nf_grouped_conv_tf32(const void* x, const void* w, const float* bias, const void* residual,
                         void* y, int N, int H, int W, int C, int Cout, int groups, int kernel,
                         int stride, int pad, int kpad, int relu, void* workspace,
                         int64_t workspace_bytes, void* stream);
int64_t nf_conv_tf32_workspace_bytes(int N, int H, int W, int C, int Cout, int groups, int kernel,
                                     int stride, int pad, int kpad);

/*
 * Fused merged QKV projection + attention for batch-1 encoders (the merged
 * graph's BatchMatMul(qkv) -> Attention pair: reference `batch_matmul`,
 * engine.py:215-235, then the attention restatement). x (G, S=128, D) bf16
 * rows at x + g*x_gs + t*x_ld; w (G, 3D, D) K-major bf16 with head-major
 * rows: row h*192 + p*64 + j holds output feature p*D + h*64 + j (p = 0 q,
 * 1 k, 2 v), so a head's 192 rows are one TMA box; bias (G, 3D) fp32 in
 * feature order or NULL; out (G, S, D) bf16 context of heads of 64; D a
 * multiple of 64. One CTA per (instance, head); QKV never reaches HBM.
 */
int nf_qkv_attention(const void* x, int64_t x_ld, int64_t x_gs, const void* w, const float* bias,
                     void* out, int64_t groups, int64_t seq, int64_t d_model, int64_t heads,
                     float scale, void* stream);

/*
 * Folded LayerNorm (batch-1 encoders). The merged graph's Add -> GroupNorm
 * over each instance's D features (reference add engine.py:322-325,
 * group_norm 263-284) is not launched: the Linear producing the Add's
 * operand adds the residual in its epilogue and writes per-token statistics
 * `out_stats` [g][part][token] (sum, centred sum of squares M2 about the
 * part's own mean; part = 128-feature tile, n/128 parts). Consumers merge the
 * parts (Chan et al.: no E[x^2] - mean^2 cancellation, so the result does not
 * degrade with |mean| / std) and rebuild LN(v) from the raw v:
 *  - as the activations of a Linear (in_*): w holds gamma-scaled weights
 *    W'[g][n][k] = W[g][n][k] * gamma[g][k], bias b' = b + W beta, in_colsum
 *    (G, n) = sum_k W'[g][n][k]; y = rstd * (x W'^T - mean * colsum) + b';
 *  - as the residual (res_*): (r - mean) * rstd * res_gamma + res_beta.
 * nf_linear_fold_supported(...) is 1 where the kernel implements it (the
 * swapped 128-token tile path, n a multiple of 128); elsewhere the fold
 * entry points return 2.
 * Statistics are fp32 and the reduction order fixed (deterministic).
 */
int nf_linear_fold_supported(int64_t groups, int64_t rows, int64_t k, int64_t n);
int nf_grouped_linear_fold(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                           const void* bias, const void* residual, void* y, int64_t y_ld,
                           int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                           int act, void* workspace, int64_t workspace_bytes,
                           const float* in_stats, int in_parts, const float* in_colsum,
                           float in_eps, const float* res_stats, int res_parts,
                           const float* res_gamma, const float* res_beta, float res_eps,
                           float* out_stats, void* stream);
int nf_qkv_attention_fold(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                          const float* bias, void* out, int64_t groups, int64_t seq,
                          int64_t d_model, int64_t heads, float scale, const float* in_stats,
                          int in_parts, const float* in_colsum, float in_eps, void* stream);

/*
 * Chained batch-1 merged Linears: n_ops (1..3) consecutive merged-Linear
 * nodes of one instance-packed model -- e.g. a BERT layer's attention
 * projection -> FF1 (+GELU) -> FF2, each the reference's `batch_matmul`
 * (engine.py:215-235) with the fused epilogue / folded LayerNorm operands of
 * nf_grouped_linear_fold -- in ONE persistent launch. ops[j].x must be
 * ops[j-1].y: op j's units of instance g load activations once op j-1 has
 * stored all of g's output tiles; weight tiles are requested before that,
 * so the weight stream never pauses at an op boundary. Results are bit-identical to calling nf_grouped_linear_fold per
 * op. Every op must satisfy nf_linear_chain_supported (the swapped 128-token
 * tile of batch-1 shapes: k % 64 == 0,
 * n % 128 == 0) and take at most one of the in_/res_ folds. `counters` holds
 * nf_linear_chain_counter_bytes(n_ops, groups) bytes, zeroed once; the
 * kernel leaves them zeroed (replayable). Each op's workspace enables its
 * split-K exactly as for nf_grouped_linear_ws.
 */
typedef struct nf_linear_op {
  const void* x;
  int64_t x_ld, x_gs;
  const void* w;
  const float* bias;
  const void* residual;
  void* y;
  int64_t y_ld, y_gs, rows, k, n;
  int act;
  void* workspace;
  int64_t workspace_bytes;
  const float* in_stats;
  int in_parts;
  const float* in_colsum;
  float in_eps;
  const float* res_stats;
  int res_parts;
  const float* res_gamma;
  const float* res_beta;
  float res_eps;
  float* out_stats;
} nf_linear_op;
int nf_linear_chain_supported(int64_t groups, int64_t rows, int64_t k, int64_t n);
int64_t nf_linear_chain_counter_bytes(int n_ops, int64_t groups);
int nf_grouped_linear_chain(int n_ops, const nf_linear_op* ops, int64_t groups, void* counters,
                            void* stream);
/*
 * Chained launch with options. flags: NF_CHAIN_KEEP_COUNTERS leaves the
 * per-instance counters set after the launch (counters[j*groups + g] = op
 * j's output tiles of instance g) for a later kernel to wait on (see
 * nf_qkv_attention_after); the caller zeroes them before every launch.
 * dep_counters (or NULL): a [groups] completion counter of the kernel that
 * produces ops[0]'s inputs (e.g. nf_qkv_attention_after's done_counters);
 * instance g's units of ops[0] start once dep_counters[g] >= dep_target
 * instead of waiting for that whole launch.
 */
#define NF_CHAIN_KEEP_COUNTERS 1
int nf_grouped_linear_chain_ex(int n_ops, const nf_linear_op* ops, int64_t groups,
                               void* counters, int flags, const void* dep_counters,
                               uint32_t dep_target, void* stream);
/*
 * nf_qkv_attention_fold with per-instance ordering. dep_counters (or NULL):
 * x (and its LayerNorm statistics) is the output of an earlier chained launch
 * (NF_CHAIN_KEEP_COUNTERS); instance g's CTAs start once dep_counters[g] >=
 * dep_target (that launch stored g's output tiles) instead of waiting for the
 * whole launch. done_counters (or NULL): each CTA adds 1 to done_counters[g]
 * once its head's context is stored (heads per instance = all done).
 */
int nf_qkv_attention_after(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                           const float* bias, void* out, int64_t groups, int64_t seq,
                           int64_t d_model, int64_t heads, float scale, const float* in_stats,
                           int in_parts, const float* in_colsum, float in_eps,
                           const void* dep_counters, uint32_t dep_target,
                           void* done_counters, void* stream);

/*
 * Per-instance launch linking for merged CNN / GEMM pipelines. Counters are
 * uint32 per instance (zeroed by the caller before each forward); instance of
 * group g = g / groups_per_instance. dep_x / dep_r (or NULL): counters of the
 * launches that produced x / the residual, with the number of output tiles
 * one instance of them publishes (dep_*_target, from nf_linear_link_units /
 * nf_conv_link_units x their groups per instance); a unit of instance m
 * starts once those counts are reached instead of waiting for the whole
 * previous launch. done (or NULL): this launch's counters, bumped once per
 * stored output tile. NULL dependencies wait for the previous launch as the
 * plain entry points do. Results are bit-identical to the plain entry points.
 */
int nf_linear_link_units(int64_t groups, int64_t rows, int64_t k, int64_t n);
int nf_conv_link_units(int N, int H, int W, int C, int Cout, int groups, int kernel, int stride,
                       int pad);
int nf_grouped_linear_linked(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                             const void* bias, const void* residual, void* y, int64_t y_ld,
                             int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                             int act, void* workspace, int64_t workspace_bytes,
                             const void* dep_x, uint32_t dep_x_target, const void* dep_r,
                             uint32_t dep_r_target, void* done, int groups_per_instance,
                             void* stream);
int nf_grouped_conv_tc_linked(const void* x, const void* w, const float* bias,
                              const void* residual, void* y, int N, int H, int W, int C, int Cout,
                              int groups, int kernel, int stride, int pad, int kpad, int relu,
                              void* workspace, int64_t workspace_bytes, const void* dep_x,
                              uint32_t dep_x_target, const void* dep_r, uint32_t dep_r_target,
                              void* done, int groups_per_instance, void* stream);

/* NHWC 2-D pooling (max: -inf padding; mean: window sum / k^2). */
int nf_pool2d_nhwc(const void* x, void* y, int N, int H, int W, int C, int kind, int kernel,
                   int stride, int pad, int dtype, void* stream);

/*
 * Split-K workspace for nf_grouped_linear_ws: bytes needed for this shape (0
 * when the tile count already covers the GPU). The workspace must be
 * zero-initialised once; kernels restore its semaphores before returning.
 */
int64_t nf_linear_workspace_bytes(int64_t groups, int64_t rows, int64_t k, int64_t n);

/*
 * nf_grouped_linear_strided plus a split-K workspace (NULL / 0 disables
 * split-K). Low-tile-count shapes (e.g. 8 instances x 768 features) split K
 * across otherwise idle SMs; partials reduce in split order (deterministic).
 */
int nf_grouped_linear_ws(const void* x, int64_t x_ld, int64_t x_gs, const void* w,
                         const void* bias, const void* residual, void* y, int64_t y_ld,
                         int64_t y_gs, int64_t groups, int64_t rows, int64_t k, int64_t n,
                         int dtype, int w_layout, int act, int mode, void* workspace,
                         int64_t workspace_bytes, void* stream);

/*
 * Merged Conv2d == reference `grouped_conv2d` (engine.py:155-191), and with
 * groups=1 `conv2d` (engine.py:122-152). NCHW x (N, Cin, H, W), w
 * (Cout, Cin/groups, k, k), y (N, Cout, Ho, Wo). Epilogue (FAST, for the
 * BN-folded CNN plans): y = relu?((acc * scale[c]) + bias[c] + residual);
 * scale/bias fp32 or NULL, residual like y or NULL. EXACT f32 follows the
 * reference accumulation order (ci, kh, kw; rounded mul then add; bias after).
 */
int nf_grouped_conv2d(const void* x, const void* w, const float* bias, const float* scale,
                      const void* residual, void* y, int64_t N, int64_t Cin, int64_t H,
                      int64_t W, int64_t Cout, int kernel, int stride, int pad, int groups,
                      int relu, int dtype, int mode, void* stream);

/*
 * Pointwise ops == reference `add`/`mul`/`relu`/`tanh` (engine.py:305-331)
 * plus GELU (extension). Dense over `n` elements; pointers 16-byte aligned.
 * add/mul are IEEE-rounded with no contraction: bit-exact vs numpy.
 */
int nf_elementwise(int op, const void* a, const void* b, void* y, int64_t n, int dtype,
                   void* stream);

/*
 * Space-to-depth repack of a merged RGB stem input (layout glue of the
 * 7x7/s2 stem lowered to a 4x4/s1 conv over 2x2 pixel blocks): x bf16 NCHW
 * (N, groups*cg, H, W) with cg <= 4 channels per instance and even H, W;
 * y bf16 NHWC (N, H/2+1, W/2+1, groups*16), row 0 and column 0 left untouched
 * (the caller zeroes them once): y[n, i+1, j+1, g*16 + (bh*2+bw)*4 + c] =
 * x[n, g*cg + c, 2i+bh, 2j+bw], channels c >= cg written as zero.
 */
int nf_space_to_depth_stem(const void* x, void* y, int N, int groups, int cg, int H, int W,
                           void* stream);

/*
 * Re-arm per-instance completion counters (linked launches) for the next
 * forward: zeroes `bytes` at `counters` with a memset on `stream`, ordered
 * with the stream's kernels (capturable into a CUDA graph). Replaces no
 * reference interface: the linked launches are this port's own schedule.
 */
int nf_counters_rearm(void* counters, int64_t bytes, void* stream);

/*
 * Layout glue: y[i0..] = x[i0..] over an up-to-8-D index space with
 * arbitrary element strides on both sides. Realises the merger's
 * Transpose/Reshape junctions (merger.py:237-301) and Pack/Unpack
 * (engine.py:380-420) when they cannot be zero-copy views.
 */
int nf_copy_strided(const void* x, void* y, int rank, const int64_t* dims,
                    const int64_t* x_strides, const int64_t* y_strides, int elem_bytes,
                    void* stream);

/*
 * Merged LayerNorm == reference `group_norm` (engine.py:263-284), and with
 * groups=1 `layer_norm` (engine.py:246-260). y = GN(x [+ residual]).
 * Row r = (r1, r2) at element offset r1*s1 + r2*s2 (r1 < R1, r2 < R2);
 * channel (g, c) of a row at g*sg + c*sc (g < G, c < Cg). gamma/beta are fp32
 * of length G*Cg, or (rows/rows_per_affine) blocks of G*Cg when
 * rows_per_affine > 0 (per-instance affine on a model-major layout). The
 * same geometry addresses y and residual. Covers the channel-packed layout
 * (B, S, M*D) and the model-major layout (M, B, S, D) without glue.
 */
int nf_group_norm(const void* x, const void* residual, const float* gamma, const float* beta,
                  void* y, int64_t R1, int64_t R2, int64_t s1, int64_t s2, int64_t G,
                  int64_t Cg, int64_t sg, int64_t sc, int64_t rows_per_affine, float eps,
                  int dtype, void* stream);

/*
 * Softmax along one axis == reference `softmax` (engine.py:313-319):
 * element (o, l, i) at o*so + l*sl + i*si for o < outer, l < L, i < inner.
 */
int nf_softmax(const void* x, void* y, int64_t outer, int64_t L, int64_t inner, int64_t so,
               int64_t sl, int64_t si, int dtype, void* stream);

/*
 * Merged attention (extension; the reference composes batch_matmul +
 * softmax): qkv (Bt, S, 3*H*dh) fused projection rows [Q | K | V], out
 * (Bt, S, H*dh) = softmax(Q K^T * scale) V per (sequence, head).
 * bf16 FAST with dh == 64 and S <= 128 runs the tcgen05/TMEM kernel.
 */
int nf_attention(const void* qkv, void* out, int64_t Bt, int64_t S, int64_t H, int64_t dh,
                 float scale, int dtype, int mode, void* stream);

/*
 * XLNet relative attention (extension; transformers XLNetRelativeAttention.
 * rel_attn_core, attn_type "bi", no segment term / mask): qkv (Bt, S, 3*H*dh),
 * r (Bt/seqs_per_r, 2S, H*dh) projected positional keys (one per
 * seqs_per_r consecutive sequences: the positional embedding is the same for
 * every sequence of an instance), r_w_bias / r_r_bias fp32
 * (Bt/seqs_per_bias, H, dh) per instance; out (Bt, S, H*dh) with
 * score_ij = ((q_i + r_w_bias) . k_j + (q_i + r_r_bias) . kr_{S-i+j}) * scale.
 */
int nf_rel_attention(const void* qkv, const void* r, const float* r_w_bias,
                     const float* r_r_bias, void* out, int64_t Bt, int64_t S, int64_t H,
                     int64_t dh, int64_t seqs_per_bias, int64_t seqs_per_r, float scale,
                     int dtype, int mode, void* stream);

/*
 * Inference batch norm == reference `batch_norm_inference`
 * (engine.py:287-302) on an NCHW tensor (N, C, inner); fp32 parameters.
 * Same operation order as numpy: bit-exact for f32.
 */
int nf_batch_norm(const void* x, const float* gamma, const float* beta, const float* mean,
                  const float* var, void* y, int64_t N, int64_t C, int64_t inner, float eps,
                  int dtype, void* stream);

/*
 * 2-D pooling == reference `max_pool2d` / `mean_pool2d` (engine.py:334-365)
 * on NCHW; extension: symmetric `pad` (-inf for max, zeros for mean).
 */
int nf_pool2d(const void* x, void* y, int64_t N, int64_t C, int H, int W, int kind, int kernel,
              int stride, int pad, int dtype, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NETFUSE_B200_H */
