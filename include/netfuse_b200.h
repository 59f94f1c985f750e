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
 *   y[g, t, :] = act(x[g, t, :] @ W[g] + bias[g]) + residual[g, t, :]
 * x: (groups, rows, k) row-major; W per `w_layout`; bias: (groups, n) or NULL;
 * residual: (groups, rows, n) or NULL; y: (groups, rows, n).
 * FAST bf16 runs a tcgen05/TMEM/TMA tile kernel (weights streamed once per
 * instance); EXACT f32 reproduces the reference accumulation order bit for
 * bit (k ascending, mul and add each rounded, bias added after).
 */
int nf_grouped_linear(const void* x, const void* w, const void* bias, const void* residual,
                      void* y, int64_t groups, int64_t rows, int64_t k, int64_t n, int dtype,
                      int w_layout, int act, int mode, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NETFUSE_B200_H */
