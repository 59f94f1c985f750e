// extern "C" entry points: argument validation, dispatch to the kernel
// launchers, status mapping. See include/netfuse_b200.h for the contract.
#include "common.cuh"
#include "kernels.h"

extern "C" {

int nf_abi_version(void) { return 1; }

const char* nf_status_string(int status) {
  switch (status) {
    case NF_OK: return "ok";
    case NF_ERR_SHAPE: return "bad shape or argument";
    case NF_ERR_UNSUPPORTED: return "unsupported dtype or configuration";
    case NF_ERR_LAUNCH: return "CUDA launch failure";
    default: return "unknown status";
  }
}

int nf_grouped_linear(const void* x, const void* w, const void* bias, const void* residual,
                      void* y, int64_t groups, int64_t rows, int64_t k, int64_t n, int dtype,
                      int w_layout, int act, int mode, void* stream) {
  if (!x || !w || !y || groups < 1 || rows < 1 || k < 1 || n < 1) return NF_ERR_SHAPE;
  if (dtype != NF_F32 && dtype != NF_BF16) return NF_ERR_UNSUPPORTED;
  if (w_layout != NF_W_NK && w_layout != NF_W_KN) return NF_ERR_UNSUPPORTED;
  if (act < NF_ACT_NONE || act > NF_ACT_TANH) return NF_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float* b = static_cast<const float*>(bias);
  if (mode == NF_MODE_FAST && dtype == NF_BF16 && w_layout == NF_W_NK) {
    int st = nf::grouped_linear_tc(x, w, b, residual, y, groups, rows, k, n, dtype, act, s);
    if (st != NF_ERR_UNSUPPORTED) return st;
  }
  return nf::grouped_linear_simt(x, w, b, residual, y, groups, rows, k, n, dtype, w_layout, act,
                                 mode == NF_MODE_EXACT, s);
}

}  // extern "C"
