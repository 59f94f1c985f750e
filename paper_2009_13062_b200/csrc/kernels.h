// Internal (C++) launcher declarations shared between the kernel translation
// units and the C ABI in capi.cu. Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

// gemm_sm100.cu — tcgen05 grouped GEMM (bf16 in, fp32 accumulate).
int grouped_linear_tc(const void* x, const void* w, const float* bias, const void* residual,
                      void* y, int64_t G, int64_t T, int64_t K, int64_t N, int out_dtype, int act,
                      cudaStream_t stream);

// linear_simt.cu — CUDA-core grouped linear (exact reference order or FMA).
int grouped_linear_simt(const void* x, const void* w, const float* bias, const void* residual,
                        void* y, int64_t G, int64_t T, int64_t K, int64_t N, int dtype,
                        int w_layout, int act, int exact, cudaStream_t stream);

}  // namespace nf
