// Standalone instrumented run of the tcgen05 grouped GEMM: timestamps
// (globaltimer, ns) of CTA (0,0,0)'s pipeline events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNF_GEMM_TRACE \
//        -I include -I paper_2009_13062_b200/csrc tools/gemm_trace.cu -o build/gemm_trace -lcuda
#include "../paper_2009_13062_b200/csrc/gemm_sm100.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  int G = argc > 1 ? atoi(argv[1]) : 8, T = argc > 2 ? atoi(argv[2]) : 128;
  int K = argc > 3 ? atoi(argv[3]) : 3072, N = argc > 4 ? atoi(argv[4]) : 768;
  size_t nx = size_t(G) * T * K, nw = size_t(G) * N * K, ny = size_t(G) * T * N;
  void *x, *w, *y;
  cudaMalloc(&x, nx * 2);
  cudaMalloc(&w, nw * 2);
  cudaMalloc(&y, ny * 2);
  cudaMemset(x, 0, nx * 2);
  cudaMemset(w, 0, nw * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    int st = nf::grouped_linear_tc(x, w, nullptr, nullptr, y, G, T, K, N, NF_BF16, 0, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("iter %d status %d err %s  %.2f us\n", it, st, cudaGetErrorString(e), ms * 1e3);
  }
  std::vector<unsigned long long> tr(4096);
  cudaMemcpyFromSymbol(tr.data(), nf::g_gemm_trace, sizeof(unsigned long long) * 4096);
  unsigned long long t0 = tr[0];
  int num_kb = (K + 63) / 64;
  printf("start=0  epi_start=%lld  end=%lld\n", (long long)(tr[1] - t0), (long long)(tr[2] - t0));
  for (int i = 10; i < 18; ++i) if (tr[i]) printf("  chunk %d ld done %lld\n", i - 10, (long long)(tr[i] - t0));
  printf("  staged %lld  barrier %lld  stored %lld\n", (long long)(tr[3] - t0), (long long)(tr[4] - t0), (long long)(tr[5] - t0));
  for (int kb = 0; kb < num_kb; ++kb)
    printf("kb %3d  producer_free %8lld  mma_full %8lld\n", kb,
           tr[100 + kb] ? (long long)(tr[100 + kb] - t0) : -1LL,
           (long long)(tr[1000 + kb] - t0));
  return 0;
}
