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
  int64_t ws_bytes = nf::linear_workspace_bytes(G, T, K, N);
  void* ws = nullptr;
  if (ws_bytes) { cudaMalloc(&ws, ws_bytes); cudaMemset(ws, 0, ws_bytes); }
  printf("workspace %lld bytes\n", (long long)ws_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    int st = nf::grouped_linear_tc(x, K, int64_t(T) * K, w, nullptr, nullptr, y, N, int64_t(T) * N,
                                   G, T, K, N, NF_BF16, 0, ws, ws_bytes, 0);
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
  printf("end=%lld\n", (long long)(tr[2] - t0));
  for (int l = 0; l < 4; ++l)
    if (tr[1 + 4 * l] > t0)
      printf("unit %d: acc ready %lld  partial published %lld  stored %lld\n", l,
             (long long)(tr[1 + 4 * l] - t0), tr[3 + 4 * l] > t0 ? (long long)(tr[3 + 4 * l] - t0) : -1LL,
             tr[4 + 4 * l] > t0 ? (long long)(tr[4 + 4 * l] - t0) : -1LL);
  (void)num_kb;
  return 0;
}
