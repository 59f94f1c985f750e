// Per-CTA pipeline timeline of the tcgen05 grouped GEMM (globaltimer ns,
// relative to the end of a stamp kernel launched just before it, PDL off).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DNF_GEMM_TRACE \
//        -I include -I paper_2009_13062_b200/csrc tools/gemm_trace.cu -o build/gemm_trace -lcuda
//   NF_PDL=0 build/gemm_trace G T K N
#include "../paper_2009_13062_b200/csrc/gemm_sm100.cu"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ unsigned long long g_stamp;
__global__ void stamp_kernel() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_stamp = t;
}

int main(int argc, char** argv) {
  int G = argc > 1 ? atoi(argv[1]) : 8, T = argc > 2 ? atoi(argv[2]) : 128;
  int K = argc > 3 ? atoi(argv[3]) : 768, N = argc > 4 ? atoi(argv[4]) : 2304;
  size_t nx = size_t(G) * T * K, nw = size_t(G) * N * K, ny = size_t(G) * T * N;
  void *x, *w, *y, *flush;
  cudaMalloc(&x, nx * 2);
  cudaMalloc(&w, nw * 2);
  cudaMalloc(&y, ny * 2);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(x, 0, nx * 2);
  cudaMemset(w, 0, nw * 2);
  int64_t ws_bytes = nf::linear_workspace_bytes(G, T, K, N);
  void* ws = nullptr;
  if (ws_bytes) { cudaMalloc(&ws, ws_bytes); cudaMemset(ws, 0, ws_bytes); }
  const char* names[8] = {"entry", "setup", "first_stage|ln_partials", "last_mma", "acc0_ready",
                          "epi_done", "exit", "ln_stats"};
  const bool warm = getenv("NF_TRACE_WARM") != nullptr;  // keep operands L2-resident
  const char* acts = getenv("NF_TRACE_ACT");            // none | relu | gelu
  const int act = !acts ? NF_ACT_NONE : (acts[0] == 'g' ? NF_ACT_GELU : acts[0] == 'r' ? NF_ACT_RELU : NF_ACT_NONE);
  void* res = nullptr;
  if (getenv("NF_TRACE_RES")) { cudaMalloc(&res, ny * 2); cudaMemset(res, 0, ny * 2); }
  float* bias = nullptr;
  cudaMalloc(&bias, size_t(G) * N * 4);
  cudaMemset(bias, 0, size_t(G) * N * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    if (!warm) cudaMemset(flush, it, 256 << 20);
    stamp_kernel<<<1, 1>>>();
    cudaEventRecord(e0);
    int st = nf::grouped_linear_tc(x, K, int64_t(T) * K, w, bias, res, y, N, int64_t(T) * N, G, T,
                                   K, N, NF_BF16, act, ws, ws_bytes, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (st || e) { printf("status %d err %s\n", st, cudaGetErrorString(e)); return 1; }
    if (it < 2) continue;
    std::vector<unsigned long long> tr(148 * 8);
    unsigned long long t0;
    cudaMemcpyFromSymbol(tr.data(), nf::g_gemm_trace, sizeof(unsigned long long) * 148 * 8);
    cudaMemcpyFromSymbol(&t0, g_stamp, sizeof(t0));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("G=%d T=%d K=%d N=%d act=%d res=%d workspace=%lld  kernel %.2f us  %.1f TFLOP/s\n", G, T, K,
           N, act, res != nullptr, (long long)ws_bytes, ms * 1e3,
           2.0 * G * T * K * N / (ms * 1e-3) / 1e12);
    {
      std::vector<unsigned long long> wt(148 * 8);
      cudaMemcpyFromSymbol(wt.data(), nf::g_gemm_wait, sizeof(unsigned long long) * 148 * 8);
      const char* wn[5] = {"prod<-empty", "mma<-full", "mma<-tempty", "epi<-tfull", "epi busy"};
      for (int s = 0; s < 5; ++s) {
        double tot = 0, mx = 0;
        for (int b = 0; b < 148; ++b) { tot += wt[b * 8 + s]; mx = std::max(mx, double(wt[b * 8 + s])); }
        printf("  wait %-12s mean %8.2f us  max %8.2f us (summed over 3 runs; mma/epi rows: lane 0 / thread 0 only)\n", wn[s], tot / 148 * 1e-3, mx * 1e-3);
      }
    }
    for (int s = 0; s < 8; ++s) {
      std::vector<double> v;
      for (int b = 0; b < 148; ++b)
        if (tr[b * 8 + s] > t0 && tr[b * 8 + s] - t0 < 100000000ull) v.push_back((tr[b * 8 + s] - t0) * 1e-3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      printf("  %-12s n=%3zu  min %7.2f  med %7.2f  max %7.2f us\n", names[s], v.size(), v[0],
             v[v.size() / 2], v.back());
    }
  }
  return 0;
}
