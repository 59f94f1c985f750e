// Per-CTA timeline of the 3xTF32 implicit-GEMM conv (k_conv_tf32x3), PDL off:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DNF_TF32_TRACE -I include -I paper_2009_13062_b200/csrc tools/tf32_trace.cu \
//        -o tools/bin_tf32_trace -lcuda
//   tools/bin_tf32_trace N H W G cg coutg k stride pad
#include "../paper_2009_13062_b200/csrc/conv_tf32.cu"

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
  int v[9] = {1, 14, 14, 2, 256, 256, 3, 1, 1};
  for (int i = 0; i < 9 && i + 1 < argc; ++i) v[i] = atoi(argv[i + 1]);
  const int N = v[0], H = v[1], W = v[2], G = v[3], cg = v[4], coutg = v[5], k = v[6], st = v[7],
            pad = v[8];
  const int C = G * cg, Cout = G * coutg;
  const int Ho = (H + 2 * pad - k) / st + 1, Wo = (W + 2 * pad - k) / st + 1;
  const int kpad = (k * k * cg + 31) / 32 * 32;
  void *x, *w, *y, *b, *flush;
  cudaMalloc(&x, size_t(N) * H * W * C * 4);
  cudaMalloc(&w, size_t(2 * G) * coutg * kpad * 4);
  cudaMalloc(&y, size_t(N) * Ho * Wo * Cout * 4);
  cudaMalloc(&b, size_t(Cout) * 4);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(x, 0, size_t(N) * H * W * C * 4);
  cudaMemset(w, 0, size_t(2 * G) * coutg * kpad * 4);
  cudaMemset(b, 0, size_t(Cout) * 4);
  int64_t ws_bytes = nf::conv_tf32_workspace_bytes(N, H, W, C, Cout, G, k, st, pad, kpad);
  void* ws = nullptr;
  if (ws_bytes) { cudaMalloc(&ws, ws_bytes); cudaMemset(ws, 0, ws_bytes); }
  const char* names[8] = {"entry", "setup", "first_stage", "last_mma", "acc_ready",
                          "partial_pub", "all_partials", "-"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemset(flush, it, 256 << 20);
    stamp_kernel<<<1, 1>>>();
    cudaEventRecord(e0);
    int s = nf::grouped_conv_tf32(x, w, static_cast<float*>(b), nullptr, y, N, H, W, C, Cout, G,
                                  k, st, pad, kpad, 1, ws, ws_bytes, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (s || e) { printf("status %d err %s\n", s, cudaGetErrorString(e)); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it < 2) continue;
    printf("tf32 conv N=%d %dx%d G=%d cg=%d coutg=%d k=%d s=%d p=%d ws=%lld  event %.2f us\n", N,
           H, W, G, cg, coutg, k, st, pad, (long long)ws_bytes, ms * 1e3);
    std::vector<unsigned long long> tr(148 * 8);
    unsigned long long t0;
    cudaMemcpyFromSymbol(tr.data(), nf::g_tf32_trace, sizeof(unsigned long long) * 148 * 8);
    cudaMemcpyFromSymbol(&t0, g_stamp, sizeof(t0));
    for (int q = 0; q < 7; ++q) {
      std::vector<double> vv;
      for (int bb = 0; bb < 148; ++bb)
        if (tr[bb * 8 + q] > t0 && tr[bb * 8 + q] - t0 < 100000000ull)
          vv.push_back((tr[bb * 8 + q] - t0) * 1e-3);
      if (vv.empty()) continue;
      std::sort(vv.begin(), vv.end());
      printf("  %-12s n=%3zu  min %7.2f  med %7.2f  max %7.2f us\n", names[q], vv.size(), vv[0],
             vv[vv.size() / 2], vv.back());
    }
  }
  return 0;
}
