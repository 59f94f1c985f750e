// Standalone phase trace of k_attention_tc (CTA 0), BERT shapes.
#include "../paper_2009_13062_b200/csrc/attention.cu"
#include <cstdio>
#include <vector>
int main() {
  const int Bt = 8, S = 128, H = 12, dh = 64;
  size_t n = size_t(Bt) * S * 3 * H * dh;
  void *qkv, *out;
  cudaMalloc(&qkv, n * 2); cudaMalloc(&out, n / 3 * 2); cudaMemset(qkv, 0, n * 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0);
    int st = nf::attention(qkv, out, Bt, S, H, dh, 0.125f, NF_BF16, NF_MODE_FAST, 0);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("iter %d st %d %.2f us\n", it, st, ms * 1e3);
  }
  unsigned long long tr[64];
  cudaMemcpyFromSymbol(tr, nf::g_attn_trace, sizeof(tr));
  const char* names[] = {"start(after alloc)", "qkv loaded", "S=QK^T ready", "P staged", "O ready", "end"};
  for (int i = 0; i < 6; ++i) printf("%-20s %6lld ns\n", names[i], (long long)(tr[i] - tr[0]));
  printf("tmem loaded %lld, max done %lld, exp+stores done %lld\n", (long long)(tr[10] - tr[0]),
         (long long)(tr[11] - tr[0]), (long long)(tr[12] - tr[0]));
}
