// TMA delivery-bandwidth probe: how many operand bytes per clock can each SM
// ingest from L2 through cp.async.bulk.tensor, unicast vs cluster multicast?
// Every CTA consumes 32 KB stages (A 128x64 + B 128x64 bf16 boxes, the
// pair-GEMM per-CTA stage). With multicast (cluster of C), the C CTAs of a
// cluster share the A tile: CTA r loads rows [r*128/C, (r+1)*128/C) once and
// multicasts them into every cluster CTA; B stays per CTA. No MMA — pure
// delivery rate, so the GEMM main loop's ceiling is this number.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2009_13062_b200/csrc tools/tma_mc_probe.cu -o tools/bin_tma_mc_probe -lcuda
#include "../paper_2009_13062_b200/csrc/gemm_sm100.cuh"

#include <cstdio>
#include <cstdlib>

using namespace nf;

constexpr int kStages = 6;
constexpr int kStageBytes = 32768;

NF_DEVICE void tma_load_3d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                              int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

template <int C>
__global__ void __launch_bounds__(64, 1)
    k_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int iters,
            int G, int rows_a, int rows_b, int kblocks) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = C > 1 ? cluster_ctarank() : 0;
  const int cluster_id = blockIdx.x / C, clusters = gridDim.x / C;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C);
    }
    fence_barrier_init();
  }
  if (C > 1) cluster_sync(); else __syncthreads();
  const int tiles_a = rows_a / 128, tiles_b = rows_b / 128;
  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      // unit: (instance, A tile shared by the cluster, B tile per CTA), k block
      const int kb = it % kblocks;
      const int u = it / kblocks;
      const int g = (cluster_id + u * clusters) % G;
      const int ta = (cluster_id / G + u) % tiles_a;
      const int tb = (int(rank) + cluster_id + u) % tiles_b;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      uint8_t* st = smem + s * kStageBytes;
      if (C == 1) {
        tma_load_3d(st, &ma, &full[s], kb * 64, ta * 128, g, kEvictNormal);
      } else {
        constexpr int rows = 128 / C;
        tma_load_3d_mc(st + rank * rows * 128, &ma, &full[s], kb * 64, ta * 128 + rank * rows, g,
                       uint16_t((1u << C) - 1));
      }
      tma_load_3d(st + 16384, &mb, &full[s], kb * 64, tb * 128, g, kEvictNormal);
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // consumer: one lane per cluster CTA releases the stage in that CTA
    // (relaxed remote arrivals issued in parallel; a serial chain of
    // release.cluster arrivals costs ~0.5 us each)
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[s], ph);
      if (C == 1) {
        if (lane == 0) mbar_arrive(&empty[s]);
      } else if (lane < C) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(lane));
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
      __syncwarp();
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
  }
  if (C > 1) cluster_sync(); else __syncthreads();
}

static bool map3(CUtensorMap* m, void* base, int G, int rows, int K, int box_rows) {
  cuuint64_t dims[3] = {cuuint64_t(K), cuuint64_t(rows), cuuint64_t(G)};
  cuuint64_t strides[2] = {cuuint64_t(K) * 2, cuuint64_t(rows) * K * 2};
  cuuint32_t box[3] = {64, cuuint32_t(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == 0;
}

template <int C>
static void run(void* a, void* b, int G, int ra, int rb, int K, int grid, int iters) {
  CUtensorMap ma, mb;
  if (!map3(&ma, a, G, ra, K, 128 / C) || !map3(&mb, b, G, rb, K, 128)) { printf("map fail\n"); exit(1); }
  const int smem = kStages * kStageBytes + 1024;
  cudaFuncSetAttribute(k_probe<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  grid = grid / C * C;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k_probe<C>, ma, mb, iters, G, ra, rb, K / 64);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    if (err || e2) { printf("C=%d err %s %s\n", C, cudaGetErrorString(err), cudaGetErrorString(e2)); exit(1); }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double bytes = double(grid) * iters * kStageBytes;
  const double l2_bytes = double(grid) * iters * (16384 + 16384.0 / C);
  printf("{\"cluster\": %d, \"grid\": %d, \"ms\": %.3f, \"delivered_TBps\": %.2f, \"delivered_B_per_clk_per_SM\": %.1f, "
         "\"l2_read_TBps\": %.2f}\n",
         C, grid, best, bytes / best / 1e9, bytes / (best * 1e-3) / 1.965e9 / grid,
         l2_bytes / best / 1e9);
}

int main(int argc, char** argv) {
  const int G = 32, K = 768;
  const int ra = argc > 1 ? atoi(argv[1]) : 1024, rb = argc > 2 ? atoi(argv[2]) : 768;
  const int iters = argc > 3 ? atoi(argv[3]) : 4000;
  void *a, *b;
  cudaMalloc(&a, size_t(G) * ra * K * 2);
  cudaMalloc(&b, size_t(G) * rb * K * 2);
  cudaMemset(a, 0, size_t(G) * ra * K * 2);
  cudaMemset(b, 0, size_t(G) * rb * K * 2);
  run<1>(a, b, G, ra, rb, K, 148, iters);
  run<2>(a, b, G, ra, rb, K, 148, iters);
  run<4>(a, b, G, ra, rb, K, 148, iters);
  run<8>(a, b, G, ra, rb, K, 144, iters);
  run<1>(a, b, G, ra, rb, K, 144, iters);
  return 0;
}
