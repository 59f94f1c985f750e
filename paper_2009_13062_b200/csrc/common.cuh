// Shared device helpers for the NetFuse B200 kernels (sm_100a only).
//
// Everything here is a thin inline-PTX wrapper: mbarriers, TMA bulk-tensor
// loads, tcgen05 (TMEM alloc / MMA / commit / ld) and the UMMA shared-memory
// and instruction descriptors. No global state lives in this header.
#pragma once
#include <atomic>

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/netfuse_b200.h"

#ifndef NF_DEVICE
#define NF_DEVICE __device__ __forceinline__
#endif

namespace nf {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// Dtype helpers
// ---------------------------------------------------------------------------
NF_DEVICE float to_f32(float v) { return v; }
NF_DEVICE float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> NF_DEVICE T from_f32(float v);
template <> NF_DEVICE float from_f32<float>(float v) { return v; }
template <> NF_DEVICE __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// erf via Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7): one exp, one
// reciprocal and a degree-5 polynomial instead of the libdevice erff.
NF_DEVICE float erf_fast(float x) {
  const float a = fabsf(x);
  const float t = __fdividef(1.0f, fmaf(0.3275911f, a, 1.0f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  const float r = 1.0f - p * t * __expf(-a * a);
  return copysignf(r, x);
}

NF_DEVICE float gelu_erf(float x) {
  // 0.5 x (1 + erf(x / sqrt(2))): the transformers "gelu" (exact erf form).
  return 0.5f * x * (1.0f + erf_fast(x * 0.70710678118654752440f));
}

NF_DEVICE float apply_act(float v, int act) {
  switch (act) {
    case NF_ACT_RELU: return fmaxf(v, 0.0f);
    case NF_ACT_GELU: return gelu_erf(v);
    case NF_ACT_TANH: return tanhf(v);
    default: return v;
  }
}

// GELU for the bf16 tensor-core epilogues: the tanh form on MUFU.TANH (one
// SFU op instead of erf's exp + reciprocal). |gelu_tanh - gelu_erf| <= 4.8e-4
// over the reals (at x ~ 2.7, i.e. 2e-4 relative), and tanh.approx adds
// <= 2^-11 relative: both far below the bf16 output rounding (2^-9), so the
// result is the erf GELU at bf16 precision. fp32 / exact paths use gelu_erf.
NF_DEVICE float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
NF_DEVICE float gelu_bf16_epilogue(float x) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(u), hx);
}

// bf16-output epilogue activations: GELU (tanh form) and tanh on the SFU's
// tanh.approx (relative error ~2^-11, below the bf16 output rounding).
template <int ACT>
NF_DEVICE float act_t(float v) {
  if constexpr (ACT == NF_ACT_RELU) return fmaxf(v, 0.0f);
  else if constexpr (ACT == NF_ACT_GELU) return gelu_bf16_epilogue(v);
  else if constexpr (ACT == NF_ACT_TANH) return tanh_approx(v);
  else return v;
}

// Epilogue activation chosen at run time (a launch-uniform branch around the
// whole chunk, so each case is a straight unrolled loop). RELU_ONLY kernels
// (implicit-GEMM convs: folded BN + ReLU) compile only that case.
template <bool RELU_ONLY = false, int N>
NF_DEVICE void apply_act(int act, float (&v)[N]) {
  if constexpr (RELU_ONLY) {
    if (act == NF_ACT_RELU) {
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = act_t<NF_ACT_RELU>(v[j]);
    }
    return;
  }
  switch (act) {
    case NF_ACT_RELU:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = act_t<NF_ACT_RELU>(v[j]);
      break;
    case NF_ACT_GELU:
      if constexpr (N % 2 == 0) {
        // element pairs in packed fp32x2 arithmetic (FMUL2 / FFMA2): the same
        // per-element IEEE operations as gelu_bf16_epilogue (bit-identical),
        // half the FP instructions of the epilogue's longest activation
#pragma unroll
        for (int j = 0; j < N; j += 2) {
          const float2 x = make_float2(v[j], v[j + 1]);
          const float2 c = __ffma2_rn(__fmul2_rn(make_float2(0.044715f, 0.044715f), x),
                                      __fmul2_rn(x, x), x);
          const float2 u = __fmul2_rn(make_float2(0.7978845608028654f, 0.7978845608028654f), c);
          const float2 hx = __fmul2_rn(make_float2(0.5f, 0.5f), x);
          const float2 y = __ffma2_rn(hx, make_float2(tanh_approx(u.x), tanh_approx(u.y)), hx);
          v[j] = y.x;
          v[j + 1] = y.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = act_t<NF_ACT_GELU>(v[j]);
      }
      break;
    case NF_ACT_TANH:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = act_t<NF_ACT_TANH>(v[j]);
      break;
    default:
      break;
  }
}

// 2^x, flush-to-zero approximate (MUFU.EX2, one instruction).
NF_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

NF_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
NF_DEVICE float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// Shared-memory addressing and mbarriers
// ---------------------------------------------------------------------------
NF_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

NF_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

NF_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

NF_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

NF_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

NF_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Wait with cluster-scope acquire: remote (DSMEM) writes released by peer
// CTAs' mbarrier arrivals are visible after it returns.
NF_DEVICE void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC;\n\t"
      "bra LAB_WAITC;\n\t"
      "DONEC:\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// float2 store into the same-offset shared memory of cluster CTA `rank`.
NF_DEVICE void st_cluster_f2(const void* local, uint32_t rank, float a, float b) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(remote), "f"(a), "f"(b) : "memory");
}
// Release-arrive on the same-offset mbarrier of cluster CTA `rank`.
NF_DEVICE void mbar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
NF_DEVICE void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) loads with an L2 cache-policy hint
// ---------------------------------------------------------------------------
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

NF_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

NF_DEVICE void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                           int c2, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(hint)
      : "memory");
}

NF_DEVICE void tma_load_4d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                           int c2, int c3, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3), "l"(hint)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, no tensor map), completing
// `bytes` (multiple of 16, 16-byte aligned both sides) on an mbarrier.
NF_DEVICE void bulk_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of a contiguous global range (bytes multiple of 16).
// TMA bulk-tensor store smem -> global (bulk-group completion).
NF_DEVICE void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
NF_DEVICE void tma_store_4d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2,
                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
NF_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
NF_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
NF_DEVICE void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Make generic-proxy shared-memory writes visible to the async (TMA) proxy.
NF_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
NF_DEVICE void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
NF_DEVICE void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
NF_DEVICE uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
NF_DEVICE void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
NF_DEVICE uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

// Programmatic dependent launch: wait for the producing grid's memory to be
// visible / allow the next grid in the stream to start its prologue.
NF_DEVICE void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
NF_DEVICE void grid_dependents_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA issue, commit, TMEM -> register loads
// ---------------------------------------------------------------------------
NF_DEVICE void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

NF_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

NF_DEVICE void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
NF_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16/f16 inputs, fp32 accumulate.
NF_DEVICE void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync).
NF_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp receives
// columns [col, col+32) of TMEM lane (warp_quarter*32 + t).
NF_DEVICE void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// ---------------------------------------------------------------------------
// CTA pairs (cta_group::2): two SMs of one TPC share an M=256 MMA. Rank 0
// (the leader) owns the mbarriers the MMA waits on and issues the MMA; each
// CTA holds its own 128 A rows and half of B in its shared memory.
// ---------------------------------------------------------------------------
NF_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
NF_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// Same shared::cta offset in the leader CTA (clear the peer bit).
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

NF_DEVICE void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, uint64_t* leader_bar,
                                int c0, int c1, int c2, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(leader_bar) & kPeerBitMask), "r"(c0),
      "r"(c1), "r"(c2), "l"(hint)
      : "memory");
}

NF_DEVICE void tmem_alloc_pair(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
NF_DEVICE void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// Leader-issued M=256 MMA over the pair.
NF_DEVICE void umma_f16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on the same-offset mbarrier of both CTAs once the leader's MMAs retire.
NF_DEVICE void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
// Arrive on the leader CTA's copy of a local mbarrier.
NF_DEVICE void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns.
NF_DEVICE void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int N>
NF_DEVICE void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
  static_assert(N == 16 || N == 32, "x16 / x32 only");
  if constexpr (N == 32) tmem_ld_32x32b_x32(taddr, r);
  else tmem_ld_32x32b_x16(taddr, r);
}

NF_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------
// UMMA descriptors
// ---------------------------------------------------------------------------
// Shared-memory matrix descriptor for a K-major operand tile written by TMA
// with SWIZZLE_128B: rows of 128 bytes, 8-row (1024 B) swizzle atoms stacked
// along M/N. Tile base must be 1024-byte aligned. Bit layout (sm_100):
//   [0,14) start>>4  [16,30) LBO>>4  [32,46) SBO>>4  [46,48) version=1
//   [49,52) base offset  [61,64) layout (2 = SWIZZLE_128B)
NF_DEVICE uint64_t make_sw128_kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1u) << 16;           // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;   // SBO: next 8-row group
  d |= static_cast<uint64_t>(1u) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;           // SWIZZLE_128B
  return d;
}

// Shared-memory descriptor for an MN-major operand in the SWIZZLE_128B
// canonical layout ((64 MN elems, n), (8 K rows, k)) : ((contig, LBO), (128 B,
// SBO)) for 16-bit types: 128-byte rows hold 64 consecutive MN elements, one
// row per K index, 8-row (1 KB) swizzle atoms stacked along K at `sbo` bytes
// and further 64-element MN chunks at `lbo` bytes (CUTLASS make_umma_desc).
NF_DEVICE uint64_t make_sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor, kind::f16 with bf16 A/B, fp32 D, both K-major.
//   [4,6) D fmt (1=f32)  [7,10) A fmt (1=bf16)  [10,13) B fmt (1=bf16)
//   [15] A major  [16] B major  [17,23) N>>3  [24,29) M>>4
__host__ __device__ constexpr uint32_t make_idesc_bf16_f32(int M, int N, int a_mn_major = 0,
                                                          int b_mn_major = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
         (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// Launch with programmatic dependent launch enabled: the kernel may start
// while its predecessor in the stream drains; kernels call
// grid_dependency_wait() before touching data the predecessor writes.
// (Always on: every launch carries the programmatic-serialization attribute.)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and
// device: function attributes live in each device's context, so a process
// driving several GPUs must set them on each. One instance per kernel (a
// function-local static next to the launch); idempotent, so two threads
// racing on the first launch both just set the same value.
// n / d for 0 <= n < 2^31 by a multiply-high and a shift (Granlund-Montgomery
// round-up reciprocal; exhaustively checked for the divisor ranges used).
// The GEMM unit decode and the implicit-GEMM gathers divide by run-time
// extents per unit / per k-block: ~20 instructions each as integer
// divisions, which the short-K gather warps of the grouped 3x3 convs spent
// ~10% of their stall samples on.
struct FastDiv {
  uint32_t m = 0, s = 0;
  static FastDiv make(int d) {
    FastDiv f;
    while ((1u << f.s) < uint32_t(d)) ++f.s;
    f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << f.s) - uint64_t(d))) / uint64_t(d) + 1);
    return f;
  }
  NF_DEVICE int div(int n) const {
    return int((__umulhi(uint32_t(n), m) + uint32_t(n)) >> s);
  }
};

struct SmemAttrOnce {
  std::atomic<unsigned long long> done{0};
  template <typename F>
  void set(F kern, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Entry of every non-TMA kernel: wait for the producer grid, then let the
// next grid in the stream begin scheduling.
NF_DEVICE void pdl_enter() {
  grid_dependency_wait();
  grid_dependents_launch();
}

// Cross-CTA / cross-kernel completion counters (chained launches): spin
// until `*ctr >= target` with acquire loads, then order later async-proxy
// (TMA) reads of the producer's data after it. The spin is bounded (~2 s):
// a counter that never arrives is a bug, and trapping turns it into a launch
// error instead of a hung device.
NF_DEVICE void wait_counter(const unsigned* ctr, unsigned target) {
  unsigned v;
  for (uint32_t n = 0;; ++n) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    if (n > (1u << 25)) __trap();
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Producer side of wait_counter: one release reduction (the writes ordered
// before it -- this thread's and, through the barrier the caller passed,
// its CTA's -- are visible to an acquire that sees the count). Replaces a
// sequentially consistent __threadfence() + atomicAdd (MEMBAR.SC + L1
// invalidate on the publishing thread).
NF_DEVICE void publish_count(unsigned* ctr) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

// Split-K arrival: one acq_rel increment by one thread after a CTA barrier
// (the CUTLASS semaphore pattern): releases the CTA's partials written
// before the barrier, and the last arriver acquires the other splits'.
NF_DEVICE unsigned arrive_acq_rel(unsigned* ctr) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
  return old;
}

// Non-blocking form of wait_counter: true (and the acquire + proxy fence
// done) when the counter has arrived.
NF_DEVICE bool counter_ready(const unsigned* ctr, unsigned target) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  if (v < target) return false;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return true;
}

// Per-token (mean, rstd) of a folded LayerNorm over D features from its
// producer's statistics of `parts` equal parts (the producer's 128-feature
// tiles): (sum, M2 = centred sum of squares about the part's own mean).
// Parts merge in index order with Chan et al.'s pairwise update
//   (n_a, mean_a, M2_a) + (n_p, mean_b, M2_b): delta = mean_b - mean_a,
//   mean += delta * n_p / n,  M2 += M2_b + delta^2 * n_a * n_p / n,
// so the variance never forms E[x^2] - mean^2 (no cancellation when
// |mean| >> std) and the reduction order is fixed (deterministic).
NF_DEVICE float2 fold_stats(const float2* st, int parts, int rows, int g, int tok, float inv_d,
                            float eps) {
  const float n_p = 1.0f / (inv_d * float(parts));  // features per part
  const float inv_np = inv_d * float(parts);
  const float2* base = st + int64_t(g) * parts * rows + tok;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  for (int q0 = 0; q0 < parts; q0 += 8) {
    float2 v[8];  // up to 8 parts in flight (D <= 1024 in one round trip)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = q0 + i < parts ? __ldcg(base + int64_t(q0 + i) * rows) : make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (q0 + i >= parts) break;
      const float nn = n + n_p;
      const float delta = v[i].x * inv_np - mean;
      mean = fmaf(delta, n_p / nn, mean);
      m2 += v[i].y + delta * delta * (n * n_p / nn);
      n = nn;
    }
  }
  return make_float2(mean, rsqrtf(fmaxf(m2 * inv_d, 0.f) + eps));
}

}  // namespace nf
