// Shared device helpers for the B200 dichotomy kernels (sm_100a).
//
// FP64 products go through the warp-level tensor-core instruction
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured on this pool's B200
// (profiles/r01_fp64_rates.txt): DMMA sustains 37.2 TFLOP/s = 64 FMA/clk/SM
// from 4 warps/SM, plain DFMA tops out at 33.5 TFLOP/s (issue-bound), cuBLAS
// DGEMM 35.5 TFLOP/s.  tcgen05 has no f64 kind on sm_100a, so DMMA is the
// fp64 tensor path.
//
// Fragment conventions for m8n8k4 (lane l, g = l>>2, t = l&3):
//   A (8x4, row):  a = A[g][t]          B (4x8, col): b = B[t][g]
//   C (8x8):       c0 = C[g][2t], c1 = C[g][2t+1]
// A "pair step" covers k = 8s..8s+7 with two DMMAs: the first uses k-slots
// {8s+2t}, the second {8s+2t+1}.  The reduction order is a permutation of k,
// which lets every lane fetch its two A values with one 16-byte load.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define BTD_DEVINL __device__ __forceinline__

BTD_DEVINL void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// acc[i][j] += a[i].x (Y=0) or a[i].y (Y=1) (8x4 fragments) x b[j] (4x8): one k4 step
// of a TM x TN warp tile, TM*TN independent DMMAs back to back.  (mma.m16n8k4.f64
// is no wider on sm_100a: ptxas lowers it to two DMMA.8x8x4, checked in the SASS.)
template <int TM, int TN, bool Y>
BTD_DEVINL void mma_k4(double (&acc)[TM][TN][2], const double2 (&a)[TM], const double (&b)[TN]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], Y ? a[i].y : a[i].x, b[j]);
}

BTD_DEVINL unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

BTD_DEVINL void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gmem_src));
}
BTD_DEVINL void cp_async8(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gmem_src));
}
BTD_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
BTD_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
BTD_DEVINL void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

BTD_DEVINL void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); }

// L2 prefetch of `bytes` contiguous bytes by the lanes of one warp (128 B lines)
BTD_DEVINL void warp_prefetch_l2(const void* p, int64_t bytes, int lane) {
  const char* c = static_cast<const char*>(p);
  for (int64_t o = (int64_t)lane * 128; o < bytes; o += 32 * 128) prefetch_l2(c + o);
}

// 16B read-only streaming load of a factor fragment (L2-resident factors,
// re-read by the CTAs that share a range; keep them out of L1).
#ifndef BTD_FRAG_NC
#define BTD_FRAG_NC 0
#endif
BTD_DEVINL double2 ldg_cg2(const double* p) {
  if constexpr (BTD_FRAG_NC) return __ldg(reinterpret_cast<const double2*>(p));  // L1-cached variant (A/B)
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// ---- mbarrier + bulk async copy (TMA engine, 1-D) ------------------------------
BTD_DEVINL void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
BTD_DEVINL void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
BTD_DEVINL void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
BTD_DEVINL void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
BTD_DEVINL void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
BTD_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0, 16B-aligned)
BTD_DEVINL void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
