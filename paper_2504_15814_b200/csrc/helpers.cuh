// Small device helpers shared by the fixed-window kernels (included by trihalo.cu).
#pragma once

// read-only global load the compiler may not move across the per-slice
// barrier below (a plain __ldg is treated as a constant read and hoisted,
// which multiplies the live registers by the window depth and spills)
__device__ __forceinline__ double ldg_slice(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// TMA bulk prefetch of one AoS cell (u doubles) into L2; the range is widened
// to 16-byte alignment as cp.async.bulk.prefetch requires
__device__ __forceinline__ void l2_prefetch_cell(const double* cell, int u) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(cell);
  const uintptr_t lo = a & ~uintptr_t(15);
  const unsigned bytes = unsigned((a + uintptr_t(u) * 8 - lo + 15) & ~uintptr_t(15));
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(bytes) : "memory");
}


// L2 prefetch of one AoS cell through the LSU (one prefetch.global.L2 per 128-byte
// line, spread over lanes by the caller); unlike the TMA bulk prefetch it does not
// queue behind the tensor-memory engine
__device__ __forceinline__ void l2_prefetch_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- mbarrier + 1-D TMA bulk copy (stage_slide.cuh) --------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
#ifndef TH_MBAR_HINT
#define TH_MBAR_HINT 0  // suspend-time hint (ns) of the try_wait loop; 0: none (A/B builds: -DTH_MBAR_HINT=n)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
#if TH_MBAR_HINT > 0
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2; @!P bra WAIT_%=; }" ::"r"(
          smem_u32(b)),
      "r"(parity), "n"(TH_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// global [g, g + bytes) -> shared dst, completion counted on mbarrier b
// (g, dst 16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* g, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(g), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
