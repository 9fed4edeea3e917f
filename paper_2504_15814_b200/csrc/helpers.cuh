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


// 8-byte asynchronous global -> shared copy (LDGSTS); the cells of the unpadded
// AoS layout are only 8-byte aligned, so 16-byte cp.async / TMA do not apply
__device__ __forceinline__ void cp_async8(unsigned smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// L2 prefetch of one AoS cell through the LSU (one prefetch.global.L2 per 128-byte
// line, spread over lanes by the caller); unlike the TMA bulk prefetch it does not
// queue behind the tensor-memory engine
__device__ __forceinline__ void l2_prefetch_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
