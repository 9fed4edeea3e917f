// Which load path streams AoS cells (u = 59 doubles, 472 B, or padded 64 -> 512 B)
// fastest on B200?  Each warp reads runs of 9 consecutive-ish cells ("slices")
// from a 4+ GB buffer and reduces them.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda/barrier>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int SLICE = 9;

// cells are visited slice by slice: slice s covers cells [s*SLICE, s*SLICE+SLICE) (contiguous)
__global__ void ldg_regs(const double* __restrict__ src, long n_slices, int cell_stride, int u, double* out) {
  int lane = threadIdx.x & 31;
  long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  double acc = 0;
  for (long s = w; s < n_slices; s += nw) {
    const double* b = src + s * SLICE * (long)cell_stride + lane;
    double v[SLICE][2];
#pragma unroll
    for (int c = 0; c < SLICE; ++c) {
      v[c][0] = __ldg(b + c * cell_stride);
      v[c][1] = lane + 32 < u ? __ldg(b + c * cell_stride + 32) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < SLICE; ++c) acc += v[c][0] * 1.0000001 + v[c][1];
  }
  if (acc == 1.2345) out[0] = acc;
}

__device__ __forceinline__ void cp8(unsigned d, const void* g) { asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(g)); }
__device__ __forceinline__ void cp16(unsigned d, const void* g) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g)); }
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int NST, int W, bool SIXTEEN>
__global__ void __launch_bounds__(W * 32) cpasync_ring(const double* __restrict__ src, long n_slices, int cell_stride, int u, double* out) {
  extern __shared__ double ring[];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* my = ring + (size_t)warp * NST * SLICE * 64;
  unsigned mys = (unsigned)__cvta_generic_to_shared(my);
  long nw = gridDim.x * (long)W, w = blockIdx.x * (long)W + warp;
  long per = (n_slices + nw - 1) / nw, b0 = w * per, b1 = min(n_slices, b0 + per);
  long n = b1 > b0 ? b1 - b0 : 0;
  auto issue = [&](long i) {
    if (i < n) {
      const double* b = src + (b0 + i) * SLICE * (long)cell_stride;
      unsigned slot = mys + (unsigned)((i % NST) * SLICE * 64 * 8);
#pragma unroll
      for (int c = 0; c < SLICE; ++c) {
        if (SIXTEEN) {
          cp16(slot + c * 512 + lane * 16, b + c * cell_stride + lane * 2);
        } else {
          cp8(slot + c * 512 + lane * 8, b + c * cell_stride + lane);
          if (lane + 32 < u) cp8(slot + c * 512 + 256 + lane * 8, b + c * cell_stride + lane + 32);
        }
      }
    }
    commit();
  };
  for (int i = 0; i < NST - 1; ++i) issue(i);
  double acc = 0;
  for (long i = 0; i < n; ++i) {
    issue(i + NST - 1);
    waitg<NST - 1>();
    __syncwarp();
    const double* slot = my + (i % NST) * SLICE * 64;
#pragma unroll
    for (int c = 0; c < SLICE; ++c) acc += slot[c * 64 + lane] * 1.0000001 + slot[c * 64 + 32 + lane];
    __syncwarp();
  }
  waitg<0>();
  if (acc == 1.2345) out[0] = acc;
}

// TMA 1-D bulk copy of a whole slice (9 contiguous cells) per stage, mbarrier completion
template <int NST, int W>
__global__ void __launch_bounds__(W * 32) bulk_ring(const double* __restrict__ src, long n_slices, int cell_stride, double* out) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) unsigned long long bar[W][NST];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* my = ring + (size_t)warp * NST * SLICE * 64;
  long nw = gridDim.x * (long)W, w = blockIdx.x * (long)W + warp;
  long per = (n_slices + nw - 1) / nw, b0 = w * per, b1 = min(n_slices, b0 + per);
  long n = b1 > b0 ? b1 - b0 : 0;
  const unsigned bytes = SLICE * cell_stride * 8;
  if (lane == 0)
    for (int k = 0; k < NST; ++k) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[warp][k]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](long i) {
    if (i < n && lane == 0) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[warp][i % NST]);
      unsigned d = (unsigned)__cvta_generic_to_shared(my + (i % NST) * SLICE * 64);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src + (b0 + i) * SLICE * (long)cell_stride), "r"(bytes), "r"(a) : "memory");
    }
  };
  for (int i = 0; i < NST - 1; ++i) issue(i);
  double acc = 0;
  for (long i = 0; i < n; ++i) {
    issue(i + NST - 1);
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[warp][i % NST]);
    unsigned phase = (unsigned)((i / NST) & 1);
    asm volatile("{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(a), "r"(phase));
    const double* slot = my + (i % NST) * SLICE * 64;
#pragma unroll
    for (int c = 0; c < SLICE; ++c) acc += slot[c * cell_stride + lane] * 1.0000001 + (lane + 32 < 59 ? slot[c * cell_stride + 32 + lane] : 0.0);
    __syncwarp();
  }
  if (acc == 1.2345) out[0] = acc;
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)5 << 30;
  double* buf; CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  double* out; CK(cudaMalloc(&out, 64));
  for (int stride : {59, 64}) {
    long n_slices = (long)(bytes / 8 / stride / SLICE) - 1;
    double gb = n_slices * SLICE * 59.0 * 8 / 1e9;  // useful bytes
    for (int bpm : {4, 8, 16}) {
      float ms = time_it([&] { ldg_regs<<<sms * bpm, 128>>>(buf, n_slices, stride, 59, out); }, 3);
      printf("stride %d ldg_regs        CTAs/SM %2d : %7.1f GB/s useful\n", stride, bpm, gb / ms * 1e3);
    }
    {
      auto k = cpasync_ring<6, 4, false>;
      int smem = 4 * 6 * SLICE * 64 * 8;
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      float ms = time_it([&] { k<<<sms * 2, 128, smem>>>(buf, n_slices, stride, 59, out); }, 3);
      printf("stride %d cp.async 8B  NST6 W4 x2: %7.1f GB/s useful\n", stride, gb / ms * 1e3);
      auto k2 = cpasync_ring<3, 8, false>;
      smem = 8 * 3 * SLICE * 64 * 8;
      CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      ms = time_it([&] { k2<<<sms * 2, 256, smem>>>(buf, n_slices, stride, 59, out); }, 3);
      printf("stride %d cp.async 8B  NST3 W8 x2: %7.1f GB/s useful\n", stride, gb / ms * 1e3);
    }
    if (stride == 64) {
      auto k = cpasync_ring<6, 4, true>;
      int smem = 4 * 6 * SLICE * 64 * 8;
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      float ms = time_it([&] { k<<<sms * 2, 128, smem>>>(buf, n_slices, stride, 59, out); }, 3);
      printf("stride %d cp.async 16B NST6 W4 x2: %7.1f GB/s useful\n", stride, gb / ms * 1e3);
    }
    {
      auto k = bulk_ring<6, 4>;
      int smem = 4 * 6 * SLICE * 64 * 8;
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (stride == 64) {
        float ms = time_it([&] { k<<<sms * 2, 128, smem>>>(buf, n_slices, stride, out); }, 3);
        printf("stride %d TMA bulk    NST6 W4 x2: %7.1f GB/s useful\n", stride, gb / ms * 1e3);
      }
    }
  }
  return 0;
}
