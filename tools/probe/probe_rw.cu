// DRAM ceiling of a read-mostly stream (the restriction's byte mix: ~10 bytes read per byte
// written) on one B200: nvcc -O3 -gencode arch=compute_100a,code=sm_100a probe_rw.cu -o probe_rw
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

// R reads per write, 4 independent loads in flight per thread and iteration
template <int R>
__global__ void rw(const double* __restrict__ src, double* __restrict__ dst, size_t n_out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += stride) {
    double acc = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) acc += __ldg(src + i + (size_t)r * n_out);
    dst[i] = acc;
  }
}

__global__ void fill(double* p, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = (double)(i & 1023);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_out = size_t(1) << 27;  // 1 GB out
  const int R = 10;                       // 10 GB in
  double *src, *dst;
  CK(cudaMalloc(&src, n_out * R * 8));
  CK(cudaMalloc(&dst, n_out * 8));
  fill<<<sms * 8, 256>>>(src, n_out * R);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int bpm : {2, 4, 8}) {
    const int blocks = sms * bpm;
    rw<R><<<blocks, 256>>>(src, dst, n_out);
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) rw<R><<<blocks, 256>>>(src, dst, n_out);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 5;
    printf("read %d : write 1, 256 x %d CTAs/SM: %.1f GB/s (read+write bytes)\n", R, bpm, n_out * 8.0 * (R + 1) / ms / 1e6);
  }
  return 0;
}
