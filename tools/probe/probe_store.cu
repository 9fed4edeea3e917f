// Write-bandwidth probe: is interpolation (~80% of its bytes are stores) bound by
// HBM write bandwidth?  Compares cudaMemset, fully coalesced 16-byte stores, and
// the interpolation kernels' store pattern (AoS cells of u = 59 doubles written
// as two 32-lane chunks of 8-byte stores, cells scattered in 27-cell blocks).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void store16(double2* __restrict__ out, long n) {
  const double2 v = make_double2(1.0, 2.0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) out[i] = v;
}

// warp w writes cell chunks: cell c = w / 2, chunk = w % 2 (32 or 27 lanes of 8 bytes)
__global__ void store_cells(double* __restrict__ out, long n_cells, int u) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; w < n_cells * 2; w += nw) {
    const long c = w >> 1;
    const int q = (int)(w & 1) * 32 + lane;
    if (q < u) out[c * u + q] = 1.0;
  }
}

// one warp per (cell block of 27 cells, chunk): 27 stores per lane, like one interpolation block
__global__ void store_blocks(double* __restrict__ out, long n_blocks, int u) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; w < n_blocks * 2; w += nw) {
    const long b = w >> 1;
    const int q = (int)(w & 1) * 32 + lane;
    if (q >= u) continue;
#pragma unroll
    for (int c = 0; c < 27; ++c) out[(b * 27 + c) * u + q] = 1.0 + c;
  }
}

// one warp writes both chunks of each cell back to back (two unknowns per lane)
__global__ void store_cells_nu2(double* __restrict__ out, long n_cells, int u) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long c = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; c < n_cells; c += nw) {
    out[c * u + lane] = 1.0;
    if (lane + 32 < u) out[c * u + 32 + lane] = 2.0;
  }
}

// one warp writes a contiguous run of R cells as a flat array of R*u doubles
template <int R>
__global__ void store_runs(double* __restrict__ out, long n_runs, int u) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; r < n_runs; r += nw) {
    double* o = out + r * R * u;
    for (int i = lane; i < R * u; i += 32) o[i] = 1.0;
  }
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
  const size_t bytes = (size_t)4 << 30;
  double* buf; CK(cudaMalloc(&buf, bytes));
  float ms = time_it([&] { CK(cudaMemsetAsync(buf, 0, bytes)); }, 5);
  printf("cudaMemset          : %7.1f GB/s\n", bytes / ms / 1e6);
  for (int per : {4, 8, 16}) {
    ms = time_it([&] { store16<<<sms * per, 256>>>((double2*)buf, bytes / 16); }, 5);
    printf("store16  CTAs/SM %2d : %7.1f GB/s\n", per, bytes / ms / 1e6);
  }
  const int u = 59;
  const long n_cells = bytes / (u * 8);
  for (int per : {4, 8, 16}) {
    ms = time_it([&] { store_cells<<<sms * per, 256>>>(buf, n_cells, u); }, 5);
    printf("cells    CTAs/SM %2d : %7.1f GB/s (u = 59, 2 chunks)\n", per, n_cells * u * 8.0 / ms / 1e6);
  }
  const long n_blocks = n_cells / 27;
  for (int per : {4, 8, 16}) {
    ms = time_it([&] { store_blocks<<<sms * per, 128>>>(buf, n_blocks, u); }, 5);
    printf("blocks27 CTAs/SM %2d : %7.1f GB/s (27 cells per warp-chunk)\n", per, n_blocks * 27 * u * 8.0 / ms / 1e6);
  }
  for (int per : {4, 8, 16}) {
    ms = time_it([&] { store_cells_nu2<<<sms * per, 256>>>(buf, n_cells, u); }, 5);
    printf("cellsNU2 CTAs/SM %2d : %7.1f GB/s (one warp per cell)\n", per, n_cells * u * 8.0 / ms / 1e6);
  }
  for (int per : {4, 8, 16}) {
    ms = time_it([&] { store_runs<3><<<sms * per, 256>>>(buf, n_cells / 3, u); }, 5);
    printf("runs3    CTAs/SM %2d : %7.1f GB/s (3-cell runs flat)\n", per, (n_cells / 3) * 3 * u * 8.0 / ms / 1e6);
  }
  for (int per : {4, 8}) {
    ms = time_it([&] { store_runs<27><<<sms * per, 256>>>(buf, n_cells / 27, u); }, 5);
    printf("runs27   CTAs/SM %2d : %7.1f GB/s (27-cell runs flat)\n", per, (n_cells / 27) * 27 * u * 8.0 / ms / 1e6);
  }
  return 0;
}
