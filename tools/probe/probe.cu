// Microbenchmarks that decide the kernel design: FP64 FMA peak (register,
// constant-bank and shared-memory-broadcast operands), DMMA m8n8k4 peak and
// streaming HBM read bandwidth for the AoS u=59 access pattern.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__constant__ double c_w[4096];

__global__ void dfma_reg(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// weights from the constant bank at compile-time offsets (DFMA R, R, c[][], R)
__global__ void dfma_const(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it += 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], c_w[j * 8 + i], 1e-9);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// one warp-uniform LDS.64 per DFMA
__global__ void dfma_lds64(double* out, int iters) {
  __shared__ double w[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) w[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  int base = 0;
  for (int it = 0; it < iters; it += 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], w[(base + j * 8 + i) & 1023], 1e-9);
    }
    base += 7;
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// one warp-uniform LDS.128 per 2 DFMA, each weight used by 2 accumulators
__global__ void dfma_lds128_r2(double* out, int iters) {
  __shared__ double2 w[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) w[i] = make_double2(1.0 + i * 1e-9, 1.0 - i * 1e-9);
  __syncthreads();
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  int base = 0;
  for (int it = 0; it < iters; it += 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int i = 0; i < 8; i += 4) {
        double2 ww = w[(base + j * 4 + i) & 511];
        x[i] = fma(x[i], ww.x, 1e-9);
        x[i + 1] = fma(x[i + 1], ww.y, 1e-9);
        x[i + 2] = fma(x[i + 2], ww.x, 1e-9);
        x[i + 3] = fma(x[i + 3], ww.y, 1e-9);
      }
    }
    base += 7;
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void hbm_read(const double* __restrict__ src, size_t n, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    acc += a + b + c + d;
  }
  for (; i < n; i += stride) acc += __ldg(src + i);
  if (acc == 12345.678) out[0] = acc;
}

__global__ void fill(double* p, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = (double)(i & 1023) * 1e-3;
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d max clock %d kHz\n", sms, clk);
  double* out; CK(cudaMalloc(&out, 64));
  double hw[4096]; for (int i = 0; i < 4096; ++i) hw[i] = 1.0 + i * 1e-9;
  CK(cudaMemcpyToSymbol(c_w, hw, sizeof(hw)));
  int iters = 1 << 14;
  for (int tpb : {256, 512}) {
    int blocks = sms * (2048 / tpb);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    float ms = time_it([&] { dfma_reg<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9); }, 5);
    printf("dfma_reg        tpb=%d  %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms);
    ms = time_it([&] { dfma_const<<<blocks, tpb>>>(out, iters); }, 5);
    printf("dfma_const      tpb=%d  %.2f TFLOP/s\n", tpb, flops / ms / 1e9);
    ms = time_it([&] { dfma_lds64<<<blocks, tpb>>>(out, iters); }, 5);
    printf("dfma_lds64      tpb=%d  %.2f TFLOP/s\n", tpb, flops / ms / 1e9);
    ms = time_it([&] { dfma_lds128_r2<<<blocks, tpb>>>(out, iters); }, 5);
    printf("dfma_lds128_r2  tpb=%d  %.2f TFLOP/s\n", tpb, flops / ms / 1e9);
    int diters = 1 << 12;
    double dflops = 2.0 * 8 * 256 * diters * (double)blocks * (tpb / 32);
    ms = time_it([&] { dmma_peak<<<blocks, tpb>>>(out, diters); }, 5);
    printf("dmma_m8n8k4     tpb=%d  %.2f TFLOP/s\n", tpb, dflops / ms / 1e9);
  }
  size_t n = (size_t)1 << 29;  // 4 GiB of doubles
  double* big; CK(cudaMalloc(&big, n * 8));
  fill<<<sms * 8, 256>>>(big, n); CK(cudaDeviceSynchronize());
  for (int bpm : {2, 4, 8}) {
    int blocks = sms * bpm;
    float ms = time_it([&] { hbm_read<<<blocks, 256>>>(big, n, out); }, 5);
    printf("hbm_read blocks/SM=%d  %.1f GB/s\n", bpm, n * 8.0 / ms / 1e6);
  }
  CK(cudaFree(big));
  return 0;
}
