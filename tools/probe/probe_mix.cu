// Do FP64 tensor-core MMAs (DMMA) and FP64 FMAs (DFMA) share one pipe on B200?
// Same kernel shape three ways: DFMA chains only, DMMA chains only, both interleaved.
// If the mixed kernel's time ~= max(alone) the pipes are independent; ~= sum: shared.
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int NM>
__global__ void mix(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double f[NF > 0 ? NF : 1], c[NM > 0 ? NM : 1][2];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i;
#pragma unroll
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < NF; ++i) f[i] = fma(f[i], b, a);
  }
  double s = 0;
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float time_it(K k) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000, tpb = 256, blocks = sms * 4;
  const double thr = double(blocks) * tpb;
  // per iteration and thread: DFMA: 4 * NF fmas (2 flops); DMMA: NM * 256 fmas per warp = 8 NM per thread
  auto rep = [&](const char* name, float ms, int nf, int nm) {
    const double fl = thr * iters * (4.0 * nf * 2 + 8.0 * nm * 2);
    printf("%-22s %8.3f ms  %6.2f TFLOP/s (dfma %d chains x4, dmma %d chains)\n", name, ms, fl / ms / 1e9, nf, nm);
  };
  rep("dfma only", time_it([&] { mix<8, 0><<<blocks, tpb>>>(out, iters); }), 8, 0);
  rep("dmma only", time_it([&] { mix<0, 4><<<blocks, tpb>>>(out, iters); }), 0, 4);
  rep("dfma + dmma", time_it([&] { mix<8, 4><<<blocks, tpb>>>(out, iters); }), 8, 4);
  rep("dfma + dmma (2x mma)", time_it([&] { mix<8, 8><<<blocks, tpb>>>(out, iters); }), 8, 8);
  return 0;
}
