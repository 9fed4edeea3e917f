// Restriction kernel (included by trihalo.cu): the HBM-bound hot loop.
//
// Restriction streams ~9x more fine-source bytes than it writes (SURVEY
// §8a A1: 1.15 MB per p = 9 face for order2, 1.84 MB for order3).  Measured
// on B200 (profiles/r01_probe_load_paths.txt), the fastest way to stream the
// unpadded u = 59 AoS cells (472 B, 8-byte aligned) is plain LDG.64 into
// registers at >= 24-32 resident warps per SM; 8-byte cp.async tops out near
// 5.5 TB/s and TMA needs 16-byte aligned cells.  So this kernel is built for
// occupancy and lean address math: one warp per (face, coarse column) item,
// NU unknowns per lane (u in chunks of 32 NU), the window streamed one
// z-slice (L x L cells) at a time, dense weights broadcast from shared memory,
// tensor rows from the constant bank (__grid_constant__ kernel parameter).
//   MODE 1  dense  out[c] = sum_cell W[cls][cell][c] v[cell]     (order2/3, matrix_linear)
//   MODE 2  tensor normal, then t1, then t2 1-D rows              (tensor_linear, linear.py:115-151)
// Requirements (checked on the host): k = 3 restriction with one normal group
// of 3 children and window L, every tangential group 1 child with window L,
// <= NCLS distinct dense blocks; for MODE 2 all tangential rows equal.
#pragma once

template <int MODE, int L, int NCLS>
struct RestrictParams {
  double w[MODE == 1 ? NCLS : 1][MODE == 1 ? L * L * L : 1][3];  // dense blocks [cls][cell][child]
  double r0[3][L];                                               // tensor rows: normal
  double rt[L];                                                  //              tangential
};

template <int MODE, int L, int NCLS, int NU, int MINB>
__global__ void __launch_bounds__(128, MINB) restrict_reg_kernel(DevOp op,
                                                                 const __grid_constant__ RestrictParams<MODE, L, NCLS> P,
                                                                 const double* __restrict__ src,
                                                                 double* __restrict__ dst,
                                                                 const th_face* __restrict__ faces, int64_t n_faces,
                                                                 int u, int32_t* flag) {
  // dense weights are staged once per CTA in shared memory and read as
  // broadcast LDS: left in the constant bank, the compiler hoists all of them
  // into (uniform) registers and spills
  __shared__ double sw[MODE == 1 ? NCLS * L * L * L * 3 : 1];
  if constexpr (MODE == 1) {
    const double* pw = &P.w[0][0][0];
    for (int i = threadIdx.x; i < NCLS * L * L * L * 3; i += blockDim.x) sw[i] = pw[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int p = op.p;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = n_faces * op.max_items;
  for (int64_t item = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; item < total; item += nwarps) {
    const int64_t f = item / op.max_items;
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face_restrict(fp, op, fr);
    int g0, g1, g2;
    if (!decode_item(op, fr, int(item - f * op.max_items), g0, g1, g2)) continue;
    const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]), G2 = __ldg(&op.grp1[g2]);
    const int cls = (MODE == 1 && NCLS > 1) ? __ldg(&op.block_id[(g0 * op.G1 + g1) * op.G1 + g2]) : 0;
    const double* const wcls = sw + cls * (L * L * L * 3);
    const int64_t adj = fr.src0 - __ldg(&fp->src[0]) + int64_t(G0.x) * fr.sn + lane;
    // per-row (t1) offsets and fine-block column
    int64_t yo[L];
    int yb[L];
#pragma unroll
    for (int y = 0; y < L; ++y) {
      const int a1 = G1.x + y;
      yb[y] = (a1 >= p) + (a1 >= 2 * p);
      yo[y] = int64_t(a1 - yb[y] * p) * fr.s1;
    }
    // L2 bulk prefetch of the whole window (one cell per lane): the slices
    // below then stream from L2 while only one slice is held in registers
    // (3x3x3 windows only: for 5x5x5 windows the 125 TMA prefetch ops per item
    //  cost more than they save, measured 0.38 vs 0.47 of HBM on config 3)
    for (int cell = lane; L == 3 && op.prefetch && cell < L * L * L; cell += 32) {
      const int x = cell % L, y = (cell / L) % L, z = cell / (L * L);
      const int a1 = G1.x + y, a2 = G2.x + z;
      const int b1 = (a1 >= p) + (a1 >= 2 * p), b2 = (a2 >= p) + (a2 >= 2 * p);
      const int64_t e = __ldg(&fp->src[b1 + 3 * b2]) + int64_t(a1 - b1 * p) * fr.s1 +
                        int64_t(a2 - b2 * p) * fr.s2 + adj - lane + int64_t(x) * fr.sn;
      l2_prefetch_cell(src + e, u);
    }
    const int t1 = G1.z, t2 = G2.z;
    const bool in_box = t1 >= fr.lo1 && t1 < fr.lo1 + p && t2 >= fr.lo2 && t2 < fr.lo2 + p;
    const int64_t obase = fr.dst + (t1 - fr.lo1) * fr.d1 + (t2 - fr.lo2) * fr.d2 + lane;
    for (int cb = 0; cb < u; cb += 32 * NU) {
      bool ok[NU];
#pragma unroll
      for (int q = 0; q < NU; ++q) ok[q] = cb + lane + 32 * q < u;
      double acc[3][NU];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < NU; ++q) acc[c][q] = 0.0;
      constexpr int ZU = (L == 3) ? L : 1;  // 3x3x3 windows unroll fully, 5x5x5 stream slice by slice
#pragma unroll 1
      for (int z0 = 0; z0 < L; z0 += ZU)
#pragma unroll
        for (int dz = 0; dz < ZU; ++dz) {
          const int z = z0 + dz;
          const int a2 = G2.x + z;
          const int b2 = (a2 >= p) + (a2 >= 2 * p);
          const int64_t zo = int64_t(a2 - b2 * p) * fr.s2 + adj + cb;
          if (L == 5 && (op.prefetch & 4) && z + 1 < L) {
            // per-line L2 prefetch of slice z+1 (25 cells x 4 lines over the 32 lanes)
            const int a2n = a2 + 1, b2n = (a2n >= p) + (a2n >= 2 * p);
            const int64_t zon = int64_t(a2n - b2n * p) * fr.s2 + adj - lane;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int line = lane + 32 * r;
              if (line < L * L * 4) {
                const int cell = line >> 2, part = line & 3;
                const int x = cell % L, y = cell / L;
                const double* g = src + (__ldg(&fp->src[yb[y] + 3 * b2n]) + yo[y] + zon + int64_t(x) * fr.sn) + part * 16;
                l2_prefetch_line(g);
              }
            }
          }
          double v[L][L][NU];
#pragma unroll
          for (int y = 0; y < L; ++y) {
            const double* row = src + (__ldg(&fp->src[yb[y] + 3 * b2]) + yo[y] + zo);
#pragma unroll
            for (int x = 0; x < L; ++x)
#pragma unroll
              for (int q = 0; q < NU; ++q) v[y][x][q] = ok[q] ? ldg_slice(row + int64_t(x) * fr.sn + 32 * q) : 0.0;
          }
          if constexpr (MODE == 1) {
#pragma unroll
            for (int y = 0; y < L; ++y)
#pragma unroll
              for (int x = 0; x < L; ++x) {
                const double* w = wcls + (x + L * (y + L * z)) * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                  const double wc = w[c];
#pragma unroll
                  for (int q = 0; q < NU; ++q) acc[c][q] = fma(wc, v[y][x][q], acc[c][q]);
                }
              }
          } else {
            double T[3][NU];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int q = 0; q < NU; ++q) T[c][q] = 0.0;
#pragma unroll
            for (int y = 0; y < L; ++y)
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int q = 0; q < NU; ++q) {
                  double t = 0.0;
#pragma unroll
                  for (int x = 0; x < L; ++x) t = fma(P.r0[c][x], v[y][x][q], t);
                  T[c][q] = fma(P.rt[y], t, T[c][q]);
                }
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int q = 0; q < NU; ++q) acc[c][q] = fma(P.rt[z], T[c][q], acc[c][q]);
          }
          // keep the next slice's loads below this slice's math: registers stay
          // at one slice (occupancy, not per-warp depth, hides the latency)
          asm volatile("" ::: "memory");
        }
      bool bad = false;
      if (in_box) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int t0 = G0.z + c;
          if (c < G0.w && t0 >= fr.lo0 && t0 < fr.hi0) {
            double* dp = dst + obase + cb + (t0 - fr.lo0) * fr.dn;
#pragma unroll
            for (int q = 0; q < NU; ++q)
              if (ok[q]) {
                dp[32 * q] = acc[c][q];
                bad |= !isfinite(acc[c][q]);
              }
          }
        }
      }
      raise_flag(flag, bad);
    }
  }
}
