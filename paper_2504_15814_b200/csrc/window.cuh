// Fixed-window kernels: the hot path at k = 3 (included by trihalo.cu).
//
// Every group of the operator has a window of exactly L0 (normal) / LT
// (tangential) source cells and at most C0 / CT children.  One warp owns a
// work unit = (face, normal group g0, t1 group g1) and walks the t2 groups g2
// of the face's box, so the face record is decoded and the per-row offsets,
// tables and store offsets are computed once per column of blocks.  Lanes run
// over unknowns (NU per lane: lane, lane+32); every window line (L0 cells
// along the normal) of a z-slice is loaded before it is consumed.
//   MODE 1  dense weights W[cell][child]; restriction blocks (<= 4 children)
//           are staged in shared memory and feed NU = 2 unknowns per load
//   MODE 2  tensor_linear: 1-D passes in the reference's order (normal, t1,
//           t2; linear.py:115-151)
//   MODE 3  order2 / order3 least squares as the orthogonal projection onto
//           total degree <= ORDER with the window's discrete Gram
//           polynomials (integer weights, so the moments are adds), then a
//           separable evaluation at the children with the builder's
//           synthesis tables P_a(e)/|P_a|^2.  Equal to the reference's
//           basis(delta) @ A+ rows (taylor.py:171-219) up to rounding,
//           because the projection does not depend on the basis.
#pragma once

template <int L>
struct Gram;
template <>
struct Gram<3> {  // points {-1, 0, 1}: 1 | x | 3x^2 - 2
  __device__ static constexpr double P(int a, int x) {
    return a == 0 ? 1.0 : a == 1 ? double(x - 1) : (x == 1 ? -2.0 : 1.0);
  }
};
template <>
struct Gram<5> {  // points {-2..2}: 1 | x | x^2 - 2 | (5x^3 - 17x) / 6
  __device__ static constexpr double P(int a, int x) {
    return a == 0 ? 1.0
         : a == 1 ? double(x - 2)
         : a == 2 ? double((x - 2) * (x - 2) - 2)
                  : (x == 0 ? -1.0 : x == 1 ? 2.0 : x == 2 ? 0.0 : x == 3 ? -2.0 : 1.0);
  }
};

// The first N discrete Gram moments  m_a = sum_x P_a(x) v[x]  of an L-point window,
// through the weights' symmetry about the centre (pair sums / differences):
//   L = 5:  m0 = s04 + s13 + v2, m1 = 2 d40 + d31, m2 = 2 (s04 - v2) - s13, m3 = d40 - 2 d31
//   L = 3:  m0 = s02 + v1,       m1 = v2 - v0,     m2 = s02 - 2 v1
// (10 / 4 FP64 ops instead of 18 / 6; rounding differs from the sequential sum by ~1 ulp)
template <int L, int N>
__device__ __forceinline__ void gram_moments(const double (&v)[L], double (&m)[N]) {
  static_assert(L == 3 || L == 5, "Gram windows of 3 or 5 points");
  if constexpr (L == 5) {
    const double s04 = v[0] + v[4], s13 = v[1] + v[3];
    m[0] = (s04 + s13) + v[2];
    if constexpr (N > 1) {
      const double d40 = v[4] - v[0], d31 = v[3] - v[1];
      m[1] = fma(2.0, d40, d31);
      if constexpr (N > 2) m[2] = fma(2.0, s04 - v[2], -s13);
      if constexpr (N > 3) m[3] = fma(-2.0, d31, d40);
    }
  } else {
    const double s02 = v[0] + v[2];
    m[0] = s02 + v[1];
    if constexpr (N > 1) m[1] = v[2] - v[0];
    if constexpr (N > 2) m[2] = fma(-2.0, v[1], s02);
  }
}

// gram_moments with the moment count n given at run time (a constant after unrolling)
template <int L>
__device__ __forceinline__ void gram_moments_n(const double (&v)[L], double* m, int n) {
  if constexpr (L == 5) {
    const double s04 = v[0] + v[4], s13 = v[1] + v[3];
    m[0] = (s04 + s13) + v[2];
    if (n > 1) {
      const double d40 = v[4] - v[0], d31 = v[3] - v[1];
      m[1] = fma(2.0, d40, d31);
      if (n > 2) m[2] = fma(2.0, s04 - v[2], -s13);
      if (n > 3) m[3] = fma(-2.0, d31, d40);
    }
  } else {
    const double s02 = v[0] + v[2];
    m[0] = s02 + v[1];
    if (n > 1) m[1] = v[2] - v[0];
    if (n > 2) m[2] = fma(-2.0, v[1], s02);
  }
}

// y-pass of the per-line x moments mm[y][a]: T_ab = sum_y P_b(y) mm[y][a] for a + b < D,
// pairs ordered a-major (T index = a D - a(a-1)/2 + b), each column through gram_moments
template <int L, int D, int A = 0, int NT>
__device__ __forceinline__ void gram_y(const double (&mm)[L][D], double (&T)[NT]) {
  if constexpr (A < D) {
    constexpr int OFF = A * D - A * (A - 1) / 2;
    double col[L], tb[D - A];
#pragma unroll
    for (int y = 0; y < L; ++y) col[y] = mm[y][A];
    gram_moments<L, D - A>(col, tb);
#pragma unroll
    for (int b = 0; b < D - A; ++b) T[OFF + b] = tb[b];
    gram_y<L, D, A + 1>(mm, T);
  }
}

// acc += g * v for a compile-time integer weight g (adds / subs when |g| = 1)
__device__ __forceinline__ void gacc(double& acc, double g, double v) {
  if (g == 1.0) acc += v;
  else if (g == -1.0) acc -= v;
  else if (g != 0.0) acc = fma(g, v, acc);
}

template <int MODE, int L0, int LT, int C0, int CT, int ORDER, int NU, int MINB>
__global__ void __launch_bounds__(128, MINB) window_kernel(DevOp op, const double* __restrict__ src,
                                                     double* __restrict__ dst, const th_face* __restrict__ faces,
                                                     int64_t n_faces, int u, int32_t* flag) {
  constexpr int S = L0 * LT * LT;
  constexpr int CH = C0 * CT * CT;
  constexpr bool SMEM_W = (MODE == 1 && CH <= 4);
  constexpr int D = (MODE == 3) ? ORDER + 1 : 1;
  constexpr int NT = (MODE == 3) ? (ORDER == 2 ? 6 : 10) : C0 * CT;   // pairs a + b <= ORDER
  constexpr int NM = (MODE == 3) ? (ORDER == 2 ? 10 : 20) : CH;       // triples a + b + c <= ORDER
  extern __shared__ double4 sw4[];
  if constexpr (SMEM_W) {
    const double4* gw = reinterpret_cast<const double4*>(op.weights);
    for (int i = threadIdx.x; i < op.n_blocks * S; i += blockDim.x) sw4[i] = gw[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int upf = op.units_per_face;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = n_faces * upf;
  for (int64_t unit = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; unit < total; unit += nwarps) {
    const int64_t f = unit / upf;
    const int r = int(unit - f * upf);
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face(fp, op, fr);
    if (r >= fr.n0 * fr.n1) continue;
    const int g1 = fr.g1 + r % fr.n1, g0 = fr.g0 + r / fr.n1;
    const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]);
    // ---- per-unit offsets -------------------------------------------------
    int64_t xo[L0], yo[LT];
    int yb[LT];
#pragma unroll
    for (int x = 0; x < L0; ++x) xo[x] = int64_t(G0.x + x) * fr.sn;
#pragma unroll
    for (int y = 0; y < LT; ++y) {
      const int a1 = G1.x + y;
      yb[y] = op.role == 0 ? 0 : (a1 >= op.p) + (a1 >= 2 * op.p);
      yo[y] = int64_t(a1 - yb[y] * op.p) * fr.s1;
    }
    const int64_t adj = fr.src0 - __ldg(&fp->src[0]);
    int64_t do0[C0], do1[CT];
    bool ok0[C0], ok1[CT];
#pragma unroll
    for (int i = 0; i < C0; ++i) {
      const int t = G0.z + i;
      ok0[i] = i < G0.w && t >= fr.lo0 && t < fr.hi0;
      do0[i] = int64_t(t - fr.lo0) * fr.dn;
    }
#pragma unroll
    for (int i = 0; i < CT; ++i) {
      const int t = G1.z + i;
      ok1[i] = i < G1.w && t >= fr.lo1 && t < fr.lo1 + op.p;
      do1[i] = int64_t(t - fr.lo1) * fr.d1;
    }
    double R0[MODE == 2 ? C0 : 1][MODE == 2 ? L0 : 1], R1[MODE == 2 ? CT : 1][MODE == 2 ? LT : 1];
    if constexpr (MODE == 2) {
      const double* r0 = op.rows0 + __ldg(&op.row_off0[g0]);
      const double* r1 = op.rows1 + __ldg(&op.row_off1[g1]);
#pragma unroll
      for (int c = 0; c < C0; ++c)
#pragma unroll
        for (int x = 0; x < L0; ++x) R0[c][x] = c < G0.w ? __ldg(r0 + c * L0 + x) : 0.0;
#pragma unroll
      for (int c = 0; c < CT; ++c)
#pragma unroll
        for (int y = 0; y < LT; ++y) R1[c][y] = c < G1.w ? __ldg(r1 + c * LT + y) : 0.0;
    }
    const double* s0 = op.synth0 + g0 * 12;
    const double* s1 = op.synth1 + g1 * 12;
    // ---- walk the t2 groups of the box ----------------------------------------
    for (int g2 = fr.g2; g2 < fr.g2 + fr.n2; ++g2) {
      const int4 G2 = __ldg(&op.grp1[g2]);
      // bulk-prefetch this block's window into L2 (one cell per lane): the
      // slices below then stream from L2 with one slice held in registers
      for (int cell = lane; op.prefetch && cell < S; cell += 32)
        l2_prefetch_cell(src + src_addr(fp, op, fr, G0.x + cell % L0, G1.x + (cell / L0) % LT, G2.x + cell / (L0 * LT)),
                         u);
      int64_t zrow[LT];  // source offset of (x = 0, y = 0 block column, z) without the y part
      int zb[LT];
#pragma unroll
      for (int z = 0; z < LT; ++z) {
        const int a2 = G2.x + z;
        zb[z] = op.role == 0 ? 0 : (a2 >= op.p) + (a2 >= 2 * op.p);
        zrow[z] = int64_t(a2 - zb[z] * op.p) * fr.s2;
      }
      int64_t do2[CT];
      bool ok2[CT];
#pragma unroll
      for (int i = 0; i < CT; ++i) {
        const int t = G2.z + i;
        ok2[i] = i < G2.w && t >= fr.lo2 && t < fr.lo2 + op.p;
        do2[i] = int64_t(t - fr.lo2) * fr.d2;
      }
      double R2[MODE == 2 ? CT : 1][MODE == 2 ? LT : 1];
      if constexpr (MODE == 2) {
        const double* r2 = op.rows1 + __ldg(&op.row_off1[g2]);
#pragma unroll
        for (int c = 0; c < CT; ++c)
#pragma unroll
          for (int z = 0; z < LT; ++z) R2[c][z] = c < G2.w ? __ldg(r2 + c * LT + z) : 0.0;
      }
      const int bid = (MODE == 1) ? __ldg(&op.block_id[(g0 * op.G1 + g1) * op.G1 + g2]) : 0;
      const double* __restrict__ Wg = op.weights + (MODE == 1 ? __ldg(&op.block_off[bid]) : 0);
      const double4* __restrict__ Ws = sw4 + (SMEM_W ? bid * S : 0);
      for (int cb = 0; cb < u; cb += 32 * NU) {
        bool okq[NU];
#pragma unroll
        for (int q = 0; q < NU; ++q) okq[q] = cb + lane + 32 * q < u;
        double acc[NM][NU];
#pragma unroll
        for (int c = 0; c < NM; ++c)
#pragma unroll
          for (int q = 0; q < NU; ++q) acc[c][q] = 0.0;
#pragma unroll((LT == 3 && MODE == 3) ? LT : 1)  // MODE 1 / 2: acc[CH] and a slice stay in registers
        for (int z = 0; z < LT; ++z) {
          double v[LT][L0][NU];
#pragma unroll
          for (int y = 0; y < LT; ++y) {
            const int64_t base =
                (op.role == 0 ? fr.src0 : __ldg(&fp->src[yb[y] + 3 * zb[z]]) + adj) + yo[y] + zrow[z] + cb + lane;
#pragma unroll
            for (int x = 0; x < L0; ++x)
#pragma unroll
              for (int q = 0; q < NU; ++q) v[y][x][q] = okq[q] ? ldg_slice(src + base + xo[x] + 32 * q) : 0.0;
          }
          double T[NT][NU];
#pragma unroll
          for (int c = 0; c < NT; ++c)
#pragma unroll
            for (int q = 0; q < NU; ++q) T[c][q] = 0.0;
#pragma unroll
          for (int y = 0; y < LT; ++y) {
            if constexpr (MODE == 1) {
#pragma unroll
              for (int x = 0; x < L0; ++x) {
                const int cell = x + L0 * (y + LT * z);
                if constexpr (SMEM_W) {
                  const double4 w = Ws[cell];
                  const double wc[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                  for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int q = 0; q < NU; ++q) acc[c][q] = fma(wc[c], v[y][x][q], acc[c][q]);
                } else {
                  const double2* wr = reinterpret_cast<const double2*>(Wg + int64_t(cell) * ((CH + 1) & ~1));
#pragma unroll
                  for (int c = 0; c < CH; c += 2) {
                    const double2 w = __ldg(wr + c / 2);
#pragma unroll
                    for (int q = 0; q < NU; ++q) {
                      acc[c][q] = fma(w.x, v[y][x][q], acc[c][q]);
                      if (c + 1 < CH) acc[c + 1][q] = fma(w.y, v[y][x][q], acc[c + 1][q]);
                    }
                  }
                }
              }
            } else if constexpr (MODE == 2) {
#pragma unroll
              for (int c0 = 0; c0 < C0; ++c0)
#pragma unroll
                for (int q = 0; q < NU; ++q) {
                  double tx = 0.0;
#pragma unroll
                  for (int x = 0; x < L0; ++x) tx = fma(R0[c0][x], v[y][x][q], tx);
#pragma unroll
                  for (int c1 = 0; c1 < CT; ++c1) T[c0 + C0 * c1][q] = fma(R1[c1][y], tx, T[c0 + C0 * c1][q]);
                }
            } else {
#pragma unroll
              for (int q = 0; q < NU; ++q) {
                double m[D], vx[L0];
#pragma unroll
                for (int x = 0; x < L0; ++x) vx[x] = v[y][x][q];
                gram_moments<L0, D>(vx, m);
                int t = 0;
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                  for (int b = 0; b + a < D; ++b, ++t) gacc(T[t][q], Gram<LT>::P(b, y), m[a]);
              }
            }
          }
          if constexpr (MODE == 2) {
#pragma unroll
            for (int c2 = 0; c2 < CT; ++c2)
#pragma unroll
              for (int c01 = 0; c01 < C0 * CT; ++c01)
#pragma unroll
                for (int q = 0; q < NU; ++q)
                  acc[c01 + C0 * CT * c2][q] = fma(R2[c2][z], T[c01][q], acc[c01 + C0 * CT * c2][q]);
          } else if constexpr (MODE == 3) {
            // z-pass with the slice's Gram values (z is a runtime index for LT = 5)
            const double tz = double(z - (LT - 1) / 2);
            double pz[D];
            pz[0] = 1.0;
            if (D > 1) pz[1] = tz;
            if (D > 2) pz[2] = LT == 3 ? 3.0 * tz * tz - 2.0 : tz * tz - 2.0;
            if (D > 3) pz[D > 3 ? 3 : 0] = (5.0 * tz * tz * tz - 17.0 * tz) / 6.0;
            int t = 0, mi = 0;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int b = 0; b + a < D; ++b, ++t)
#pragma unroll
                for (int c = 0; c + b + a < D; ++c, ++mi)
#pragma unroll
                  for (int q = 0; q < NU; ++q) acc[mi][q] = fma(pz[c], T[t][q], acc[mi][q]);
          }
          asm volatile("" ::: "memory");  // one slice of loads live at a time
        }
        // ---- store ------------------------------------------------------------
        bool bad = false;
        double* const dbase = dst + fr.dst + cb + lane;
        if constexpr (MODE == 3) {
          const double* s2 = op.synth1 + g2 * 12;
#pragma unroll
          for (int l = 0; l < CT; ++l) {
            if (!ok2[l]) continue;
            double Q[NT][NU];
            int t = 0, mi = 0;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int b = 0; b + a < D; ++b, ++t) {
#pragma unroll
                for (int q = 0; q < NU; ++q) Q[t][q] = 0.0;
#pragma unroll
                for (int c = 0; c + b + a < D; ++c, ++mi) {
                  const double sz = __ldg(s2 + l * 4 + c);
#pragma unroll
                  for (int q = 0; q < NU; ++q) Q[t][q] = fma(sz, acc[mi][q], Q[t][q]);
                }
              }
#pragma unroll
            for (int j = 0; j < CT; ++j) {
              if (!ok1[j]) continue;
              double Rv[D][NU];
              int tt = 0;
#pragma unroll
              for (int a = 0; a < D; ++a) {
#pragma unroll
                for (int q = 0; q < NU; ++q) Rv[a][q] = 0.0;
#pragma unroll
                for (int b = 0; b + a < D; ++b, ++tt) {
                  const double sy = __ldg(s1 + j * 4 + b);
#pragma unroll
                  for (int q = 0; q < NU; ++q) Rv[a][q] = fma(sy, Q[tt][q], Rv[a][q]);
                }
              }
#pragma unroll
              for (int i = 0; i < C0; ++i) {
                if (!ok0[i]) continue;
                double* dp = dbase + do0[i] + do1[j] + do2[l];
#pragma unroll
                for (int q = 0; q < NU; ++q) {
                  double s = 0.0;
#pragma unroll
                  for (int a = 0; a < D; ++a) s = fma(__ldg(s0 + i * 4 + a), Rv[a][q], s);
                  if (okq[q]) {
                    dp[32 * q] = s;
                    bad |= !isfinite(s);
                  }
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int i0 = c % C0, i1 = (c / C0) % CT, i2 = c / (C0 * CT);
            if (ok0[i0] && ok1[i1] && ok2[i2]) {
              double* dp = dbase + do0[i0] + do1[i1] + do2[i2];
#pragma unroll
              for (int q = 0; q < NU; ++q)
                if (okq[q]) {
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
}
