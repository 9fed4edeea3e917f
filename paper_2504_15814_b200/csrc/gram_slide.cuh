// Gram sliding kernel for the least-squares schemes (order2 / order3), both
// roles (included by trihalo.cu after window.cuh).
//
// The reference row of a target cell is its least-squares fit over a full
// tensor window, evaluated at the target (taylor.py:171-219).  That fit is the
// orthogonal projection onto total degree <= ORDER, so it can be computed with
// the window's discrete Gram polynomials, separably:
//   x (normal) moments per source line    m_a      = sum_x P_a(x) v
//   y (t1) moments per window and slice   T_ab(a2) = sum_y P_b(y) m_a
//   z (t2) moments per block              M_abc    = sum_z P_c(z) T_ab(w2 + z)
//   synthesis at the children             out      = sum S0[a] S1[b] S2[c] M_abc
// with S_d = P(e)/|P|^2 from the builder (builder.cpp choose_fast_path), read
// with non-hoistable loads at each use (hoisted, they pin ~50 registers).
// Integer Gram weights are immediates: no weight loads at all.
//
// One warp owns a work unit = (face, t1 group, 32-unknown chunk) and streams
// the t2 source slices its blocks need, in order.  Consecutive blocks' windows
// overlap along t2 (4 of 5 slices for interpolation, 2 of 5 for restriction),
// so each slice is loaded and x/y-projected once into a per-lane ring of L
// moment slices in shared memory; a block whose window is complete then only
// does its z-pass and synthesis.  Slice a2+1 is loaded into registers before
// slice a2 is projected (two register buffers), so every warp keeps a slice of
// loads in flight.
#pragma once

template <int ORDER, int ROLE, int MINB>
__global__ void __launch_bounds__(128, MINB) gram_slide_kernel(DevOp op, const double* __restrict__ src,
                                                               double* __restrict__ dst,
                                                               const th_face* __restrict__ faces, int64_t n_faces,
                                                               int u, int32_t* flag) {
  constexpr int L = ORDER == 2 ? 3 : 5;
  constexpr int D = ORDER + 1;
  constexpr int NT = ORDER == 2 ? 6 : 10;   // pairs a + b <= ORDER
  constexpr int NM = ORDER == 2 ? 10 : 20;  // triples a + b + c <= ORDER
  constexpr int C0 = 3, CT = ROLE == 0 ? 3 : 1;
  extern __shared__ double ring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const ring = ring_all + warp * (L * NT * 32) + lane;  // [slot][t] x 32 lanes, lane-private
  const int p = op.p;
  const int upf = op.units_per_face;
  const int nch = (u + 31) / 32;
  const int64_t total = n_faces * upf * nch;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t unit = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; unit < total; unit += nw) {
    const int64_t fu = unit / nch;
    const int cb = int(unit - fu * nch) * 32;
    const int64_t f = fu / upf;
    const int r = int(fu - f * upf);
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face(fp, op, fr);
    if (r >= fr.n0 * fr.n1) continue;
    const int g1 = fr.g1 + r % fr.n1, g0 = fr.g0 + r / fr.n1;
    const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]);
    const bool ok = cb + lane < u;
    // source line bases per t1 row y (restriction adds the fine block of (y, z))
    const int64_t adj = ROLE == 0 ? 0 : fr.src0 - __ldg(&fp->src[0]);
    int64_t ybase[L];
    int yb[L];
#pragma unroll
    for (int y = 0; y < L; ++y) {
      const int a1 = G1.x + y;
      yb[y] = ROLE == 0 ? 0 : (a1 >= p) + (a1 >= 2 * p);
      ybase[y] = (ROLE == 0 ? fr.src0 : adj) + int64_t(a1 - yb[y] * p) * fr.s1 + int64_t(G0.x) * fr.sn + cb + lane;
    }
    // target offsets of the normal and t1 children
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
      ok1[i] = i < G1.w && t >= fr.lo1 && t < fr.lo1 + p;
      do1[i] = int64_t(t - fr.lo1) * fr.d1;
    }
    const double* s0 = op.synth0 + g0 * 12;
    const double* s1 = op.synth1 + g1 * 12;

    auto load_slice = [&](int a2, double (&v)[L][L]) {
      const int b2 = ROLE == 0 ? 0 : (a2 >= p) + (a2 >= 2 * p);
      const int64_t zo = int64_t(a2 - b2 * p) * fr.s2;
#pragma unroll
      for (int y = 0; y < L; ++y) {
        const int64_t base = ybase[y] + zo + (ROLE == 0 ? 0 : __ldg(&fp->src[yb[y] + 3 * b2]));
#pragma unroll
        for (int x = 0; x < L; ++x) v[y][x] = ok ? ldg_slice(src + base + int64_t(x) * fr.sn) : 0.0;
      }
    };
    auto project = [&](int a2, const double (&v)[L][L]) {
      double T[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) T[t] = 0.0;
#pragma unroll
      for (int y = 0; y < L; ++y) {
        double m[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          m[a] = 0.0;
#pragma unroll
          for (int x = 0; x < L; ++x) gacc(m[a], Gram<L>::P(a, x), v[y][x]);
        }
        int t = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b + a < D; ++b, ++t) gacc(T[t], Gram<L>::P(b, y), m[a]);
      }
      double* slot = ring + (a2 % L) * (NT * 32);
#pragma unroll
      for (int t = 0; t < NT; ++t) slot[t * 32] = T[t];
    };
    auto finish = [&](int g2, int w2, const int4& G2) {
      // z-pass over the ring, synthesis at the children, store
      double M[NM];
#pragma unroll
      for (int i = 0; i < NM; ++i) M[i] = 0.0;
      const int slot0 = w2 % L;
#pragma unroll
      for (int z = 0; z < L; ++z) {
        const int sl = slot0 + z >= L ? slot0 + z - L : slot0 + z;
        const double* slot = ring + sl * (NT * 32);
        int t = 0, mi = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b + a < D; ++b, ++t) {
            const double Tz = slot[t * 32];
#pragma unroll
            for (int c = 0; c + b + a < D; ++c, ++mi) gacc(M[mi], Gram<L>::P(c, z), Tz);
          }
      }
      const double* s2 = op.synth1 + g2 * 12;
      bool bad = false;
      double* const dbase = dst + fr.dst + cb + lane;
#pragma unroll
      for (int l = 0; l < CT; ++l) {
        const int tz = G2.z + l;
        if (!(l < G2.w && tz >= fr.lo2 && tz < fr.lo2 + p)) continue;
        const int64_t do2 = int64_t(tz - fr.lo2) * fr.d2;
        double Q[NT];
        int t = 0, mi = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b + a < D; ++b, ++t) {
            Q[t] = 0.0;
#pragma unroll
            for (int c = 0; c + b + a < D; ++c, ++mi) Q[t] = fma(ldg_slice(s2 + l * 4 + c), M[mi], Q[t]);
          }
#pragma unroll
        for (int j = 0; j < CT; ++j) {
          if (!ok1[j]) continue;
          double R[D];
          int tt = 0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            R[a] = 0.0;
#pragma unroll
            for (int b = 0; b + a < D; ++b, ++tt) R[a] = fma(ldg_slice(s1 + j * 4 + b), Q[tt], R[a]);
          }
#pragma unroll
          for (int i = 0; i < C0; ++i) {
            if (!ok0[i]) continue;
            double o = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) o = fma(ldg_slice(s0 + i * 4 + a), R[a], o);
            if (ok) {
              dbase[do0[i] + do1[j] + do2] = o;
              bad |= !isfinite(o);
            }
          }
        }
      }
      raise_flag(flag, bad);
    };

    // ---- stream the t2 slices of all blocks in order ------------------------------
    // windows of consecutive groups advance monotonically without gaps, so the
    // slices needed are exactly [w2(first), w2(last) + L)
    int g2n = fr.g2;  // next block to complete
    const int g2e = fr.g2 + fr.n2;
    if (g2n >= g2e) continue;
    int4 Gn = __ldg(&op.grp1[g2n]);
    const int a_begin = Gn.x, a_end = __ldg(&op.grp1[g2e - 1]).x + L;
    double v[2][L][L];
    load_slice(a_begin, v[0]);
#pragma unroll 1
    for (int a2 = a_begin; a2 < a_end; a2 += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a2 + h;
        if (a < a_end) {
          if (a + 1 < a_end) load_slice(a + 1, v[1 - h]);
          project(a, v[h]);
          while (g2n < g2e && Gn.x + L - 1 == a) {
            finish(g2n, Gn.x, Gn);
            if (++g2n < g2e) Gn = __ldg(&op.grp1[g2n]);
          }
          asm volatile("" ::: "memory");  // the next slice's loads stay one slice ahead
        }
      }
    }
  }
}
