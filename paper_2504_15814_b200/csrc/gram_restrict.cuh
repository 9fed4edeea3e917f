// order3 restriction, Gram-separable, asynchronous slice pipeline (included by
// trihalo.cu after gram_slide.cuh).
//
// Same projection as gram_slide.cuh (least-squares fit over the 5x5x5 window =
// orthogonal projection onto total degree <= 3 with the window's Gram
// polynomials, evaluated at the three coarse layers), organised for the
// restriction's access pattern:
//   * a warp owns (face, coarse t1 column j1, 32-unknown chunk) and streams the
//     face's 3p fine t2 slices a2 = 0 .. 3p-1; each slice is the 5 (normal) x 5
//     (t1 window) cells of that t2 row;
//   * slices arrive through an NST-deep ring in shared memory filled with
//     8-byte cp.async (the unpadded u = 59 cells are only 8-byte aligned), so
//     NST-1 slices per warp are in flight without holding registers; every lane
//     copies and later reads only its own unknown, so no warp synchronisation
//     is needed;
//   * a slice belongs to at most two coarse t2 columns (windows of 5 fine cells
//     at stride 3), so the z-moments accumulate in two register sets and a
//     column is synthesised and stored the moment its last slice is in.
#pragma once

template <int NST, int MINB>
__global__ void __launch_bounds__(128, MINB) gram_restrict3_kernel(DevOp op, const double* __restrict__ src,
                                                                   double* __restrict__ dst,
                                                                   const th_face* __restrict__ faces,
                                                                   int64_t n_faces, int u, int32_t* flag) {
  constexpr int L = 5, D = 4, NT = 10, NM = 20, SL = L * L;
  extern __shared__ double ring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const ring = ring_all + size_t(warp) * NST * SL * 32 + lane;  // [slot][cell][lane]
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
  const int p = op.p;
  const int G1n = op.G1;
  const int nch = (u + 31) / 32;
  const int64_t total = n_faces * G1n * nch;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t unit = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; unit < total; unit += nw) {
    const int64_t fu = unit / nch;
    const int cb = int(unit - fu * nch) * 32;
    const int64_t f = fu / G1n;
    const int g1 = int(fu - f * G1n);
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face(fp, op, fr);
    const int4 G0 = __ldg(&op.grp0[fr.g0]), G1 = __ldg(&op.grp1[g1]);
    const bool ok = cb + lane < u;
    const int64_t adj = fr.src0 - __ldg(&fp->src[0]) + int64_t(G0.x) * fr.sn + cb + lane;
    int64_t ybase[L];
    int yb[L];
#pragma unroll
    for (int y = 0; y < L; ++y) {
      const int a1 = G1.x + y;
      yb[y] = (a1 >= p) + (a1 >= 2 * p);
      ybase[y] = adj + int64_t(a1 - yb[y] * p) * fr.s1;
    }
    const int n_slices = op.ns_t;  // 3p fine t2 rows, all covered by the columns' windows

    auto issue = [&](int s) {
      if (s < n_slices) {
        const int b2 = (s >= p) + (s >= 2 * p);
        const int64_t zo = int64_t(s - b2 * p) * fr.s2;
        const unsigned slot = ring_s + unsigned((s % NST) * SL * 32) * 8u;
#pragma unroll
        for (int y = 0; y < L; ++y) {
          const double* row = src + (ybase[y] + zo + __ldg(&fp->src[yb[y] + 3 * b2]));
#pragma unroll
          for (int x = 0; x < L; ++x)
            if (ok) cp_async8(slot + unsigned((y * L + x) * 32) * 8u, row + int64_t(x) * fr.sn);
        }
      }
      cp_async_commit();
    };

    // z-moment accumulators of the (at most two) columns the current slice feeds
    int jc = 0;
    int4 Gc = __ldg(&op.grp1[0]), Gn = __ldg(&op.grp1[G1n > 1 ? 1 : 0]);
    double MA[NM], MB[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) MA[i] = MB[i] = 0.0;
    const double* s0 = op.synth0 + fr.g0 * 12;
    const double* s1 = op.synth1 + g1 * 12;
    const int t1 = G1.z;
    const bool t1_in = t1 >= fr.lo1 && t1 < fr.lo1 + p;
    bool bad = false;

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) issue(s);
#pragma unroll 1
    for (int s = 0; s < n_slices; ++s) {
      issue(s + NST - 1);
      cp_async_wait<NST - 1>();
      // x / y projection of slice s from the ring (lane-private data)
      const double* slot = ring + (s % NST) * SL * 32;
      double T[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) T[t] = 0.0;
#pragma unroll
      for (int y = 0; y < L; ++y) {
        double v[L];
#pragma unroll
        for (int x = 0; x < L; ++x) v[x] = slot[(y * L + x) * 32];
        double m[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          m[a] = 0.0;
#pragma unroll
          for (int x = 0; x < L; ++x) gacc(m[a], Gram<L>::P(a, x), v[x]);
        }
        int t = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b + a < D; ++b, ++t) gacc(T[t], Gram<L>::P(b, y), m[a]);
      }
      // z-pass into the columns whose window holds slice s
      auto zacc = [&](double (&M)[NM], int z) {
        const double tz = double(z - 2);
        const double pz[D] = {1.0, tz, tz * tz - 2.0, (5.0 * tz * tz * tz - 17.0 * tz) / 6.0};
        int t = 0, mi = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b + a < D; ++b, ++t)
#pragma unroll
            for (int c = 0; c + b + a < D; ++c, ++mi) M[mi] = fma(pz[c], T[t], M[mi]);
      };
      if (s >= Gc.x && s < Gc.x + L) zacc(MA, s - Gc.x);
      if (jc + 1 < G1n && s >= Gn.x && s < Gn.x + L) zacc(MB, s - Gn.x);
      if (s == Gc.x + L - 1) {
        // column jc complete: synthesis at the three coarse layers, store
        const int t2 = Gc.z;
        if (t1_in && t2 >= fr.lo2 && t2 < fr.lo2 + p) {
          const double* s2 = op.synth1 + jc * 12;
          double Q[NT];
          int t = 0, mi = 0;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b + a < D; ++b, ++t) {
              Q[t] = 0.0;
#pragma unroll
              for (int c = 0; c + b + a < D; ++c, ++mi) Q[t] = fma(ldg_slice(s2 + c), MA[mi], Q[t]);
            }
          double R[D];
          int tt = 0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            R[a] = 0.0;
#pragma unroll
            for (int b = 0; b + a < D; ++b, ++tt) R[a] = fma(ldg_slice(s1 + b), Q[tt], R[a]);
          }
          double* dbase = dst + fr.dst + (t1 - fr.lo1) * fr.d1 + (t2 - fr.lo2) * fr.d2 + cb + lane;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int t0 = G0.z + i;
            if (i < G0.w && t0 >= fr.lo0 && t0 < fr.hi0) {
              double o = 0.0;
#pragma unroll
              for (int a = 0; a < D; ++a) o = fma(ldg_slice(s0 + i * 4 + a), R[a], o);
              if (ok) {
                dbase[(t0 - fr.lo0) * fr.dn] = o;
                bad |= !isfinite(o);
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NM; ++i) {
          MA[i] = MB[i];
          MB[i] = 0.0;
        }
        ++jc;
        Gc = Gn;
        if (jc + 1 < G1n) Gn = __ldg(&op.grp1[jc + 1]);
      }
    }
    cp_async_wait<0>();
    raise_flag(flag, bad);
  }
}
