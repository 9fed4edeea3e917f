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
// with S_d = P(e)/|P|^2 from the builder (builder.cpp choose_fast_path).
// Integer Gram weights are immediates: no weight loads at all.
//
// One warp owns a work unit = (face, t1 group, 32-unknown chunk) and walks the
// face's t2 groups.  Consecutive blocks' windows overlap along t2 (by 4 of 5
// slices for interpolation, 2 of 5 for restriction), so each source slice is
// loaded and x/y-projected once into a per-lane ring of L moment slices in
// shared memory; a block then only does its z-pass and synthesis.
#pragma once

// TENSOR = true runs tensor_linear through the same slice ring: the x / y / z
// passes apply the d-linear 1-D rows (normal, t1, t2 — the reference's
// contraction order, linear.py:115-151) instead of Gram projections, with
// ORDER = 2 standing for the 3-cell windows.
template <int ORDER, int ROLE, int MINB, bool TENSOR = false>
__global__ void __launch_bounds__(128, MINB) gram_slide_kernel(DevOp op, const double* __restrict__ src,
                                                               double* __restrict__ dst,
                                                               const th_face* __restrict__ faces, int64_t n_faces,
                                                               int u, int32_t* flag) {
  constexpr int L = ORDER == 2 ? 3 : 5;
  constexpr int D = ORDER + 1;
  constexpr int C0 = 3, CT = ROLE == 0 ? 3 : 1;
  constexpr int NT = TENSOR ? C0 * CT : (ORDER == 2 ? 6 : 10);  // per-slice values: pairs a + b <= ORDER
  constexpr int NM = ORDER == 2 ? 10 : 20;                      // triples a + b + c <= ORDER
  extern __shared__ double ring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const ring = ring_all + warp * (L * NT * 32) + lane;  // [slot][t] x 32 lanes, lane-private
  // synthesis tables of all groups in shared memory (broadcast reads; from global memory their
  // load latency was ~1/3 of the order3 interpolation's stalls)
  double* const ssyn0 = ring_all + (blockDim.x >> 5) * (L * NT * 32);
  double* const ssyn1 = ssyn0 + op.G0 * 12;
  if constexpr (!TENSOR) {
    for (int i = threadIdx.x; i < op.G0 * 12; i += blockDim.x) ssyn0[i] = __ldg(op.synth0 + i);
    for (int i = threadIdx.x; i < op.G1 * 12; i += blockDim.x) ssyn1[i] = __ldg(op.synth1 + i);
    __syncthreads();
  }
  const int p = op.p;
  const int upf = op.units_per_face;
  // finiteness of the inputs: every value of a source slice enters its T[0] (Gram: the plain
  // sum; tensor: an fma chain through all of them), so fma(T0, 0, chk) turns NaN for any
  // Inf / NaN in the support and stays 0 otherwise (checked once, at the end)
  double chk = 0.0;
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
    const int64_t ibase = fr.src0 + int64_t(G1.x) * fr.s1 + int64_t(G0.x) * fr.sn + cb + lane;
    int64_t ybase[ROLE == 0 ? 1 : L];
    int yb[ROLE == 0 ? 1 : L];
#pragma unroll
    for (int y = 0; y < (ROLE == 0 ? 1 : L); ++y) {
      const int a1 = G1.x + y;
      yb[y] = ROLE == 0 ? 0 : (a1 >= p) + (a1 >= 2 * p);
      ybase[y] = adj + int64_t(a1 - yb[y] * p) * fr.s1 + int64_t(G0.x) * fr.sn + cb + lane;
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
    // every normal / t1 child of this unit is a target (always at p = 9): the stores below
    // then need no per-child test (warp-uniform, but the compiler cannot know that)
    bool all01 = true;
#pragma unroll
    for (int i = 0; i < C0; ++i) all01 &= ok0[i];
#pragma unroll
    for (int i = 0; i < CT; ++i) all01 &= ok1[i];
    const double* s0 = ssyn0 + g0 * 12;
    const double* s1 = ssyn1 + g1 * 12;
    double R0[TENSOR ? C0 : 1][TENSOR ? L : 1], R1[TENSOR ? CT : 1][TENSOR ? L : 1];
    if constexpr (TENSOR) {
      const double* r0 = op.rows0 + __ldg(&op.row_off0[g0]);
      const double* r1 = op.rows1 + __ldg(&op.row_off1[g1]);
#pragma unroll
      for (int c = 0; c < C0; ++c)
#pragma unroll
        for (int x = 0; x < L; ++x) R0[c][x] = c < G0.w ? __ldg(r0 + c * L + x) : 0.0;
#pragma unroll
      for (int c = 0; c < CT; ++c)
#pragma unroll
        for (int y = 0; y < L; ++y) R1[c][y] = c < G1.w ? __ldg(r1 + c * L + y) : 0.0;
    }
    if (ROLE == 0 && (op.prefetch & 8)) {
      // L2 prefetch of the unit's whole source window (this chunk's <= 3 lines of every cell)
      // through the LSU, so that the slices walked below load at L2 rather than DRAM latency
      // (config 2 interpolation 0.55 -> 0.61 / 0.47 -> 0.51 of HBM; prefetching the warp's
      //  next unit as well measured slower: profiles/r01_ab_stage.txt)
      const int z0 = __ldg(&op.grp1[fr.g2]).x, nz = __ldg(&op.grp1[fr.g2 + fr.n2 - 1]).x + L - z0;
      const char* const c0 = reinterpret_cast<const char*>(src + (ibase - lane + int64_t(z0) * fr.s2));
      // a cell per lane and iteration, its <= 3 lines of this chunk (256 bytes at 8-byte alignment)
      for (int c = lane; c < L * L * nz; c += 32) {
        const int x = c % L, yz = c / L, y = yz % L, z = yz / L;
        const char* const pc = c0 + 8 * (int64_t(x) * fr.sn + int64_t(y) * fr.s1 + int64_t(z) * fr.s2);
        l2_prefetch_line(pc);
        l2_prefetch_line(pc + 128);
        l2_prefetch_line(pc + 255);
      }
    }
    int hi = -1;  // highest t2 source slice held in the ring
    for (int g2 = fr.g2; g2 < fr.g2 + fr.n2; ++g2) {
      const int4 G2 = __ldg(&op.grp1[g2]);
      const int w2 = G2.x;
      // ---- new source slices: load, x-pass, y-pass, into the ring ----------
#pragma unroll 1
      for (int a2 = max(hi + 1, w2); a2 < w2 + L; ++a2) {
        const int b2 = ROLE == 0 ? 0 : (a2 >= p) + (a2 >= 2 * p);
        const int64_t zo = int64_t(a2 - b2 * p) * fr.s2;
        // (no prefetch of the next slice: TMA bulk and per-line L2 prefetches both measured
        //  slower here, and indexing ybase[] at run time would push it to local memory)
        if (ok) {  // lanes past u skip the slice (one divergent region, no per-load predicate)
          double v[L][L];
  #pragma unroll
          for (int y = 0; y < L; ++y) {
            // interpolation rows are affine in y (one base + y * s1, fewer live registers);
            // restriction rows may cross a fine-block boundary, so they use the per-row table
            const int64_t base = ROLE == 0 ? ibase + zo + int64_t(y) * fr.s1
                                           : ybase[y] + zo + __ldg(&fp->src[yb[y] + 3 * b2]);
  #pragma unroll
            for (int x = 0; x < L; ++x) v[y][x] = ldg_slice(src + base + int64_t(x) * fr.sn);
          }
          double T[NT];
  #pragma unroll
          for (int t = 0; t < NT; ++t) T[t] = 0.0;
  #pragma unroll
          for (int y = 0; y < L; ++y) {
            if constexpr (TENSOR) {
  #pragma unroll
              for (int c0 = 0; c0 < C0; ++c0) {
                double tx = 0.0;
  #pragma unroll
                for (int x = 0; x < L; ++x) tx = fma(R0[c0][x], v[y][x], tx);
  #pragma unroll
                for (int c1 = 0; c1 < CT; ++c1) T[c0 + C0 * c1] = fma(R1[c1][y], tx, T[c0 + C0 * c1]);
              }
            } else {
              double m[D];
              gram_moments<L, D>(v[y], m);
              int t = 0;
  #pragma unroll
              for (int a = 0; a < D; ++a)
  #pragma unroll
                for (int b = 0; b + a < D; ++b, ++t) gacc(T[t], Gram<L>::P(b, y), m[a]);
            }
          }
          chk = fma(T[0], 0.0, chk);
          double* slot = ring + (a2 % L) * (NT * 32);
  #pragma unroll
          for (int t = 0; t < NT; ++t) slot[t * 32] = T[t];
        }
        asm volatile("" ::: "memory");  // one slice of loads live at a time
      }
      hi = max(hi, w2 + L - 1);
      if constexpr (TENSOR) {
        // ---- z-pass with the t2 rows straight into the children, store --------
        const double* r2 = op.rows1 + __ldg(&op.row_off1[g2]);
        const int slot0 = w2 % L;
        double* const dbase = dst + fr.dst + cb + lane;
#pragma unroll
        for (int l = 0; l < CT && ok; ++l) {  // lanes past u skip the z-pass and stores
          const int tz = G2.z + l;
          if (!(l < G2.w && tz >= fr.lo2 && tz < fr.lo2 + p)) continue;
          const int64_t do2 = int64_t(tz - fr.lo2) * fr.d2;
          double o[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) o[t] = 0.0;
#pragma unroll
          for (int z = 0; z < L; ++z) {
            const double w = ldg_slice(r2 + l * L + z);
            const int sl = slot0 + z >= L ? slot0 + z - L : slot0 + z;
            const double* slot = ring + sl * (NT * 32);
#pragma unroll
            for (int t = 0; t < NT; ++t) o[t] = fma(w, slot[t * 32], o[t]);
          }
          double* const dl = dbase + do2;
          if (all01) {
#pragma unroll
            for (int j = 0; j < CT; ++j)
#pragma unroll
              for (int i = 0; i < C0; ++i) {
                dl[do1[j] + do0[i]] = o[i + C0 * j];
              }
          } else {
#pragma unroll
            for (int j = 0; j < CT; ++j) {
              if (!ok1[j]) continue;
              double* const dj = dl + do1[j];
#pragma unroll
              for (int i = 0; i < C0; ++i)
                if (ok0[i]) dj[do0[i]] = o[i + C0 * j];
            }
          }
        }
        continue;
      }
      // ---- z-pass of this block (lanes past u skip it and the synthesis) -----------
      if (ok) {
        double M[NM];
        const int slot0 = w2 % L;
        {
          int t = 0, mi = 0;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b + a < D; ++b, ++t) {
              double col[L];  // T_ab over the window's slices -> its z moments
#pragma unroll
              for (int z = 0; z < L; ++z) {
                const int sl = slot0 + z >= L ? slot0 + z - L : slot0 + z;
                col[z] = ring[sl * (NT * 32) + t * 32];
              }
              gram_moments_n<L>(col, M + mi, D - a - b);
              mi += D - a - b;
            }
        }
        // ---- synthesis at the children and store -----------------------------------
        const double* s2 = ssyn1 + g2 * 12;
        double* const dbase = dst + fr.dst + cb + lane;
#pragma unroll
        for (int l = 0; l < CT; ++l) {
          const int tz = G2.z + l;
          if (!(l < G2.w && tz >= fr.lo2 && tz < fr.lo2 + p)) continue;
          double* const dl = dbase + int64_t(tz - fr.lo2) * fr.d2;
          double Q[NT];
          int t = 0, mi = 0;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b + a < D; ++b, ++t) {
              Q[t] = 0.0;
#pragma unroll
              for (int c = 0; c + b + a < D; ++c, ++mi) Q[t] = fma(s2[l * 4 + c], M[mi], Q[t]);
            }
#pragma unroll
          for (int j = 0; j < CT; ++j) {
            if (!all01 && !ok1[j]) continue;
            double R[D];
            int tt = 0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              R[a] = 0.0;
#pragma unroll
              for (int b = 0; b + a < D; ++b, ++tt) R[a] = fma(s1[j * 4 + b], Q[tt], R[a]);
            }
            double* const dj = dl + do1[j];
#pragma unroll
            for (int i = 0; i < C0; ++i) {
              if (!all01 && !ok0[i]) continue;
              double o = 0.0;
#pragma unroll
              for (int a = 0; a < D; ++a) o = fma(s0[i * 4 + a], R[a], o);
              dj[do0[i]] = o;
            }
          }
        }
      }  // ok
    }
  }
  raise_flag(flag, !isfinite(chk));
}
