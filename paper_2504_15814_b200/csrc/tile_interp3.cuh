// Staged tile interpolation for order3 (5-cell Gram windows), included by
// trihalo.cu after tile_interp.cuh.
//
// Same arithmetic as gram_slide_kernel<3, 0> (the reference's least-squares rows,
// taylor.py:171-219, as the projection onto total degree <= 3 with the window's
// discrete Gram polynomials), organised so that no source load sits on a thread's
// critical path and the normal / t1 passes are shared by every block that needs them:
//
//  * a tile = (face, chunk of <= 30 unknowns); its source support (5 normal x <= 7 x <= 7
//    coarse cells: the whole segment at p <= 9) is copied into a shared-memory box with
//    8-byte cp.async two tiles ahead, and the tile after that is L2-prefetched;
//  * phase A (lane = unknown, one warp per t2 slice z of the box): the x (normal) Gram
//    moments of the slice's <= 7 lines, then the y moments of each distinct t1 window start
//    s (<= 3), written as T[s][z][pair] to a second shared region;
//  * phase B (warp = block of the segment's 3 x 3 coarse blocks, lane = unknown): the
//    block's z moments from its 5 T slices, the synthesis at its <= 27 children, direct
//    stores (a warp writes contiguous runs of unknowns);
//  * the two phases run in different warps of one CTA per SM, on consecutive tiles (see
//    tile3p_interp_kernel below).
#pragma once

constexpr int T3Y = 7;                    // box extent along t1 / t2 (three 5-cell windows within 7 cells)
constexpr int T3BOX = 5 * T3Y * T3Y;      // 245 cells: odd pitch, conflict-free 8-byte accesses
constexpr int T3TP = 3 * T3Y * 10;        // T region per unknown: [start s][z][pair t]; 210 = 2 mod 16
                                          // doubles: 16-byte accesses of consecutive unknowns are
                                          // conflict-free (pairs of T values per LDS.128 / STS.128)

// the normal synthesis table of the operator's single normal group, [child][4], passed as a
// kernel parameter: the synthesis FMAs take it straight from the constant bank
struct T3Syn0 {
  double v[12];
};

struct Tile3Hdr {
  int64_t src_off;     // source cell (normal window start, box origin along t1 / t2)
  int64_t dst_off;     // target origin of the face
  int64_t sn, s1, s2;  // signed source strides (reference frame)
  int64_t dn, d1, d2;  // target strides
  int lo1, lo2;        // target index origin of the segment along t1 / t2
  int g0, g1, n1, g2, n2;
  int y0, ny, z0, nz;  // the box along t1 / t2
  int cb, cn;          // the tile's unknowns [cb, cb + cn)
  unsigned n1mag, cnmag, nymag;
  int narrow;          // every target offset inside the face fits 32 bits
  int4 G0;             // the normal group (window start, length, first target, children)
};

// 4 table doubles through two 16-byte shared-memory loads (p 16-byte aligned)
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}

// first unknown of chunk c of nch; align: boundaries rounded down to 4 unknowns (32-byte
// sectors of the AoS cells) when the host asks for it
__device__ __forceinline__ int tile3_bound(int c, int nch, int u, int align) {
  if (c >= nch) return u;
  const int b = c * u / nch;
  return align ? (b & ~3) : b;
}

// tile = ((face, t2 tile, t1 tile), chunk): a face splits into nt x nt spatial tiles of <= 3 x 3
// blocks (nt = 1 at p <= 9) and every spatial tile into nch chunks of unknowns
__device__ __forceinline__ void tile3_decode(const DevOp& op, const th_face* __restrict__ faces, int64_t tile,
                                             int nt, int nch, int align, int u, Tile3Hdr& H, const int4* grp) {
  const int64_t st = tile / nch;
  const int c = int(tile - st * nch);
  const int64_t f = st / (nt * nt);
  const int tt = int(st - f * (nt * nt));
  const int ti2 = tt / nt, ti1 = tt - ti2 * nt;
  FaceRef fr;
  decode_face_interp(faces + f, op, fr);
  const int a1 = ti1 * fr.n1 / nt, b1 = (ti1 + 1) * fr.n1 / nt;
  const int a2 = ti2 * fr.n2 / nt, b2 = (ti2 + 1) * fr.n2 / nt;
  H.g0 = fr.g0;
  H.g1 = fr.g1 + a1;
  H.n1 = b1 - a1;
  H.g2 = fr.g2 + a2;
  H.n2 = b2 - a2;
  H.dst_off = fr.dst;
  H.sn = fr.sn;
  H.s1 = fr.s1;
  H.s2 = fr.s2;
  H.dn = fr.dn;
  H.d1 = fr.d1;
  H.d2 = fr.d2;
  H.lo1 = fr.lo1;
  H.lo2 = fr.lo2;
  H.cb = tile3_bound(c, nch, u, align);
  H.cn = tile3_bound(c + 1, nch, u, align) - H.cb;
  if (H.n1 <= 0 || H.n2 <= 0) {
    H.n1 = H.n2 = 1;
    H.y0 = H.z0 = 0;
    H.ny = H.nz = 0;
    H.cn = 0;
  } else {
    H.y0 = grp[H.g1].x;
    H.ny = grp[H.g1 + H.n1 - 1].x + 5 - H.y0;
    H.z0 = grp[H.g2].x;
    H.nz = grp[H.g2 + H.n2 - 1].x + 5 - H.z0;
  }
  const int4 G0 = __ldg(&op.grp0[0]);  // the single normal group (prepare_tile3)
  H.G0 = G0;
  H.src_off = fr.src0 + int64_t(G0.x) * fr.sn + int64_t(H.y0) * fr.s1 + int64_t(H.z0) * fr.s2 + H.cb;
  H.n1mag = recip16(H.n1);
  H.cnmag = recip16(max(H.cn, 1));
  H.nymag = recip16(max(H.ny, 1));
  const int64_t lim = int64_t(1) << 21;
  auto small = [lim](int64_t s) { return s > -lim && s < lim; };
  H.narrow = small(fr.dn) && small(fr.d1) && small(fr.d2) && op.p <= 64 && u <= (1 << 20);
}

// L2 prefetch of a tile's box: one source cell per thread, the <= 3 128-byte lines of its chunk
template <int NTH>
__device__ __forceinline__ void tile3_prefetch_l2(const Tile3Hdr& H, const double* __restrict__ src, int tid = -1) {
  const int n = H.ny * H.nz * 5;
  if (H.cn <= 0) return;
  if (tid < 0) tid = threadIdx.x;
  const int last = H.cn * 8 - 1, ny = H.ny;
  const unsigned nymag = H.nymag;
  const char* const base = reinterpret_cast<const char*>(src + H.src_off);
#pragma unroll 1
  for (int c = tid; c < n; c += NTH) {
    const int r = int((unsigned(c) * 13108u) >> 16);  // c / 5 (exact for c < 16384)
    const int x = c - 5 * r;
    const int z = int((unsigned(r) * nymag) >> 16), y = r - z * ny;
    const char* const pc = base + 8 * (int64_t(x) * H.sn + int64_t(y) * H.s1 + int64_t(z) * H.s2);
    l2_prefetch_line(pc);
    l2_prefetch_line(pc + 128);
    l2_prefetch_line(pc + last);
  }
}

// phase A: item (z, q) -> T[q][s][z][t] for every window start s of the box (NY = box
// extent along t1, compile-time so the line moments stay in registers)
template <int NY>
__device__ __forceinline__ void tile3_phase_a_ny(const Tile3Hdr& H, const double* box, double* tr, double& chk,
                                                 int z) {
  const int q = threadIdx.x & 31;
  {
    const double* bz = box + q * T3BOX + 5 * T3Y * z;
    double mm[NY][4];
#pragma unroll
    for (int y = 0; y < NY; ++y) {
      double v[5];
#pragma unroll
      for (int x = 0; x < 5; ++x) v[x] = bz[5 * y + x];
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH >= 3
      for (int a = 0; a < 4; ++a) mm[y][a] = v[a] + v[4];
#else
      gram_moments<5, 4>(v, mm[y]);
#endif
      asm volatile("" ::: "memory");  // one line of loads live at a time (register budget)
    }
    double* const tq = tr + q * T3TP + 10 * z;
#pragma unroll
    for (int s = 0; s + 4 < NY; ++s) {
      double w[5][4];
#pragma unroll
      for (int y = 0; y < 5; ++y)
#pragma unroll
        for (int a = 0; a < 4; ++a) w[y][a] = mm[s + y][a];
      double T[10];
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH >= 3
      for (int t = 0; t < 10; ++t) T[t] = w[t % 5][t % 4];
#else
      gram_y<5, 4>(w, T);
#endif
      // every box value enters some window's T_00 (the windows cover the box's t1 extent)
      chk = fma(T[0], 0.0, chk);
#pragma unroll
      for (int t = 0; t < 10; t += 2)
        *reinterpret_cast<double2*>(tq + s * (10 * T3Y) + t) = make_double2(T[t], T[t + 1]);
    }
  }
}

// phase B: item (block, q): z moments from T, synthesis at the children, stores
template <int NTH, bool ALL, typename OFF>
__device__ __forceinline__ void tile3_item(const double* tq, const T3Syn0& s0, const double* r1, const double* r2,
                                           double* __restrict__ hdst, OFF qo, OFF d1, OFF d2, const OFF (&do0)[3],
                                           const bool (&ok0)[3], const bool (&ok1)[3], const bool (&ok2)[3]) {
  // z moments of the 10 (a, b) columns, two columns per 16-byte load; M index of column
  // t = (a, b) is MO[t] (a-major, 4 - a - b moments each)
  constexpr int MO[10] = {0, 4, 7, 9, 10, 13, 15, 16, 18, 19};
  constexpr int MN[10] = {4, 3, 2, 1, 3, 2, 1, 2, 1, 1};
  double M[20];
#pragma unroll
  for (int t = 0; t < 10; t += 2) {
    double ca[5], cb[5];
#pragma unroll
    for (int z = 0; z < 5; ++z) {
      const double2 v = *reinterpret_cast<const double2*>(tq + 10 * z + t);
      ca[z] = v.x;
      cb[z] = v.y;
    }
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH >= 3
    for (int k = 0; k < MN[t]; ++k) M[MO[t] + k] = ca[k] + ca[4];
    for (int k = 0; k < MN[t + 1]; ++k) M[MO[t + 1] + k] = cb[k] + cb[4];
#else
    gram_moments_n<5>(ca, M + MO[t], MN[t]);
    gram_moments_n<5>(cb, M + MO[t + 1], MN[t + 1]);
#endif
    asm volatile("" ::: "memory");  // one column pair of loads live at a time
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (!ALL && !ok2[l]) continue;
    asm volatile("" ::: "memory");  // table values re-read per child (not hoisted into registers)
    double S2[4];
    ld4(r2 + l * 4, S2);
    double Q[10];
    int t = 0, mi = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b + a < 4; ++b, ++t) {
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH >= 3
        Q[t] = M[mi] + S2[b];
        mi += 4 - a - b;
#else
        Q[t] = 0.0;
#pragma unroll
        for (int c = 0; c + b + a < 4; ++c, ++mi) Q[t] = fma(S2[c], M[mi], Q[t]);
#endif
      }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (!ALL && !ok1[j]) continue;
      asm volatile("" ::: "memory");  // S1 re-read per child
      double S1[4];
      ld4(r1 + j * 4, S1);
      double R[4];
      int tt = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH >= 2
        R[a] = Q[a + j] + S1[a];
#else
        R[a] = 0.0;
#pragma unroll
        for (int b = 0; b + a < 4; ++b, ++tt) R[a] = fma(S1[b], Q[tt], R[a]);
#endif
      }
      const OFF oj = qo + OFF(l) * d2 + OFF(j) * d1;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
#ifdef TH_AB_NOSYNTH  // diagnosis build: the stores without the last synthesis stage
        const double oi = R[i];
#else
        double oi = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) oi = fma(s0.v[i * 4 + a], R[a], oi);  // constant-bank operands
#endif
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH == 4  // ... and (almost) no stores: one child per block
        if ((ALL || ok0[i]) && (i + j + l == 0 || oi == 1.2345e300)) *elem(hdst, oj + do0[i]) = oi;
#else
        if (ALL || ok0[i]) *elem(hdst, oj + do0[i]) = oi;
#endif
      }
    }
  }
}

#ifdef TH_AB_DMMA
// A/B variant (build with -DTH_AB_DMMA; profiles/r02_ab_dmma.txt): the synthesis of phase B on
// the FP64 tensor cores.  Per block the children x moments matrix Syn[ch][mi] = S0[i][a] S1[j][b]
// S2[l][c] (27 x 20, rows padded to 32) multiplies the moments of 8 unknowns at a time:
// mma.sync.m8n8k4.f64 (one DMMA.8x8x4 per instruction on sm_100a), A = Syn tile (row = child),
// B = moments (row = moment, column = unknown), 4 row tiles x 5 k-steps per group of 8 unknowns.
// The z moments are computed as in tile3_item (lane = unknown) and reach the B fragments
// through shuffles.
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename OFF>
__device__ __forceinline__ void tile3_item_dmma(const double* tq, const T3Syn0& s0, const double* r1,
                                                const double* r2, double* __restrict__ hdst, OFF qo0, OFF d1, OFF d2,
                                                const OFF (&do0)[3], const bool (&ok0)[3], const bool (&ok1)[3],
                                                const bool (&ok2)[3], int cn) {
  constexpr int MO[10] = {0, 4, 7, 9, 10, 13, 15, 16, 18, 19};
  constexpr int MN[10] = {4, 3, 2, 1, 3, 2, 1, 2, 1, 1};
  const int lane = threadIdx.x & 31, n = lane >> 2, kq = lane & 3;
  double M[20];
#pragma unroll
  for (int t = 0; t < 10; t += 2) {
    double ca[5], cb[5];
#pragma unroll
    for (int z = 0; z < 5; ++z) {
      const double2 v = *reinterpret_cast<const double2*>(tq + 10 * z + t);
      ca[z] = v.x;
      cb[z] = v.y;
    }
    gram_moments_n<5>(ca, M + MO[t], MN[t]);
    gram_moments_n<5>(cb, M + MO[t + 1], MN[t + 1]);
  }
  // (a, b, c) of moment mi, 2 bits each, packed: mi -> bits [6 mi, 6 mi + 6)
  constexpr unsigned long long PK_LO = [] {
    unsigned long long v = 0;
    int mi = 0;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; a + b < 4; ++b)
        for (int c = 0; a + b + c < 4; ++c, ++mi)
          if (mi < 10) v |= (unsigned long long)(a | (b << 2) | (c << 4)) << (6 * mi);
    return v;
  }();
  constexpr unsigned long long PK_HI = [] {
    unsigned long long v = 0;
    int mi = 0;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; a + b < 4; ++b)
        for (int c = 0; a + b + c < 4; ++c, ++mi)
          if (mi >= 10) v |= (unsigned long long)(a | (b << 2) | (c << 4)) << (6 * (mi - 10));
    return v;
  }();
  double A[4][5];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ch = 8 * r + n;  // child (i, j, l), i fastest
    const int l = ch / 9, j = (ch / 3) % 3, i = ch % 3;
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const int mi = 4 * st + kq;
      const unsigned e = unsigned((mi < 10 ? PK_LO >> (6 * mi) : PK_HI >> (6 * (mi - 10))) & 63u);
      const int a = e & 3, b = (e >> 2) & 3, c = e >> 4;
      A[r][st] = ch < 27 ? s0.v[i * 4 + a] * r1[j * 4 + b] * r2[l * 4 + c] : 0.0;
    }
  }
#pragma unroll 1
  for (int g = 0; g * 8 < cn; ++g) {
    const int srcl = 8 * g + n;
    double B[5];
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const double v0 = __shfl_sync(0xffffffffu, M[4 * st + 0], srcl);
      const double v1 = __shfl_sync(0xffffffffu, M[4 * st + 1], srcl);
      const double v2 = __shfl_sync(0xffffffffu, M[4 * st + 2], srcl);
      const double v3 = __shfl_sync(0xffffffffu, M[4 * st + 3], srcl);
      B[st] = kq == 0 ? v0 : kq == 1 ? v1 : kq == 2 ? v2 : v3;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double C[2] = {0.0, 0.0};
#pragma unroll
      for (int st = 0; st < 5; ++st) dmma884(C, A[r][st], B[st]);
      const int ch = 8 * r + n;
      const int l = ch / 9, j = (ch / 3) % 3, i = ch % 3;
      if (ch < 27 && ok0[i] && ok1[j] && ok2[l]) {
        const int q = 8 * g + 2 * kq;
        const OFF o = qo0 + OFF(q) + OFF(l) * d2 + OFF(j) * d1 + do0[i];
        if (q < cn) *elem(hdst, o) = C[0];
        if (q + 1 < cn) *elem(hdst, o + 1) = C[1];
      }
    }
  }
}
#endif

template <int NTH, typename OFF>
__device__ __forceinline__ void tile3_phase_b(const Tile3Hdr& H, const DevOp& op, double* __restrict__ dst,
                                              const double* tr, const double* stab, const T3Syn0& s0,
                                              const int4* sgrp, int blk = -1) {
  const int4 G0 = H.G0;
  bool ok0[3];
  OFF do0[3];
  bool all0 = true;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int t = G0.z + i;
    ok0[i] = i < G0.w && t >= 0 && t < op.k;
    do0[i] = OFF(t) * OFF(H.dn);
    all0 &= ok0[i];
  }
  const OFF d1 = OFF(H.d1), d2 = OFF(H.d2);
  const int p = op.p, lo1 = H.lo1, lo2 = H.lo2, n1 = H.n1, g1b = H.g1, g2b = H.g2, y0 = H.y0, z0 = H.z0;
  const int cb = H.cb;
  double* const hdst = dst + H.dst_off;
  // item (block, q) = (warp, lane): table reads are broadcasts, T reads conflict-free
  if (blk < 0) blk = threadIdx.x >> 5;
  const int q = threadIdx.x & 31;
#ifdef TH_AB_DMMA
  if (blk < n1 * H.n2) {  // whole warps: mma.sync
    const int b2 = int((unsigned(blk) * H.n1mag) >> 16);
    const int b1 = blk - b2 * n1;
    const int g1 = g1b + b1, g2 = g2b + b2;
    const int4 G1 = sgrp[g1], G2 = sgrp[g2];
    bool ok1[3], ok2[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      ok1[j] = j < G1.w && unsigned(G1.z + j - lo1) < unsigned(p);
      ok2[j] = j < G2.w && unsigned(G2.z + j - lo2) < unsigned(p);
    }
    const int qc = min(q, H.cn - 1);  // lanes past the chunk read a valid unknown's T
    const double* tq = tr + (qc * T3TP + (G1.x - y0) * (10 * T3Y) + 10 * (G2.x - z0));
    const OFF qo0 = OFF(G1.z - lo1) * d1 + OFF(G2.z - lo2) * d2 + OFF(cb);
    tile3_item_dmma<OFF>(tq, s0, stab + g1 * 12, stab + g2 * 12, hdst, qo0, d1, d2, do0, ok0, ok1, ok2, H.cn);
  }
  return;
#endif
  if (blk < n1 * H.n2 && q < H.cn) {
    const int b2 = int((unsigned(blk) * H.n1mag) >> 16);
    const int b1 = blk - b2 * n1;
    const int g1 = g1b + b1, g2 = g2b + b2;
    const int4 G1 = sgrp[g1], G2 = sgrp[g2];
    bool ok1[3], ok2[3];
    bool all = all0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      ok1[j] = j < G1.w && unsigned(G1.z + j - lo1) < unsigned(p);
      ok2[j] = j < G2.w && unsigned(G2.z + j - lo2) < unsigned(p);
      all &= ok1[j] & ok2[j];
    }
    const double* tq = tr + (q * T3TP + (G1.x - y0) * (10 * T3Y) + 10 * (G2.x - z0));
    const OFF qo = OFF(G1.z - lo1) * d1 + OFF(G2.z - lo2) * d2 + OFF(cb + q);
    const double* r1 = stab + g1 * 12;
    const double* r2 = stab + g2 * 12;
    if (all) tile3_item<NTH, true, OFF>(tq, s0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
    else tile3_item<NTH, false, OFF>(tq, s0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
  }
}

// ---------------------------------------------------------------------------
// The kernel: phase A and phase B of consecutive tiles run at the same time.
//
// (Round 1's kernel ran both phases in one group of 9 warps: phase A kept <= 7 of them busy and
// both phases ended in a CTA barrier -- barrier the top stall, 2.1 cycles per issue; 0.526 of
// the copy peak on config 5 against 0.60 here, profiles/r02_ab_tile3p.txt.)
// Here a CTA is NA3 "A" warps + 9 "B" warps.  A warps fetch (cp.async) and project tile i
// into T[i % 2] while B warps synthesise tile i - 1 from T[(i - 1) % 2]; boxes and T are
// double-buffered, and the hand-off uses named barriers:
//   T_FULL[k] (id 1 + k, all)        T[k] written (A arrive, B sync)
//   T_EMPTY[k] (id 1 + NT + k, all)  T[k] consumed (B arrive, A sync before rewriting it)
// (mbarrier arrive / try_wait spin hand-offs instead measured 8% slower: the spinning waits
// take issue slots, profiles/r02_ab_tile3p.txt.)
// A warp w fetches and projects box slice z = w only (each lane reads only what it copied),
// so A warps never wait for one another.  They also decode the tile headers (ring of 8) and
// L2-prefetch the tile after next.
// ---------------------------------------------------------------------------
constexpr int NA3 = T3Y;               // A warps: one per t2 slice of the box
constexpr int T3P_NTH = (NA3 + 9) * 32;
__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int T3PCMAX = 30;            // unknowns per tile: NBOX boxes + NT T buffers within 227 KB
#ifndef T3P_NBOX
#define T3P_NBOX 2                     // source boxes (A / B builds: -DT3P_NBOX=1 -DT3P_NT=3)
#endif
#ifndef T3P_NT
#define T3P_NT 2                       // T buffers between the A and B warps
#endif

__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// cp.async copies of t2 slice z of a tile's box (all its t1 lines), lanes over the chunk's unknowns
__device__ __forceinline__ void tile3_fetch_slice(const Tile3Hdr& H, const double* __restrict__ src, double* box, int z) {
  const int lane = threadIdx.x & 31;
  if (lane >= H.cn || z >= H.nz) return;
  const int64_t sn = H.sn, s1 = H.s1;
  const double* const base = src + (H.src_off + lane + int64_t(z) * H.s2);
  double* const bq = box + lane * T3BOX + 5 * T3Y * z;
#pragma unroll 1
#if defined(TH_AB_NOSYNTH) && TH_AB_NOSYNTH == 5  // ... and (almost) no source copies: one line per slice
  for (int y = 0; y < min(H.ny, 1); ++y) {
#else
  for (int y = 0; y < H.ny; ++y) {
#endif
    const double* cell = base + int64_t(y) * s1;
#pragma unroll
    for (int x = 0; x < 5; ++x, cell += sn) cp_async8(bq + 5 * y + x, cell);
  }
}

// dynamic shared memory: sgrp int4[G1] | stab [G1][12] | (unused [G0][12] slot) | box[2][cmax][T3BOX]
// (each rounded to an even count) | T[2][cmax][T3TP]
__global__ void __launch_bounds__(T3P_NTH, 1)
    tile3p_interp_kernel(DevOp op, T3Syn0 syn0, const double* __restrict__ src, double* __restrict__ dst,
                         const th_face* __restrict__ faces, int64_t n_tiles, int nt, int nch, int align, int cmax,
                         int u, int32_t* flag) {
  extern __shared__ __align__(16) double smem_t3p[];
  __shared__ Tile3Hdr Hs[8];

  const int G1n = op.G1;
  int4* const sgrp = reinterpret_cast<int4*>(smem_t3p);
  double* const stab = smem_t3p + 2 * G1n;
  const int boxd = (cmax * T3BOX + 1) & ~1, trd = cmax * T3TP;
  double* const box0 = smem_t3p + tile_box_offset(12, op.G0, G1n);
  double* const tr0 = box0 + T3P_NBOX * boxd;
  for (int i = threadIdx.x; i < G1n; i += T3P_NTH) sgrp[i] = __ldg(&op.grp1[i]);
  for (int i = threadIdx.x; i < G1n * 12; i += T3P_NTH) stab[i] = __ldg(op.synth1 + i);
  const int warp = threadIdx.x >> 5;
  const int64_t t0 = blockIdx.x, step = gridDim.x;
  constexpr int ALL = T3P_NTH, ANTH = NA3 * 32;
  constexpr int NBX = T3P_NBOX, NT = T3P_NT;
  // named barriers: T_FULL[k] = 1 + k, T_EMPTY[k] = 1 + NT + k (bar.arrive by the producing
  // group, bar.sync by the consuming group; counts include both groups)
  static_assert(2 * NT + 1 <= 16 && NT + 5 <= 8 + 1, "named barriers / header ring");
  __syncthreads();  // tables filled: the header decodes read the group table from shared memory
  if (warp < NA3) {
    // ============ A warps: fetch, phase A ============
    // A warp w owns box slice z = w (NA3 == T3Y): it fetches that slice of every tile and takes
    // the slice's phase A items, each lane only ever reading the cp.async data it copied itself,
    // so the A warps need no barrier among themselves.
    static_assert(NA3 == T3Y, "one A warp per t2 slice of the box");
    const int atid = threadIdx.x;
    // tile headers are decoded 5 tiles ahead, tile i by lane 0 of A warp i mod NA3 (a warp that
    // decoded them all would reach every hand-off a global-memory latency after the others)
    if ((atid & 31) == 0)
      for (int i = warp; i < 5; i += NA3)
        if (t0 + i * step < n_tiles) tile3_decode(op, faces, t0 + i * step, nt, nch, align, u, Hs[i], sgrp);
    __syncthreads();  // (with the B warps: tables and headers 0..4 visible to everyone)
    for (int i = 0; i < NBX; ++i) {
      if (t0 + i * step < n_tiles) tile3_fetch_slice(Hs[i], src, box0 + i * boxd, warp);
      cp_async_commit();
    }
    if (t0 + NBX * step < n_tiles) tile3_prefetch_l2<ANTH>(Hs[NBX], src, atid);
    double chk = 0.0;
    int it = 0;
    for (int64_t tile = t0; tile < n_tiles; tile += step, ++it) {
      const int bx = NBX == 1 ? 0 : it % NBX, tb = it % NT;
      if constexpr (NBX == 1) cp_async_wait_all();   // this thread's slice of tile `it` landed
      else cp_async_wait_one();
      if (it >= NT) bar_sync_n(1 + NT + tb, ALL);     // B is done with T[tb] (tile it - NT)
      if ((atid & 31) == 0 && (it + 5) % NA3 == warp && tile + 5 * step < n_tiles)  // B is past tile it - NT
        tile3_decode(op, faces, tile + 5 * step, nt, nch, align, u, Hs[(it + 5) & 7], sgrp);
      const Tile3Hdr& H = Hs[it & 7];
      if (warp < H.nz && (threadIdx.x & 31) < H.cn) {
        double* const bxp = box0 + bx * boxd;
        if (H.ny == 5) tile3_phase_a_ny<5>(H, bxp, tr0 + tb * trd, chk, warp);
        else if (H.ny == 6) tile3_phase_a_ny<6>(H, bxp, tr0 + tb * trd, chk, warp);
        else if (H.ny == 7) tile3_phase_a_ny<7>(H, bxp, tr0 + tb * trd, chk, warp);
      }
      bar_arrive_n(1 + tb, ALL);                      // T[tb] ready (once every A thread arrived)
      if (tile + NBX * step < n_tiles) tile3_fetch_slice(Hs[(it + NBX) & 7], src, box0 + bx * boxd, warp);
      cp_async_commit();
      if (tile + (NBX + 1) * step < n_tiles) tile3_prefetch_l2<ANTH>(Hs[(it + NBX + 1) & 7], src, atid);
    }
    // drain: the B warps' T_EMPTY arrivals of the last NT tiles have no matching sync yet
    for (int k = it - NT; k < it; ++k)
      if (k >= 0) bar_sync_n(1 + NT + k % NT, ALL);
    cp_async_wait_all();
    raise_flag(flag, !isfinite(chk));
  } else {
    // ============ B warps: phase B (warp = block of the 3 x 3 tile) ============
    __syncthreads();
    int it = 0;
    for (int64_t tile = t0; tile < n_tiles; tile += step, ++it) {
      const int tb = it % NT;
      bar_sync_n(1 + tb, ALL);                   // T[tb] holds tile `it`
      const Tile3Hdr& H = Hs[it & 7];
      // phase B with the B warps renumbered 0..8 (tile3_phase_b maps warp -> block)
      if (H.narrow) tile3_phase_b<T3P_NTH, int>(H, op, dst, tr0 + tb * trd, stab, syn0, sgrp, warp - NA3);
      else tile3_phase_b<T3P_NTH, int64_t>(H, op, dst, tr0 + tb * trd, stab, syn0, sgrp, warp - NA3);
      bar_arrive_n(1 + NT + tb, ALL);            // T[tb] consumed
    }
  }
}
