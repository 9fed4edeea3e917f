// Slice-ring interpolation for the Gram least-squares schemes (order2: 3-cell windows,
// order3: 5-cell windows), included by trihalo.cu after tile_interp3.cuh.
//
// Same arithmetic as gram_slide_kernel<ORDER, 0> and the tiles of tile_interp3.cuh (the
// reference's least-squares rows, taylor.py:171-219, as the projection onto total degree
// <= ORDER with the window's discrete Gram polynomials, evaluated separably at the children),
// organised as a stream of t2 slices instead of whole-face tiles, so that it also fits the
// faces of large patches (p = 17: 6-7 blocks and 11 source cells per axis):
//
//  * a tile = (face, t1 part of <= 4 blocks, chunk of <= 32 unknowns); lanes run over the
//    chunk's unknowns, so every table value is warp-uniform and every lane's data chain
//    (source -> T -> children) is private to it;
//  * "A" warps each own every NA-th t2 slice of the CTA's tile sequence: cp.async the slice
//    (L x <= L + 3 cells) into a private staging slot one own-slice ahead, take the normal
//    Gram moments of its lines and the t1 moments of every window start of the part, and
//    write T[start][pair] into a slot of a ring of R slices;
//  * "B" warps take the blocks (row r of the face, block b1 of the part) round-robin: wait for
//    the L slices of the row's t2 window, take the block's t2 moments from the ring, release
//    the slices, synthesise the <= 27 children and store them;
//  * hand-offs: ready[slot] sequence numbers (written by the producing A warp, polled by the
//    blocks that read the slice), free[slot] mbarriers counting the slice's readers down
//    (transaction count), hdr[tile mod 32] (tile headers decoded 8 tiles ahead by one A
//    thread).  No warp ever waits for a warp of its own group, and an A warp only waits for
//    the blocks that read the slice it is about to overwrite.
#pragma once

constexpr int RG_NW = 16;                 // warps per CTA (one CTA per SM)
constexpr int RG_NTH = RG_NW * 32;
constexpr int RG_NS = 4;                  // blocks per row of a tile (t1 part)
constexpr int RG_NH = 32;                 // header ring
constexpr int RG_HAHEAD = 8;              // headers decoded ahead of the leading A iterator
constexpr int RG_RMAX = 32;               // T ring slots (upper bound)

#ifndef RG_DIRECT
#define RG_DIRECT 0                       // A warps load their slices straight into registers (0: cp.async staging)
#endif
#ifndef RG_PARTEST
#define RG_PARTEST 0                      // B warps test a row's new slices together before falling back to waits
#endif
#ifndef RG_PFD
#define RG_PFD 2                          // own slices between an A warp's projection and its L2 prefetch
#endif
#ifndef RG_WAIT_HINT
#define RG_WAIT_HINT 0                    // suspend-time hint (ns) of the hand-off waits; 0: none
#endif

__device__ __forceinline__ void rg_wait(uint64_t* b, unsigned parity) {
#if RG_WAIT_HINT > 0
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2; @!P bra WAIT_%=; }" ::"r"(
          smem_u32(b)),
      "r"(parity), "n"(RG_WAIT_HINT)
      : "memory");
#else
  mbar_wait(b, parity);
#endif
}

// wait of a warp that is ahead of its consumers (an A warp whose ring slot is still being
// read): back off between tries, so that the spinning does not take shared-memory issue slots
// from the warps it is waiting for
#ifndef RG_SLEEP
#define RG_SLEEP 200                      // ns between tries of an A warp's slot wait (0: plain try_wait loop)
#endif
__device__ __forceinline__ void rg_wait_relaxed(uint64_t* b, unsigned parity) {
#if RG_SLEEP > 0
  unsigned ok;
  const unsigned a = smem_u32(b);
  for (;;) {
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(RG_SLEEP);
  }
#else
  rg_wait(b, parity);
#endif
}

// slot sequence numbers: ready[slot] = 1 + index (in the CTA's slice stream) of the slice the
// slot holds.  Written by the producing A warp after its T values (fence + volatile store),
// polled by the B warps with acquire loads (plain LDS in SASS; all L slots of a row in flight
// together; a fence here would wait for the warp's outstanding stores): unlike a phase bit, a sequence number cannot be mistaken for the slot's
// previous use, so a B warp only looks at the slices of the rows it has a block in.
__device__ __forceinline__ int lds_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_volatile(int* p, int v) {
  asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// slot release: the producing A warp arrives on free[slot] with a pending transaction count =
// the number of blocks that will read the slice; every reader takes one off after its t2
// moments (its loads have returned by then); the phase completes when all have, and the slot's
// next producer waits for that phase
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_complete_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.complete_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}

// non-blocking phase test
__device__ __forceinline__ bool rg_test(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

struct RingHdr {
  int64_t src_off;     // source cell (normal window start, first t1 line / t2 slice of the part)
  int64_t dst_off;     // target origin of the face
  int64_t sn, s1, s2;  // signed source strides (reference frame)
  int64_t dn, d1, d2;  // target strides
  int lo1, lo2;        // target index origin of the segment along t1 / t2
  int g1, n1, g2, n2;  // the part's blocks along t1, the face's rows along t2
  int y0, ny, z0, nz;  // source lines / slices of the tile
  int cb, cn;          // the tile's unknowns [cb, cb + cn)
  int narrow;          // every target offset inside the face fits 32 bits
  int snarrow;         // every source offset inside a slice fits 32 bits
  int4 G0;             // the normal group
};

// tile = ((face, t1 part), chunk).  One thread decodes a tile; every field of the face record
// is loaded unconditionally (one global-memory latency instead of decode_face's record ->
// stride -> group chain) and the group table is read from its shared-memory copy.
template <int L>
__device__ __forceinline__ void ring_decode(const DevOp& op, const th_face* __restrict__ faces, int64_t tile,
                                            int ntp, int nch, int u, const int4* sgrp, int4 G0, RingHdr& H) {
  const int64_t st = tile / nch;
  const int c = int(tile - st * nch);
  const int64_t f = st / ntp;
  const int tp = int(st - f * ntp);
  const th_face* const fp = faces + f;
  const int64_t src0 = __ldg(&fp->src[0]), dst0 = __ldg(&fp->dst);
  const int64_t ss0 = __ldg(&fp->src_stride[0]), ss1 = __ldg(&fp->src_stride[1]), ss2 = __ldg(&fp->src_stride[2]);
  const int64_t ds0 = __ldg(&fp->dst_stride[0]), ds1 = __ldg(&fp->dst_stride[1]), ds2 = __ldg(&fp->dst_stride[2]);
  const int n = __ldg(&fp->normal), side = __ldg(&fp->side), seg = __ldg(&fp->segment);
  // reference frame (decode_face, role 0): normal n, tangentials t1 < t2; the normal flip of
  // geometry.py:180-190 folded into the signed strides
  const int64_t ssn = n == 0 ? ss0 : n == 1 ? ss1 : ss2, dsn = n == 0 ? ds0 : n == 1 ? ds1 : ds2;
  H.s1 = n == 0 ? ss1 : ss0;
  H.s2 = n == 2 ? ss1 : ss2;
  H.d1 = n == 0 ? ds1 : ds0;
  H.d2 = n == 2 ? ds1 : ds2;
  H.sn = side ? -ssn : ssn;
  H.dn = side ? -dsn : dsn;
  H.dst_off = dst0 + (side ? int64_t(op.k - 1) * dsn : 0);
  const int c1 = seg % 3, c2 = seg / 3;
  H.lo1 = c1 * op.p;
  H.lo2 = c2 * op.p;
  const int fg1 = op.seg_g[c1][0], fn1 = op.seg_g[c1][1] - fg1;
  const int a1 = tp * fn1 / ntp, b1 = (tp + 1) * fn1 / ntp;
  H.g1 = fg1 + a1;
  H.n1 = b1 - a1;
  H.g2 = op.seg_g[c2][0];
  H.n2 = op.seg_g[c2][1] - H.g2;
  H.cb = int(int64_t(c) * u / nch);
  H.cn = int(int64_t(c + 1) * u / nch) - H.cb;
  if (H.n1 <= 0 || H.n2 <= 0 || H.cn <= 0) {  // empty tile: no slices, no rows
    H.n1 = H.n2 = 0;
    H.y0 = H.z0 = H.ny = H.nz = 0;
    H.cn = 0;
  } else {
    H.y0 = sgrp[H.g1].x;
    H.ny = sgrp[H.g1 + H.n1 - 1].x + L - H.y0;
    H.z0 = sgrp[H.g2].x;
    H.nz = sgrp[H.g2 + H.n2 - 1].x + L - H.z0;
  }
  H.G0 = G0;
  H.src_off = src0 + (side ? int64_t(op.ns0 - 1) * ssn : 0) + int64_t(G0.x) * H.sn + int64_t(H.y0) * H.s1 +
              int64_t(H.z0) * H.s2 + H.cb;
  const int64_t lim = int64_t(1) << 21;
  auto small = [lim](int64_t s) { return s > -lim && s < lim; };
  H.narrow = small(H.dn) && small(H.d1) && small(H.d2) && op.p <= 64 && u <= (1 << 20);
  H.snarrow = small(H.sn) && small(H.s1) && op.p <= 64;
}

// position of an A warp in the CTA's slice stream: slice z of the it-th tile of the CTA
struct RingIt {
  int64_t tile;
  int it;     // tiles of this CTA before `tile`
  int z;      // slice of the tile
  int gz;     // slices of this CTA before the tile
  int slotb;  // ring slot of the tile's slice 0
};

// cp.async copies of slice z of a tile (all its t1 lines) into a staging slot, lanes over unknowns
template <int L>
__device__ __forceinline__ void ring_fetch(const RingHdr& H, const double* __restrict__ src, double* bslot, int bpitch,
                                           int z) {
  const int lane = threadIdx.x & 31;
  if (lane >= H.cn) return;
  const double* const base = src + (H.src_off + lane + int64_t(z) * H.s2);
  double* const bq = bslot + lane * bpitch;
  if (H.snarrow) {  // offsets inside the slice fit 32 bits: one IMAD.WIDE per copy
    const int sn = int(H.sn), s1 = int(H.s1);
#pragma unroll 1
    for (int y = 0; y < H.ny; ++y) {
      const int oy = y * s1;
#pragma unroll
      for (int x = 0; x < L; ++x) cp_async8(bq + L * y + x, base + (oy + x * sn));
    }
  } else {
    const int64_t sn = H.sn, s1 = H.s1;
#pragma unroll 1
    for (int y = 0; y < H.ny; ++y) {
      const double* cell = base + int64_t(y) * s1;
#pragma unroll
      for (int x = 0; x < L; ++x, cell += sn) cp_async8(bq + L * y + x, cell);
    }
  }
}

// L2 prefetch of slice z of a tile: a cell per lane and iteration, the <= 3 lines of its chunk
template <int L>
__device__ __forceinline__ void ring_prefetch(const RingHdr& H, const double* __restrict__ src, int z) {
  const int lane = threadIdx.x & 31;
  const int n = L * H.ny, last = H.cn * 8 - 1;
  const char* const base = reinterpret_cast<const char*>(src + (H.src_off + int64_t(z) * H.s2));
  const bool nar = H.snarrow != 0;
  const int sn32 = int(H.sn), s132 = int(H.s1);
#pragma unroll 1
  for (int c = lane; c < n; c += 32) {
    const int y = c / L, x = c - L * y;
    const char* const pc = nar ? base + int64_t(8) * (x * sn32 + y * s132)
                               : base + 8 * (int64_t(x) * H.sn + int64_t(y) * H.s1);
    l2_prefetch_line(pc);
    l2_prefetch_line(pc + 128);
    l2_prefetch_line(pc + last);
  }
}

// phase A of one slice: normal moments of its NY lines, t1 moments of every window start
template <int L, int D, int NY>
__device__ __forceinline__ void ring_phase_a(const double* bq, double* tq, double& chk) {
  constexpr int NP = D * (D + 1) / 2;
  double mm[NY][D];
#pragma unroll
  for (int y = 0; y < NY; ++y) {
    double v[L];
#pragma unroll
    for (int x = 0; x < L; ++x) v[x] = bq[L * y + x];
    gram_moments<L, D>(v, mm[y]);
    asm volatile("" ::: "memory");  // one line of loads live at a time (register budget)
  }
#pragma unroll
  for (int s = 0; s + L <= NY; ++s) {
    double w[L][D];
#pragma unroll
    for (int y = 0; y < L; ++y)
#pragma unroll
      for (int a = 0; a < D; ++a) w[y][a] = mm[s + y][a];
    double T[NP];
    gram_y<L, D>(w, T);
    // every value of the slice enters some window's T_00 (the windows cover the t1 extent)
    chk = fma(T[0], 0.0, chk);
#pragma unroll
    for (int t = 0; t < NP; t += 2) *reinterpret_cast<double2*>(tq + s * NP + t) = make_double2(T[t], T[t + 1]);
  }
}

// phase A with the slice's lines loaded straight from global memory (no staging slot): all
// loads of the slice are independent, so the compiler issues them ahead of the moments
template <int L, int D, int NY, typename SOFF>
__device__ __forceinline__ void ring_phase_a_direct(const double* __restrict__ base, SOFF sn, SOFF s1, double* tq,
                                                    double& chk) {
  constexpr int NP = D * (D + 1) / 2;
  double mm[NY][D];
  {
    double v[NY][L];
#pragma unroll
    for (int y = 0; y < NY; ++y)
#pragma unroll
      for (int x = 0; x < L; ++x) v[y][x] = __ldg(base + (SOFF(y) * s1 + SOFF(x) * sn));
#pragma unroll
    for (int y = 0; y < NY; ++y) gram_moments<L, D>(v[y], mm[y]);
  }
#pragma unroll
  for (int s = 0; s + L <= NY; ++s) {
    double w[L][D];
#pragma unroll
    for (int y = 0; y < L; ++y)
#pragma unroll
      for (int a = 0; a < D; ++a) w[y][a] = mm[s + y][a];
    double T[NP];
    gram_y<L, D>(w, T);
    chk = fma(T[0], 0.0, chk);
#pragma unroll
    for (int t = 0; t < NP; t += 2) *reinterpret_cast<double2*>(tq + s * NP + t) = make_double2(T[t], T[t + 1]);
  }
}

template <int L, int D, typename SOFF>
__device__ __forceinline__ void ring_phase_a_direct_any(int ny, const double* __restrict__ base, SOFF sn, SOFF s1,
                                                        double* tq, double& chk) {
  if (ny == L) ring_phase_a_direct<L, D, L, SOFF>(base, sn, s1, tq, chk);
  else if (ny == L + 1) ring_phase_a_direct<L, D, L + 1, SOFF>(base, sn, s1, tq, chk);
  else if (ny == L + 2) ring_phase_a_direct<L, D, L + 2, SOFF>(base, sn, s1, tq, chk);
  else if (ny == L + 3) ring_phase_a_direct<L, D, L + 3, SOFF>(base, sn, s1, tq, chk);
}

template <int L, int D>
__device__ __forceinline__ void ring_phase_a_any(int ny, const double* bq, double* tq, double& chk) {
  if (ny == L) ring_phase_a<L, D, L>(bq, tq, chk);
  else if (ny == L + 1) ring_phase_a<L, D, L + 1>(bq, tq, chk);
  else if (ny == L + 2) ring_phase_a<L, D, L + 2>(bq, tq, chk);
  else if (ny == L + 3) ring_phase_a<L, D, L + 3>(bq, tq, chk);
}

// ---- tensor_linear / matrix_linear (ORDER = 1): d-linear 1-D rows in the reference's contraction
// order, normal -> t1 -> t2 (linear.py:115-151; matrix_linear's collapsed operator is the product
// of the same rows, linear.py:202-245).  T is per block of the part (the t1 rows differ per block
// even where the 3-cell windows coincide): T[b1][c0 + 3 c1], 9 values in a slot of 10.

// phase A of one slice: the normal rows of its NY lines, then the t1 rows of every block
template <int NY>
__device__ __forceinline__ void ring_phase_a_tensor(const double* bq, double* tq, double& chk, const T3Syn0& r0,
                                                    const double* stab, const int4* sgrp, int g1, int n1, int y0) {
  double tx[NY][3];
#pragma unroll
  for (int y = 0; y < NY; ++y) {
    double v[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) v[x] = bq[3 * y + x];
#pragma unroll
    for (int c0 = 0; c0 < 3; ++c0) {
      double t = 0.0;
#pragma unroll
      for (int x = 0; x < 3; ++x) t = fma(r0.v[c0 * 4 + x], v[x], t);
      tx[y][c0] = t;
    }
    // finiteness of the inputs: every value of the line enters tx[y][0] .. [2] through a
    // product (0 x Inf and 0 x NaN are NaN), so their sum turns chk NaN for any of them
    chk = fma((tx[y][0] + tx[y][1]) + tx[y][2], 0.0, chk);
  }
#pragma unroll 1
  for (int b = 0; b < n1; ++b) {
    const int s = sgrp[g1 + b].x - y0;
    const double* r1 = stab + (g1 + b) * 12;
    double R1[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) R1[i] = r1[i];
    double T[10];
#pragma unroll
    for (int t = 0; t < 10; ++t) T[t] = 0.0;
#pragma unroll
    for (int S = 0; S + 3 <= NY; ++S) {
      if (s != S) continue;
#pragma unroll
      for (int y = 0; y < 3; ++y)
#pragma unroll
        for (int c0 = 0; c0 < 3; ++c0)
#pragma unroll
          for (int c1 = 0; c1 < 3; ++c1) T[c0 + 3 * c1] = fma(R1[c1 * 3 + y], tx[S + y][c0], T[c0 + 3 * c1]);
    }
#pragma unroll
    for (int t = 0; t < 10; t += 2) *reinterpret_cast<double2*>(tq + b * 10 + t) = make_double2(T[t], T[t + 1]);
  }
}

__device__ __forceinline__ void ring_phase_a_tensor_any(int ny, const double* bq, double* tq, double& chk,
                                                        const T3Syn0& r0, const double* stab, const int4* sgrp, int g1,
                                                        int n1, int y0) {
  if (ny == 3) ring_phase_a_tensor<3>(bq, tq, chk, r0, stab, sgrp, g1, n1, y0);
  else if (ny == 4) ring_phase_a_tensor<4>(bq, tq, chk, r0, stab, sgrp, g1, n1, y0);
  else if (ny == 5) ring_phase_a_tensor<5>(bq, tq, chk, r0, stab, sgrp, g1, n1, y0);
  else if (ny == 6) ring_phase_a_tensor<6>(bq, tq, chk, r0, stab, sgrp, g1, n1, y0);
}

// a block's T values of its 3 slices into registers
__device__ __forceinline__ void ring_tensor_load(const double* tq, const int (&zo)[3], double (&T)[3][10]) {
#pragma unroll
  for (int z = 0; z < 3; ++z)
#pragma unroll
    for (int t = 0; t < 10; t += 2) {
      const double2 v = *reinterpret_cast<const double2*>(tq + zo[z] + t);
      T[z][t] = v.x;
      T[z][t + 1] = v.y;
    }
}

// the t2 rows of the block at its children, stores
template <bool ALL, typename OFF>
__device__ __forceinline__ void ring_tensor_out(const double (&T)[3][10], const double* r2, double* __restrict__ hdst,
                                                OFF qo, OFF d1, OFF d2, const OFF (&do0)[3], const bool (&ok0)[3],
                                                const bool (&ok1)[3], const bool (&ok2)[3]) {
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (!ALL && !ok2[l]) continue;
    double o[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) o[t] = 0.0;
#pragma unroll
    for (int z = 0; z < 3; ++z) {
      const double w = r2[l * 3 + z];
#pragma unroll
      for (int t = 0; t < 9; ++t) o[t] = fma(w, T[z][t], o[t]);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (!ALL && !ok1[j]) continue;
      const OFF oj = qo + OFF(l) * d2 + OFF(j) * d1;
#pragma unroll
      for (int i = 0; i < 3; ++i)
        if (ALL || ok0[i]) *elem(hdst, oj + do0[i]) = o[i + 3 * j];
    }
  }
}

template <typename OFF>
__device__ __forceinline__ void ring_tensor_block(const RingHdr& H, const DevOp& op, double* __restrict__ dst,
                                                  const double (&T)[3][10], const double* stab, int4 G1, int4 G2,
                                                  int g2) {
  const int4 G0 = H.G0;
  bool ok0[3], ok1[3], ok2[3];
  OFF do0[3];
  bool all = true;
  const int p = op.p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int t = G0.z + i;
    ok0[i] = i < G0.w && t >= 0 && t < op.k;
    do0[i] = OFF(t) * OFF(H.dn);
    ok1[i] = i < G1.w && unsigned(G1.z + i - H.lo1) < unsigned(p);
    ok2[i] = i < G2.w && unsigned(G2.z + i - H.lo2) < unsigned(p);
    all &= ok0[i] & ok1[i] & ok2[i];
  }
  const OFF d1 = OFF(H.d1), d2 = OFF(H.d2);
  const int q = threadIdx.x & 31;
  const OFF qo = OFF(G1.z - H.lo1) * d1 + OFF(G2.z - H.lo2) * d2 + OFF(H.cb + q);
  double* const hdst = dst + H.dst_off;
  const double* r2 = stab + g2 * 12;
  if (all) ring_tensor_out<true, OFF>(T, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
  else ring_tensor_out<false, OFF>(T, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
}

// t2 moments of a block: the pairs (a, b) of its window start, L ring slices at zo[]
// (moment index: a-major, then b, then c; D - a - b moments per pair)
template <int L, int D>
__device__ __forceinline__ void ring_moments(const double* tq, const int (&zo)[L], double* M) {
  constexpr int NP = D * (D + 1) / 2;
  static_assert(D == 3 || D == 4, "order2 / order3");
  // pair t = (a, b), a-major: offset of its moments in M and their count D - a - b
  constexpr int MO4[10] = {0, 4, 7, 9, 10, 13, 15, 16, 18, 19}, MN4[10] = {4, 3, 2, 1, 3, 2, 1, 2, 1, 1};
  constexpr int MO3[6] = {0, 3, 5, 6, 8, 9}, MN3[6] = {3, 2, 1, 2, 1, 1};
#pragma unroll
  for (int t = 0; t < NP; t += 2) {
    int mo0, mn0, mo1, mn1;
    if constexpr (D == 4) mo0 = MO4[t], mn0 = MN4[t], mo1 = MO4[t + 1], mn1 = MN4[t + 1];
    else mo0 = MO3[t], mn0 = MN3[t], mo1 = MO3[t + 1], mn1 = MN3[t + 1];
    double ca[L], cb[L];
#pragma unroll
    for (int z = 0; z < L; ++z) {
      const double2 v = *reinterpret_cast<const double2*>(tq + zo[z] + t);
      ca[z] = v.x;
      cb[z] = v.y;
    }
    gram_moments_n<L>(ca, M + mo0, mn0);
    gram_moments_n<L>(cb, M + mo1, mn1);
    asm volatile("" ::: "memory");  // one column pair of loads live at a time
  }
}

// synthesis at the block's children and stores
template <int D, bool ALL, typename OFF>
__device__ __forceinline__ void ring_synth(const double* M, const T3Syn0& s0, const double* r1, const double* r2,
                                           double* __restrict__ hdst, OFF qo, OFF d1, OFF d2, const OFF (&do0)[3],
                                           const bool (&ok0)[3], const bool (&ok1)[3], const bool (&ok2)[3]) {
  constexpr int NP = D * (D + 1) / 2;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (!ALL && !ok2[l]) continue;
    asm volatile("" ::: "memory");  // table values re-read per child (not hoisted into registers)
    double S2[4];
    ld4(r2 + l * 4, S2);
    double Q[NP];
    int t = 0, mi = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b + a < D; ++b, ++t) {
        Q[t] = 0.0;
#pragma unroll
        for (int c = 0; c + b + a < D; ++c, ++mi) Q[t] = fma(S2[c], M[mi], Q[t]);
      }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (!ALL && !ok1[j]) continue;
      asm volatile("" ::: "memory");  // S1 re-read per child
      double S1[4];
      ld4(r1 + j * 4, S1);
      double R[D];
      int tt = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        R[a] = 0.0;
#pragma unroll
        for (int b = 0; b + a < D; ++b, ++tt) R[a] = fma(S1[b], Q[tt], R[a]);
      }
      const OFF oj = qo + OFF(l) * d2 + OFF(j) * d1;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double oi = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) oi = fma(s0.v[i * 4 + a], R[a], oi);  // constant-bank operands
        if (ALL || ok0[i]) *elem(hdst, oj + do0[i]) = oi;
      }
    }
  }
}

// one block of a B warp (lane = unknown): the block's children from its moments M
template <int D, typename OFF>
__device__ __forceinline__ void ring_block(const RingHdr& H, const DevOp& op, double* __restrict__ dst, const double* M,
                                           const double* stab, const T3Syn0& s0, int4 G1, int4 G2, int g1, int g2) {
  const int4 G0 = H.G0;
  bool ok0[3], ok1[3], ok2[3];
  OFF do0[3];
  bool all = true;
  const int p = op.p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int t = G0.z + i;
    ok0[i] = i < G0.w && t >= 0 && t < op.k;
    do0[i] = OFF(t) * OFF(H.dn);
    ok1[i] = i < G1.w && unsigned(G1.z + i - H.lo1) < unsigned(p);
    ok2[i] = i < G2.w && unsigned(G2.z + i - H.lo2) < unsigned(p);
    all &= ok0[i] & ok1[i] & ok2[i];
  }
  const OFF d1 = OFF(H.d1), d2 = OFF(H.d2);
  const int q = threadIdx.x & 31;
  const OFF qo = OFF(G1.z - H.lo1) * d1 + OFF(G2.z - H.lo2) * d2 + OFF(H.cb + q);
  double* const hdst = dst + H.dst_off;
  const double* r1 = stab + g1 * 12;
  const double* r2 = stab + g2 * 12;
  if (all) ring_synth<D, true, OFF>(M, s0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
  else ring_synth<D, false, OFF>(M, s0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2);
}

// dynamic shared memory: sgrp int4[G1] | stab [G1][12] | staging [NA][2][cmax][bpitch] | T ring [R][cmax][tpitch]
__host__ __device__ inline int ring_fixed_doubles(int G1) { return 2 * G1 + ((G1 * 12 + 1) & ~1); }

template <int ORDER>
__global__ void __launch_bounds__(RG_NTH, 1)
    ring_interp_kernel(DevOp op, T3Syn0 syn0, const double* __restrict__ src, double* __restrict__ dst,
                       const th_face* __restrict__ faces, int64_t n_tiles, int ntp, int nch, int cmax, int u, int NA,
                       int R, int bpitch, int tpitch, int32_t* flag) {
  // ORDER 1: tensor_linear / matrix_linear (3-cell windows, T per block); 2 / 3: Gram least squares
  constexpr bool TENSOR = ORDER == 1;
  constexpr int L = ORDER == 3 ? 5 : 3, D = TENSOR ? 3 : ORDER + 1, NP = TENSOR ? 10 : D * (D + 1) / 2;
  constexpr int NM = ORDER == 3 ? 20 : 10;
  extern __shared__ __align__(16) double smem_rg[];
  __shared__ RingHdr Hs[RG_NH];
  __shared__ __align__(8) uint64_t bar_free[RG_RMAX], bar_hdr[RG_NH];
  __shared__ int ready[RG_RMAX];

  const int G1n = op.G1;
  int4* const sgrp = reinterpret_cast<int4*>(smem_rg);
  double* const stab = smem_rg + 2 * G1n;
  const int boxd = (cmax * bpitch + 1) & ~1, trd = cmax * tpitch;
  double* const box0 = smem_rg + ring_fixed_doubles(G1n);
  double* const tr0 = box0 + (RG_DIRECT ? 0 : NA * 2 * boxd);
  const int NB = RG_NW - NA;
  for (int i = threadIdx.x; i < G1n; i += RG_NTH) sgrp[i] = __ldg(&op.grp1[i]);
  if constexpr (TENSOR) {  // t1 / t2 rows [group][child][3] in slots of 12, absent children zero
    for (int i = threadIdx.x; i < G1n * 12; i += RG_NTH) {
      const int g = i / 12, r = i - g * 12, c = r / 3;
      stab[i] = (r < 9 && c < __ldg(&op.grp1[g]).w) ? __ldg(op.rows1 + __ldg(&op.row_off1[g]) + r) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < G1n * 12; i += RG_NTH) stab[i] = __ldg(op.synth1 + i);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < RG_RMAX; ++i) ready[i] = 0;
    for (int i = 0; i < RG_RMAX; ++i) mbar_init(&bar_free[i], 1);
    for (int i = 0; i < RG_NH; ++i) mbar_init(&bar_hdr[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = blockIdx.x, step = gridDim.x;
  const int4 G0c = __ldg(&op.grp0[0]);  // the single normal group (prepare_ring)

  if (warp < NA) {
    // ============ A warps: fetch, phase A of every NA-th slice ============
    // tile headers are decoded RG_HAHEAD tiles ahead, tile i by lane 0 of A warp i mod NA (one
    // warp decoding them all falls a decode -- two dependent global loads -- per tile behind the
    // others, and every block needs slices of every A warp)
    if (lane == 0)
      for (int i = warp; i < RG_HAHEAD; i += NA)
        if (t0 + i * step < n_tiles) {
          ring_decode<L>(op, faces, t0 + i * step, ntp, nch, u, sgrp, G0c, Hs[i]);
          mbar_arrive(&bar_hdr[i]);
        }
    // move an iterator whose z ran past its tile to the tile holding that slice; the leading
    // iterator waits for headers (and decodes its share of them), the others follow it
    auto settle = [&](RingIt& I, bool lead) {
      while (I.tile < n_tiles) {
        const RingHdr& H = Hs[I.it & (RG_NH - 1)];
        if (I.z < H.nz) break;
        I.z -= H.nz;
        I.gz += H.nz;
        I.slotb += H.nz;
        while (I.slotb >= R) I.slotb -= R;  // (a tile may hold more slices than the ring)
        I.tile += step;
        ++I.it;
        if (lead && I.tile < n_tiles) {
          const int64_t nt = I.tile + int64_t(RG_HAHEAD - 1) * step;
          const int ni = I.it + RG_HAHEAD - 1;
          if (lane == 0 && ni % NA == warp && nt < n_tiles) {
            ring_decode<L>(op, faces, nt, ntp, nch, u, sgrp, G0c, Hs[ni & (RG_NH - 1)]);
            mbar_arrive(&bar_hdr[ni & (RG_NH - 1)]);
          }
          __syncwarp();
          rg_wait(&bar_hdr[I.it & (RG_NH - 1)], (I.it / RG_NH) & 1);
        }
      }
    };
    // P: the slice being projected, F: the next own slice (its copies are in flight), G: the own
    // slice RG_PFD ahead of P, whose lines are being pulled into L2
    RingIt G{t0, 0, warp, 0, 0};
    if (t0 < n_tiles) rg_wait(&bar_hdr[0], 0);
    settle(G, true);
    RingIt P = G;
    const bool pf = (op.prefetch & 16) != 0;
    for (int i = 0; i < RG_PFD; ++i) {
      if (pf && i >= (RG_DIRECT ? 1 : 2) && G.tile < n_tiles) ring_prefetch<L>(Hs[G.it & (RG_NH - 1)], src, G.z);
      G.z += NA;
      settle(G, true);
    }
#if !RG_DIRECT
    RingIt F = P;
    F.z += NA;
    settle(F, false);
    double* const mybox = box0 + warp * 2 * boxd;
    if (P.tile < n_tiles) ring_fetch<L>(Hs[P.it & (RG_NH - 1)], src, mybox, bpitch, P.z);
    cp_async_commit();
    if (F.tile < n_tiles) ring_fetch<L>(Hs[F.it & (RG_NH - 1)], src, mybox + boxd, bpitch, F.z);
    cp_async_commit();
#endif
    if (pf && G.tile < n_tiles) ring_prefetch<L>(Hs[G.it & (RG_NH - 1)], src, G.z);
    double chk = 0.0;
    int k = 0, rd = 0, rd_it = -1;
    while (P.tile < n_tiles) {
#if !RG_DIRECT
      cp_async_wait_one();  // this thread's copies of slice P landed
#endif
      const RingHdr& H = Hs[P.it & (RG_NH - 1)];
      int s = P.slotb + P.z;
      while (s >= R) s -= R;
      const int gz = P.gz + P.z;
      // the slot's previous slice (R slices back, the slot's use number gz / R - 1) has been read
      // by every block that needs it
      // (first make sure that slice has been published: its producer may be another, slower A
      //  warp, and a phase wait one phase early would pass)
      if (gz >= R) {
        while (lds_acquire(&ready[s]) != gz - R + 1) __nanosleep(100);
        rg_wait_relaxed(&bar_free[s], (gz / R - 1) & 1);
      }
#if RG_DIRECT
      static_assert(!TENSOR, "RG_DIRECT: Gram schemes only");
      if (lane < H.cn) {
        const double* const base = src + (H.src_off + lane + int64_t(P.z) * H.s2);
        double* const tq = tr0 + s * trd + lane * tpitch;
        if (H.snarrow) ring_phase_a_direct_any<L, D, int>(H.ny, base, int(H.sn), int(H.s1), tq, chk);
        else ring_phase_a_direct_any<L, D, int64_t>(H.ny, base, H.sn, H.s1, tq, chk);
      }
#else
      if (lane < H.cn) {
        const double* const bq = mybox + (k & 1) * boxd + lane * bpitch;
        double* const tq = tr0 + s * trd + lane * tpitch;
        if constexpr (TENSOR) ring_phase_a_tensor_any(H.ny, bq, tq, chk, syn0, stab, sgrp, H.g1, H.n1, H.y0);
        else ring_phase_a_any<L, D>(H.ny, bq, tq, chk);
      }
#endif
      // blocks that will read this slice: the part's blocks in every row whose window holds it
      // (lane z of the warp counts them for slice z once per tile)
      if (P.it != rd_it) {
        rd_it = P.it;
        rd = 0;
        for (int r = 0; r < H.n2; ++r) {
          const int w = sgrp[H.g2 + r].x - H.z0;
          rd += (w <= lane && lane < w + L) ? H.n1 : 0;
        }
      }
      const int readers = __shfl_sync(0xffffffffu, rd, P.z & 31);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect(&bar_free[s], readers);
        __threadfence_block();
        sts_volatile(&ready[s], gz + 1);
      }
#if RG_DIRECT
      P.z += NA;
      settle(P, false);
#else
      P = F;
      F.z += NA;
      settle(F, false);
      if (F.tile < n_tiles) ring_fetch<L>(Hs[F.it & (RG_NH - 1)], src, mybox + (k & 1) * boxd, bpitch, F.z);
      cp_async_commit();
#endif
      G.z += NA;
      settle(G, true);
      if (pf && G.tile < n_tiles) ring_prefetch<L>(Hs[G.it & (RG_NH - 1)], src, G.z);
      ++k;
    }
#if !RG_DIRECT
    cp_async_wait_all();
#endif
    raise_flag(flag, !isfinite(chk));
  } else {
    // ============ B warps: the CTA's blocks round-robin ============
    const int bw = warp - NA;
    int seq = 0, slotb = 0, gzb = 0, it = 0;
    for (int64_t tile = t0; tile < n_tiles; tile += step, ++it) {
      rg_wait(&bar_hdr[it & (RG_NH - 1)], (it / RG_NH) & 1);
      const RingHdr& H = Hs[it & (RG_NH - 1)];
      const int n1 = H.n1, nblk = n1 * H.n2, hg1 = H.g1, hg2 = H.g2, z0 = H.z0, y0 = H.y0;
      const bool active = lane < H.cn;
      int i = bw - seq;
      if (i < 0) i += NB;
      seq += nblk;  // (mod NB by subtraction: nblk <= 28, no integer division)
      while (seq >= NB) seq -= NB;
#pragma unroll 1
      for (; i < nblk; i += NB) {
        // i / n1 for n1 <= 4, i < 32 (n1 = 3: 11 i >> 5 is exact up to i = 31)
        const int r = n1 == 3 ? (i * 11) >> 5 : n1 == 4 ? i >> 2 : n1 == 2 ? i >> 1 : i;
        const int b1 = i - r * n1;
        const int g1 = hg1 + b1, g2 = hg2 + r;
        const int4 G1 = sgrp[g1], G2 = sgrp[g2];
        const int dz = G2.x - z0;
        int zo[L], sl[L];
#pragma unroll
        for (int j = 0; j < L; ++j) {
          int s = slotb + dz + j;
          while (s >= R) s -= R;
          sl[j] = s;
          zo[j] = s * trd;
        }
        // the row's L slices: all polls in flight together
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int j = 0; j < L; ++j) ok &= lds_acquire(&ready[sl[j]]) == gzb + dz + j + 1;
          if (ok) break;
        }
        if constexpr (TENSOR) {
          double T[3][10];
          if (active) ring_tensor_load(tr0 + lane * tpitch + b1 * NP, zo, T);
          __syncwarp();
          if (lane == 0) {  // this block has read its slices
#pragma unroll
            for (int j = 0; j < L; ++j) mbar_complete_tx(&bar_free[sl[j]], 1);
          }
          if (active) {
            if (H.narrow) ring_tensor_block<int>(H, op, dst, T, stab, G1, G2, g2);
            else ring_tensor_block<int64_t>(H, op, dst, T, stab, G1, G2, g2);
          }
        } else {
          double M[NM];
          if (active) ring_moments<L, D>(tr0 + lane * tpitch + (G1.x - y0) * NP, zo, M);
          __syncwarp();
          if (lane == 0) {  // this block has read its slices
#pragma unroll
            for (int j = 0; j < L; ++j) mbar_complete_tx(&bar_free[sl[j]], 1);
          }
          if (active) {
            if (H.narrow) ring_block<D, int>(H, op, dst, M, stab, syn0, G1, G2, g1, g2);
            else ring_block<D, int64_t>(H, op, dst, M, stab, syn0, G1, G2, g1, g2);
          }
        }
      }
      slotb += H.nz;
      while (slotb >= R) slotb -= R;
      gzb += H.nz;
    }
  }
}
