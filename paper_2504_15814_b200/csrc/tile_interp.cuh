// Staged tile interpolation for the 3-cell-window schemes (order2 Gram least
// squares and tensor_linear), included by trihalo.cu after window.cuh (Gram
// helpers) and gram_slide.cuh.
//
// Same arithmetic as gram_slide_kernel<2, 0, ..., TENSOR> (taylor.py:171-219 and
// linear.py:115-151), organised for latency instead of a serial per-warp walk:
//
//  * a CTA owns a tile of the face: up to 3 x 3 coarse blocks (the whole segment at
//    p = 9), whose source support is a box of 3 (normal) x <= 5 x <= 5 coarse cells;
//  * the box of the NEXT tile is copied into shared memory with cp.async while the
//    current one is computed (double buffer, one barrier per tile), so source loads
//    never sit on a thread's critical path;
//  * items = (block, unknown) are flattened with the unknown fastest: every lane is
//    busy (no 32 + 27 split at u = 59) and a warp's stores are contiguous 8-byte runs;
//    each item reads its 27 window values from shared memory at compile-time offsets
//    (box layout [unknown][cell] with an odd pitch: conflict-free 8-byte accesses),
//    does the x / y / z projections and the synthesis at its 27 children in
//    registers, and stores them.
#pragma once

// box geometry: cell (x, y, z) of the tile's support at x + 3 (y + TNY z), TNY = 5
constexpr int TNY = 5;
constexpr int TBOX = 3 * TNY * TNY;  // cells of the largest tile box

struct TileHdr {
  int64_t src_off;       // source cell (normal window start, first t1 / t2 box cell) of the tile
  int64_t dst_off;       // target origin of the face
  int64_t sn, s1, s2;    // signed element strides of the source (reference frame)
  int64_t dn, d1, d2;    // and of the target
  int lo1, lo2;          // target index origin of the segment along t1 / t2
  int g0;                // normal group (one per face)
  int g1, n1, g2, n2;    // the tile's tangential group ranges
  int y0, ny, z0, nz;    // the tile's source box along t1 / t2
  int cnt;               // items x u
  unsigned n1mag;        // 16-bit reciprocal of n1
  int narrow;            // every target offset inside the face fits 32 bits
};

__device__ __forceinline__ unsigned recip16(int d) { return 65536u / unsigned(d) + 1u; }

// a value the compiler must treat as unknown here: keeps per-item address terms out of
// loop-invariant hoisting (27 hoisted 64-bit child offsets per item do not fit in registers)
__device__ __forceinline__ int opaque(int x) {
  asm volatile("" : "+r"(x));
  return x;
}
__device__ __forceinline__ int64_t opaque(int64_t x) {
  asm volatile("" : "+l"(x));
  return x;
}

// &base[i]: one IMAD.WIDE for a 32-bit index (left to itself the compiler widens the index
// sum into 64-bit adds, 4 instructions per store address)
__device__ __forceinline__ double* elem(double* base, int i) {
  double* r;
  asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(r) : "r"(i), "l"(base));
  return r;
}
__device__ __forceinline__ double* elem(double* base, int64_t i) { return base + i; }

__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// one thread: decode tile `tile` of the launch
// (grp: the tangential group table, its shared-memory copy once that is filled)
__device__ __forceinline__ void tile_decode(const DevOp& op, const th_face* __restrict__ faces, int64_t tile, int nt,
                                            int u, TileHdr& H, const int4* grp) {
  const int64_t tpf = int64_t(nt) * nt;
  const int64_t f = tile / tpf;
  const int tt = int(tile - f * tpf);
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
  if (H.n1 <= 0 || H.n2 <= 0) {
    H.n1 = H.n2 = 1;
    H.y0 = H.z0 = 0;
    H.ny = H.nz = 0;
    H.cnt = 0;
  } else {
    H.y0 = grp[H.g1].x;
    H.ny = grp[H.g1 + H.n1 - 1].x + 3 - H.y0;
    H.z0 = grp[H.g2].x;
    H.nz = grp[H.g2 + H.n2 - 1].x + 3 - H.z0;
    H.cnt = H.n1 * H.n2 * u;
  }
  const int4 G0 = __ldg(&op.grp0[fr.g0]);
  H.src_off = fr.src0 + int64_t(G0.x) * fr.sn + int64_t(H.y0) * fr.s1 + int64_t(H.z0) * fr.s2;
  H.n1mag = recip16(H.n1);
  // target offsets inside the face stay below 3 (3 p + 2 k) |stride| + u < 2^31 (p <= 64:
  // extents <= 320 cells per axis); any practical layout has strides far below 2^21 elements
  const int64_t lim = int64_t(1) << 21;
  auto small = [lim](int64_t s) { return s > -lim && s < lim; };
  H.narrow = small(fr.dn) && small(fr.d1) && small(fr.d2) && op.p <= 64 && u <= (1 << 20);
}

// issue the cp.async copies of the tile's source box into box[u][pitch] (warps over cells,
// lanes over unknowns)
template <int NTH>
__device__ __forceinline__ void tile_fetch(const TileHdr& H, const double* __restrict__ src, double* box, int pitch,
                                           int u) {
  constexpr int NW = NTH / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ny = H.ny, nz = H.nz;
  const int64_t sn = H.sn, s1 = H.s1, s2 = H.s2;
  const double* const base = src + H.src_off + lane;
  // rows (y, z) of 3 normal cells: warp w takes rows w, w + NW, ... (ny, nz <= TNY)
  int y = warp, z = 0;
  while (y >= ny && z < nz) y -= ny, ++z;
  for (; z < nz;) {
    const double* row = base + (int64_t(y) * s1 + int64_t(z) * s2);
    double* const drow = box + lane * pitch + 3 * (y + TNY * z);
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const double* cell = row + int64_t(x) * sn;
      for (int q = 0; q + lane < u; q += 32) cp_async8(drow + x + q * pitch, cell + q);
    }
    y += NW;
    while (y >= ny && z < nz) y -= ny, ++z;
  }
}

// L2 prefetch of a tile's source box (the tile after next, so that its cp.async copies one
// iteration later find it in L2): one (cell, 128-byte line) per thread and iteration
template <int NTH>
__device__ __forceinline__ void tile_prefetch_l2(const TileHdr& H, const double* __restrict__ src, int u) {
  const int ny = H.ny, n = 3 * ny * H.nz;
  if (H.cnt <= 0) return;
  const int nl = (u * 8 + 127) / 128 + 1;  // lines a u-double cell can touch (8-byte alignment)
  const int last = u * 8 - 1;
  const char* const base = reinterpret_cast<const char*>(src + H.src_off);
#pragma unroll 1
  for (int c = threadIdx.x; c < n * nl; c += NTH) {
    const int cell = c / nl, part = c - cell * nl;
    const int x = cell % 3, r = cell / 3, z = r / ny, y = r - z * ny;
    const char* const pc = base + 8 * (int64_t(x) * H.sn + int64_t(y) * H.s1 + int64_t(z) * H.s2);
    l2_prefetch_line(pc + min(part * 128, last));
  }
}

// one item: 3 x 3 x 3 window -> 27 children.  ALL: every child is a target (always at p = 9).
template <bool TENSOR, bool ALL, typename OFF>
__device__ __forceinline__ void tile_item(const double* w, const double* r0, const double* r1, const double* r2,
                                          double* __restrict__ hdst, OFF qo, OFF d1, OFF d2, const OFF (&do0)[3],
                                          const bool (&ok0)[3], const bool (&ok1)[3], const bool (&ok2)[3],
                                          double& chk) {
  // w[x + 3 (y + TNY z)]: the window; r0 / r1 / r2: normal / t1 / t2 tables of the item's
  // groups (tensor: 1-D rows [child][3]; Gram: synthesis [child][4])
  constexpr int NT = TENSOR ? 9 : 6;
  double T[3][NT];  // per window slice z: x / y projections
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    double mm[3][3];  // Gram: x moments of the slice's three lines
    if constexpr (TENSOR) {
#pragma unroll
      for (int t = 0; t < NT; ++t) T[z][t] = 0.0;
    }
#pragma unroll
    for (int y = 0; y < 3; ++y) {
      double v[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) v[x] = w[x + 3 * (y + TNY * z)];
      if constexpr (TENSOR) {
#pragma unroll
        for (int c0 = 0; c0 < 3; ++c0) {
          double tx = 0.0;
#pragma unroll
          for (int x = 0; x < 3; ++x) tx = fma(r0[c0 * 3 + x], v[x], tx);
#pragma unroll
          for (int c1 = 0; c1 < 3; ++c1) T[z][c0 + 3 * c1] = fma(r1[c1 * 3 + y], tx, T[z][c0 + 3 * c1]);
        }
      } else {
        gram_moments<3, 3>(v, mm[y]);
      }
    }
    if constexpr (!TENSOR) gram_y<3, 3>(mm, T[z]);  // y moments of the x moments (symmetric sums)
    // finiteness of the inputs: every value of the slice enters T[z][0] (Gram: the plain sum;
    // tensor: an fma chain through all of them), so a NaN / Inf anywhere turns chk NaN
    chk = fma(T[z][0], 0.0, chk);
  }
  if constexpr (TENSOR) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (!ALL && !ok2[l]) continue;
      double o[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) o[t] = 0.0;
#pragma unroll
      for (int z = 0; z < 3; ++z)
#pragma unroll
        for (int t = 0; t < NT; ++t) o[t] = fma(r2[l * 3 + z], T[z][t], o[t]);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (!ALL && !ok1[j]) continue;
        const OFF oj = qo + OFF(l) * d2 + OFF(j) * d1;
#pragma unroll
        for (int i = 0; i < 3; ++i)
          if (ALL || ok0[i]) *elem(hdst, oj + do0[i]) = o[i + 3 * j];
      }
    }
  } else {
    double M[10];
    {
      int t = 0, mi = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b + a < 3; ++b, ++t) {
          double col[3] = {T[0][t], T[1][t], T[2][t]};
          gram_moments_n<3>(col, M + mi, 3 - a - b);
          mi += 3 - a - b;
        }
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (!ALL && !ok2[l]) continue;
      double Q[6];
      int t = 0, mi = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b + a < 3; ++b, ++t) {
          Q[t] = 0.0;
#pragma unroll
          for (int c = 0; c + b + a < 3; ++c, ++mi) Q[t] = fma(r2[l * 4 + c], M[mi], Q[t]);
        }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (!ALL && !ok1[j]) continue;
        double R[3];
        int tt = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          R[a] = 0.0;
#pragma unroll
          for (int b = 0; b + a < 3; ++b, ++tt) R[a] = fma(r1[j * 4 + b], Q[tt], R[a]);
        }
        const OFF oj = qo + OFF(l) * d2 + OFF(j) * d1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double oi = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) oi = fma(r0[i * 4 + a], R[a], oi);
          if (ALL || ok0[i]) *elem(hdst, oj + do0[i]) = oi;
        }
      }
    }
  }
}

template <bool TENSOR, int NTH, typename OFF>
__device__ __forceinline__ void tile_compute(const TileHdr& H, const DevOp& op, double* __restrict__ dst,
                                             const double* box, int pitch, const double* stab, const double* stab0,
                                             const int4* sgrp, int u, unsigned umag, double& chk) {
  constexpr int TW = TENSOR ? 9 : 12;
  const int4 G0 = __ldg(&op.grp0[H.g0]);
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
  const int g0tw = H.g0 * TW;
  const OFF d1 = OFF(H.d1), d2 = OFF(H.d2);
  const int p = op.p, lo1 = H.lo1, lo2 = H.lo2, n1 = H.n1, g1b = H.g1, g2b = H.g2, y0 = H.y0, z0 = H.z0;
  const int cnt = H.cnt;
  const unsigned n1mag = H.n1mag;
  double* const hdst = dst + H.dst_off;
#pragma unroll 1
  for (int idx = threadIdx.x; idx < cnt; idx += NTH) {
    const int blk = u == 1 ? idx : int(__umulhi(unsigned(idx), umag));  // (no 32-bit reciprocal of 1)
    const int q = idx - blk * u;
    const int b2 = int((unsigned(blk) * n1mag) >> 16);
    const int b1 = blk - b2 * n1;
    const int g1 = g1b + b1, g2 = g2b + b2;
    const int4 G1 = sgrp[g1], G2 = sgrp[g2];
    const double* w = box + (q * pitch + 3 * ((G1.x - y0) + TNY * (G2.x - z0)));
    bool ok1[3], ok2[3];
    bool all = all0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      ok1[j] = j < G1.w && unsigned(G1.z + j - lo1) < unsigned(p);
      ok2[j] = j < G2.w && unsigned(G2.z + j - lo2) < unsigned(p);
      all &= ok1[j] & ok2[j];
    }
    const OFF qo = OFF(G1.z - lo1) * d1 + OFF(G2.z - lo2) * d2 + OFF(q);
    const double* r1 = stab + g1 * TW;
    const double* r2 = stab + g2 * TW;
    // (the normal table is tile-uniform: re-read per item rather than hoisted into registers)
    const double* r0 = stab0 + opaque(g0tw);
    if (all) tile_item<TENSOR, true, OFF>(w, r0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2, chk);
    else tile_item<TENSOR, false, OFF>(w, r0, r1, r2, hdst, qo, opaque(d1), opaque(d2), do0, ok0, ok1, ok2, chk);
  }
}

// dynamic shared memory: sgrp int4[G1] | stab [G1][TW] | stab0 [G0][TW] | box[2][u][pitch]
__host__ __device__ inline int tile_box_offset(int TW, int G0, int G1) {
  return 2 * G1 + ((G1 * TW + 1) & ~1) + ((G0 * TW + 1) & ~1);
}

template <bool TENSOR, int NTH, int MINB>
__global__ void __launch_bounds__(NTH, MINB)
    tile_interp_kernel(DevOp op, const double* __restrict__ src, double* __restrict__ dst,
                       const th_face* __restrict__ faces, int64_t n_tiles, int nt, int pitch, int u, unsigned umag,
                       int32_t* flag) {
  constexpr int TW = TENSOR ? 9 : 12;
  extern __shared__ __align__(16) double smem_tile[];
  __shared__ TileHdr Hs[4];  // tiles it (computing), it + 1 (fetching), it + 2 (L2 prefetch), it + 3 (decoding)
  const int G1n = op.G1;
  int4* const sgrp = reinterpret_cast<int4*>(smem_tile);
  double* const stab = smem_tile + 2 * G1n;
  double* const stab0 = stab + ((G1n * TW + 1) & ~1);
  double* const boxes = smem_tile + tile_box_offset(TW, op.G0, G1n);
  const int box_doubles = u * pitch;
  for (int i = threadIdx.x; i < G1n; i += NTH) sgrp[i] = __ldg(&op.grp1[i]);
  if constexpr (TENSOR) {
    for (int i = threadIdx.x; i < G1n * 9; i += NTH) {
      const int g = i / 9, c = (i % 9) / 3, x = i % 3;
      stab[i] = c < __ldg(&op.grp1[g]).w ? __ldg(op.rows1 + __ldg(&op.row_off1[g]) + c * 3 + x) : 0.0;
    }
    for (int i = threadIdx.x; i < op.G0 * 9; i += NTH) {
      const int g = i / 9, c = (i % 9) / 3, x = i % 3;
      stab0[i] = c < __ldg(&op.grp0[g]).w ? __ldg(op.rows0 + __ldg(&op.row_off0[g]) + c * 3 + x) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < G1n * 12; i += NTH) stab[i] = __ldg(op.synth1 + i);
    for (int i = threadIdx.x; i < op.G0 * 12; i += NTH) stab0[i] = __ldg(op.synth0 + i);
  }
  // the decoding thread is the last one: it has the fewest items when a tile does not divide evenly
  constexpr int DEC = NTH - 1;
  const int64_t t0 = blockIdx.x, step = gridDim.x;
  const bool pf = op.prefetch & 16;  // TH_PREFETCH bit 16: L2 prefetch of the tile after next
  __syncthreads();  // tables filled: the decodes read the group table from shared memory
  // the first three headers by three threads of different warps (one latency, not three in a row)
  if ((threadIdx.x & 31) == 31 && threadIdx.x < 96) {
    const int i = threadIdx.x >> 5;
    if (t0 + i * step < n_tiles) tile_decode(op, faces, t0 + i * step, nt, u, Hs[i], sgrp);
  }
  __syncthreads();
  if (t0 < n_tiles) tile_fetch<NTH>(Hs[0], src, boxes, pitch, u);
  cp_async_commit();
  if (pf && t0 + step < n_tiles) tile_prefetch_l2<NTH>(Hs[1], src, u);
  double chk = 0.0;  // fma(T0, 0, chk) stays 0 for finite inputs, turns NaN for any Inf / NaN
  int it = 0;
  for (int64_t tile = t0; tile < n_tiles; tile += step, ++it) {
    cp_async_wait_all();
    __syncthreads();  // this tile's box landed; the previous tile's compute is done with the other box
    if (tile + step < n_tiles) tile_fetch<NTH>(Hs[(it + 1) & 3], src, boxes + ((it + 1) & 1) * box_doubles, pitch, u);
    cp_async_commit();
    if (pf && tile + 2 * step < n_tiles) tile_prefetch_l2<NTH>(Hs[(it + 2) & 3], src, u);
    if (threadIdx.x == DEC && tile + 3 * step < n_tiles) tile_decode(op, faces, tile + 3 * step, nt, u, Hs[(it + 3) & 3], sgrp);
    const TileHdr& H = Hs[it & 3];
    const double* box = boxes + (it & 1) * box_doubles;
    if (H.narrow) tile_compute<TENSOR, NTH, int>(H, op, dst, box, pitch, stab, stab0, sgrp, u, umag, chk);
    else tile_compute<TENSOR, NTH, int64_t>(H, op, dst, box, pitch, stab, stab0, sgrp, u, umag, chk);
  }
  cp_async_wait_all();
  raise_flag(flag, !isfinite(chk));
}
