// Slice-staged order3 restriction (included by trihalo.cu after gram_slide.cuh).
//
// What they compute is gram_slide.cuh's: the reference's least-squares rows
// (taylor.py:171-219) as the Gram-separable projection onto total degree <=
// ORDER, or the d-linear 1-D rows contracted normal, t1, t2 (linear.py:115-151),
// swept along t2 one source slice at a time.  What changes is who loads:
//
// The per-warp slide is latency-bound -- each warp has one window slice of
// loads in flight and 12-16 warps fit per SM (0.28-0.59 of HBM).  Here one CTA
// owns a (face, tile of t1 groups) and a PRODUCER warp streams the tile's
// source slices -- planes of NX (normal) x NY (t1 range) cells -- into an
// NST-stage shared-memory ring with 1-D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx): whole planes in flight per SM without registers, and
// the t1-overlapping windows of the tile's CONSUMER warps read them from
// shared memory instead of L2.
//
// Consumers (one per t1 group x 32-unknown chunk of the tile):
//   ROLE 1 (restriction, ORDER 3): t2 windows step by 3 and overlap by <= 2, so
//     a slice feeds at most two coarse columns and the z-pass and t2 synthesis
//     fold into one 1-D row per degree,
//       Q_ab(j) = sum_z K_{a+b}(j, z) T_ab(w_j + z),  K_d(j, z) = sum_{c <= 3-d} S2_j[c] P_c(z),
//       out_i   = sum_a S0_i[a] sum_b S1[b] Q_ab,
//     the two open windows' Q living in registers (NU = 2 unknowns per lane).
//   OWN (u <= 64, tiles of <= NCW - 1 groups, 3-stage ring + hand-over slots fit: p <= 16): the
//     t1 windows are 5 lines long and step by 3, so one warp per t1 group projects 2 of every 3
//     lines twice.  The line-owner consumers project every line once: warp i owns the lines
//     [w_i, w_{i+1}) (<= 3 per slice), accumulates them into its own group's windows and -- where a
//     line also lies in window i - 1 -- into a partial it keeps for the previous group, handed over
//     through a shared-memory slot when a t2 window completes (config 5: 0.85 -> 0.925 of the copy
//     peak; profiles/r02_ab_restriction.txt, entries 10-11).
//   (An interpolation consumer on the same producer -- ROLE 0, with TMA bulk stores of the
//   output -- measured no faster than the per-warp slide and was removed in round 2;
//   profiles/r01_ab_stage.txt.)
//
// Bulk copies need 16-byte alignment; unpadded cells (u = 59: 472 B) are only
// 8-byte aligned, and one copy per cell is op-rate bound (2.0 TB/s measured,
// tools/probe/probe_stage.cu).  So the producer copies contiguous RUNS of
// cells, widened to 16-byte boundaries (<= 8 extra bytes per end, inside the
// allocation's 16-byte granules):
//   mode 0  |sn| == u : one run per t1 line along the normal (NX cells)
//   mode 1  s1 == u   : one run per (normal position, fine block) along t1
//   mode 2  otherwise : one copy per cell (correct, slow; not used by the
//                       standard slab / pool layouts)
// Cell (x, y) of a stage then sits at  BASE + y*YS + x*XS + e(x, y)  doubles,
// e = the run's 8-byte shift plus the per-run slack, 6-bit fields of a per-line
// word written by the producer.
#pragma once

namespace stage {

struct Tile {
  int gA, gB, y0, ny, z0, z1;
};

// tile ti of a face: t1 groups [gA, gB) of the face's range, their window union
// [y0, y0 + ny) along t1 and the union [z0, z1) of all its t2 windows
// (grp: the tangential group table, its shared-memory copy in the kernel)
__device__ __forceinline__ bool tile_of(const int4* grp, const FaceRef& fr, int ti, int tg, int L, Tile& t) {
  t.gA = fr.g1 + ti * tg;
  t.gB = min(fr.g1 + fr.n1, t.gA + tg);
  if (fr.n0 != 1 || t.gA >= t.gB || fr.n2 < 1) return false;
  t.y0 = grp[t.gA].x;
  t.ny = grp[t.gB - 1].x + L - t.y0;
  t.z0 = grp[fr.g2].x;
  t.z1 = grp[fr.g2 + fr.n2 - 1].x + L;
  return true;
}

constexpr int kGrpSmem = 96;  // tangential groups copied to shared memory (3 p <= 96)

__device__ __forceinline__ int round_even(int v) { return (v + 1) & ~1; }

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace stage

template <int ROLE, int ORDER, bool TENSOR, int NCW, int NST, int NU, int MINB, bool OWN = false>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB)
    stage_slide_kernel(DevOp op, const double* __restrict__ src, double* __restrict__ dst,
                       const th_face* __restrict__ faces, int64_t n_faces, int u, int32_t* flag, int stage_d,
                       int ny_max, int tg, int tiles_per_face, int out_d) {
  using namespace stage;
  constexpr int L = ORDER == 2 ? 3 : 5;
  constexpr int D = ORDER + 1;
  static_assert(ROLE == 1 && ORDER == 3 && !TENSOR, "restriction, order3 Gram only");
  extern __shared__ __align__(128) double sm[];
  double* const stages = sm;                                                      // [NST][stage_d]
  double* const wtab = sm + NST * stage_d;                  // ROLE 1: [class pair][z][y][a] folded weights
  // ROLE 1: 20 zeros after the table, the weights of a t2 window a slice does not reach
  double* const wzero = wtab + op.st_ncls * op.st_ncls * 100;
  // OWN: hand-over slots of the line-owner consumers, [NCW - 1][NU][D][32] (see below)
  constexpr int XSLOT = NU * (ORDER + 1) * 32;
  double* const xch = wzero + 20;
  int* const hdr = reinterpret_cast<int*>(xch + (OWN ? (NCW - 1) * XSLOT : 0));     // [NST][4]
  unsigned* const eline = reinterpret_cast<unsigned*>(hdr + NST * 4);             // [NST][ny_max]
  unsigned char* const shr = reinterpret_cast<unsigned char*>(eline + NST * ny_max);  // producer scratch
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  __shared__ __align__(8) uint64_t xfull[OWN ? NCW : 1], xempty[OWN ? NCW : 1];
  // group table and synthesis-row classes in shared memory: a tile's header (face record ->
  // groups -> classes) then costs one global-memory latency instead of a chain of four, which
  // every consumer warp used to wait out at the start of each tile while the ring stood full
  __shared__ int4 sgrp_s[kGrpSmem];
  __shared__ int scls_s[kGrpSmem];
  __shared__ double s0_s[OWN ? 12 * 8 : 1];  // OWN: normal synthesis rows of up to 8 normal groups
  const bool s0sm = OWN && op.G0 <= 8;
  const bool gsm = op.G1 <= kGrpSmem;
  const int4* const grp = gsm ? sgrp_s : op.grp1;
  const int* const cls = gsm ? scls_s : op.st_cls;
  const int4 G0c = __ldg(&op.grp0[0]);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = op.p, G1 = op.G1;
  const int nch = (u + 32 * NU - 1) / (32 * NU);
  const int64_t total = n_faces * tiles_per_face;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NCW);
    }
    if constexpr (OWN)
      for (int i = 0; i < NCW; ++i) {
        mbar_init(&xfull[i], 1);
        mbar_init(&xempty[i], 1);
      }
    mbar_fence_init();
  }
  if constexpr (ROLE == 1) {
    // W_a(y, z) of every (t1, t2) synthesis-row class pair (host-built, trihalo.cu prepare_stage)
    for (int i = threadIdx.x; i < op.st_ncls * op.st_ncls * 100; i += blockDim.x) wtab[i] = __ldg(op.st_w + i);
    for (int i = threadIdx.x; i < 20; i += blockDim.x) wzero[i] = 0.0;
    if (s0sm)
      for (int i = threadIdx.x; i < op.G0 * 12; i += blockDim.x) s0_s[i] = __ldg(op.synth0 + i);
    if (gsm)
      for (int i = threadIdx.x; i < op.G1; i += blockDim.x) {
        sgrp_s[i] = __ldg(&op.grp1[i]);
        scls_s[i] = __ldg(&op.st_cls[i]);
      }
  }
  __syncthreads();

  if (warp == NCW) {
    // ===================== producer =====================
    int s = 0;
    unsigned ph = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t f = tile / tiles_per_face;
      const th_face* fp = faces + f;
      if (tile + gridDim.x < total && lane < 2)  // the next tile's face record (144 bytes) into L2
        l2_prefetch_line(reinterpret_cast<const char*>(faces + (tile + gridDim.x) / tiles_per_face) + 128 * lane);
      FaceRef fr;
      decode_face_restrict(fp, op, fr);
      Tile t;
      if (!tile_of(grp, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const int4 G0 = fr.g0 == 0 ? G0c : __ldg(&op.grp0[fr.g0]);
      const int nx = G0.y, x0 = G0.x;
      const int64_t adj = fr.src0 - __ldg(&fp->src[0]);
      const int mode = (fr.sn == u || fr.sn == -u) ? 0 : (fr.s1 == u ? 1 : 2);
      const int bfirst = t.y0 / p, nseg = (t.y0 + t.ny - 1) / p - bfirst + 1;
      const int nruns = mode == 0 ? t.ny : mode == 1 ? nx * nseg : nx * t.ny;
      // per-mode strides (doubles); mode 1's XS = sum over segments of the run slots
      int XS, YS, BASE = 0;
      if (mode == 0) {
        YS = round_even(nx * u + 2);
        XS = fr.sn > 0 ? u : -u;
        BASE = fr.sn > 0 ? 0 : (nx - 1) * u;
      } else if (mode == 1) {
        YS = u;
        XS = 0;
        for (int sg = 0; sg < nseg; ++sg) {
          const int ys = max(t.y0, (bfirst + sg) * p), ye = min(t.y0 + t.ny, (bfirst + sg + 1) * p);
          XS += round_even((ye - ys) * u + 2);
        }
      } else {
        YS = round_even(u + 2);
        XS = t.ny * YS;
      }
      // ---- per-tile run descriptors (modes 0 / 1: <= 2 runs and <= 2 lines per lane) ----
      // run r = lane + 32 k starts at  block base(b1, b2) + roff + zo(a2)  and lands at
      // stage + rdst; only the block base and zo change from slice to slice
      const bool fast = mode != 2 && nruns <= 64 && t.ny <= 64;
      int rb1[2], rdst[2];
      int64_t roff[2];
      unsigned rlen[2];
      int lsg[2], leb[2];  // mode 1 lines y = lane + 32 k: segment, per-tile part of e
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = lane + 32 * k;
        rb1[k] = 0, rdst[k] = 0, roff[k] = 0, rlen[k] = 0, lsg[k] = 0, leb[k] = 0;
        if (!fast) continue;
        if (r < nruns) {
          int x, ya, n, d;
          if (mode == 0) {
            x = fr.sn > 0 ? 0 : nx - 1;
            ya = t.y0 + r;
            n = nx;
            d = r * YS;
          } else {
            x = r / nseg;
            const int sg = r - x * nseg;
            ya = max(t.y0, (bfirst + sg) * p);
            n = min(t.y0 + t.ny, (bfirst + sg + 1) * p) - ya;
            int off = 0;
            for (int q = 0; q < sg; ++q) {
              const int ys = max(t.y0, (bfirst + q) * p), ye = min(t.y0 + t.ny, (bfirst + q + 1) * p);
              off += round_even((ye - ys) * u + 2);
            }
            d = x * XS + off;
          }
          rb1[k] = ya / p;
          roff[k] = int64_t(ya - rb1[k] * p) * fr.s1 + int64_t(x0 + x) * fr.sn + adj;
          rdst[k] = d;
          rlen[k] = unsigned(n) * unsigned(u) * 8u;
        }
        const int y = r;
        if (mode == 1 && y < t.ny) {
          const int sg = (t.y0 + y) / p - bfirst;
          int off = 0;
          for (int q = 0; q < sg; ++q) {
            const int ys = max(t.y0, (bfirst + q) * p), ye = min(t.y0 + t.ny, (bfirst + q + 1) * p);
            off += round_even((ye - ys) * u + 2);
          }
          lsg[k] = sg;
          leb[k] = off - (max(t.y0, (bfirst + sg) * p) - t.y0) * u;
        }
      }
      int64_t rbb[2] = {0, 0};
      int b2prev = -1;
      for (int a2 = t.z0; a2 < t.z1; ++a2) {
        mbar_wait(&empty[s], ph ^ 1);
        const int b2 = a2 / p;
        const int64_t zo = int64_t(a2 - b2 * p) * fr.s2;
        double* const st = stages + size_t(s) * stage_d;
        if (fast) {
          if (b2 != b2prev) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
              if (lane + 32 * k < nruns) rbb[k] = __ldg(&fp->src[rb1[k] + 3 * b2]);
            b2prev = b2;
          }
          uintptr_t lo[2];
          unsigned nb[2], sh[2];
          unsigned bytes = 0;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const uintptr_t ga = reinterpret_cast<uintptr_t>(src + (rbb[k] + roff[k] + zo));
            lo[k] = ga & ~uintptr_t(15);
            nb[k] = unsigned(((ga + rlen[k] + 15) & ~uintptr_t(15)) - lo[k]);
            sh[k] = unsigned(ga - lo[k]) >> 3;
            if (lane + 32 * k < nruns) {
              bytes += nb[k];
              if (mode == 1) shr[lane + 32 * k] = (unsigned char)sh[k];
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
          if (lane == 0) {
            mbar_expect_tx(&full[s], bytes);
            int* h = hdr + s * 4;
            h[0] = XS;
            h[1] = YS;
            h[2] = BASE;
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (lane + 32 * k < nruns) bulk_g2s(st + rdst[k], reinterpret_cast<const void*>(lo[k]), nb[k], &full[s]);
          // per-line shift words e(x, y), 6-bit fields
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int y = lane + 32 * k;
            if (y >= t.ny) continue;
            unsigned w;
            if (mode == 0) {
              w = sh[k] * 0x1041041u;  // the line's one run: same shift for every x
            } else {
              w = 0;
              for (int x = 0; x < nx; ++x) w |= unsigned(leb[k] + shr[x * nseg + lsg[k]]) << (6 * x);
            }
            eline[s * ny_max + y] = w;
          }
        } else {
          // mode 2 (no contiguous axis): one copy per cell, all recomputed per slice
          const int64_t zoa = zo + adj;
          unsigned bytes = 0;
          for (int r = lane; r < nruns; r += 32) {
            const int x = r / t.ny, ya = t.y0 + (r - x * t.ny), b1 = ya / p;
            const uintptr_t ga = reinterpret_cast<uintptr_t>(
                src + (__ldg(&fp->src[b1 + 3 * b2]) + int64_t(ya - b1 * p) * fr.s1 + zoa + int64_t(x0 + x) * fr.sn));
            const uintptr_t lo = ga & ~uintptr_t(15);
            bytes += unsigned(((ga + uintptr_t(u) * 8 + 15) & ~uintptr_t(15)) - lo);
            shr[r] = (unsigned char)((ga - lo) >> 3);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
          if (lane == 0) {
            mbar_expect_tx(&full[s], bytes);
            int* h = hdr + s * 4;
            h[0] = XS;
            h[1] = YS;
            h[2] = BASE;
          }
          __syncwarp();
          for (int r = lane; r < nruns; r += 32) {
            const int x = r / t.ny, ya = t.y0 + (r - x * t.ny), b1 = ya / p;
            const uintptr_t ga = reinterpret_cast<uintptr_t>(
                src + (__ldg(&fp->src[b1 + 3 * b2]) + int64_t(ya - b1 * p) * fr.s1 + zoa + int64_t(x0 + x) * fr.sn));
            const uintptr_t lo = ga & ~uintptr_t(15);
            bulk_g2s(st + x * XS + (ya - t.y0) * YS, reinterpret_cast<const void*>(lo),
                     unsigned(((ga + uintptr_t(u) * 8 + 15) & ~uintptr_t(15)) - lo), &full[s]);
          }
          for (int y = lane; y < t.ny; y += 32) {
            unsigned w = 0;
            for (int x = 0; x < nx; ++x) w |= unsigned(shr[x * t.ny + y]) << (6 * x);
            eline[s * ny_max + y] = w;
          }
        }
        __syncwarp();  // shr reads above precede the next stage's writes
        mbar_arrive(&full[s]);
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ===================== consumers =====================
    if constexpr (ROLE == 1 && OWN) {
    // LINE-OWNER consumers (u <= 64, tiles of <= NCW - 1 groups).  t1 windows step by 3 and are 5
    // lines long, so with one warp per t1 group every warp projects 5 lines per slice and 2 of
    // every 3 lines are projected twice.  Here every line of the slice has ONE owner: warp i < ng
    // owns the lines [w_i, w_{i+1}) -- the lines group i shares with group i - 1 plus its own --
    // (the last group: its first 3 lines; warp ng, the helper, its last 2): <= 3 lines per warp
    // and slice.  A line's normal moments feed the owner's OWN group (window i) and, where the
    // line also lies in window i - 1, the partial sums it keeps for the PREVIOUS group.  When a
    // t2 window completes, warp i hands its partial of group i - 1 to warp i - 1 through a
    // shared-memory slot (full / empty mbarriers per slot, one writer and one reader warp each;
    // partials are written before the own group's are awaited, so the chain resolves from the
    // helper down) and warp i - 1 adds it to its own before the normal synthesis.
    // U_a += W_a m_a for the line's four folded weights (two 16-byte broadcast loads; the tables sit
    // on 32-byte boundaries); windows the slice does not reach are skipped (warp-uniform)
    auto accumulate = [](const double* w, const double (&m)[NU][D], double (&U)[NU][D]) {
      const double2 w0 = *reinterpret_cast<const double2*>(w), w1 = *reinterpret_cast<const double2*>(w + 2);
      const double W[D] = {w0.x, w0.y, w1.x, w1.y};
#pragma unroll
      for (int q = 0; q < NU; ++q)
#pragma unroll
        for (int a = 0; a < D; ++a) U[q][a] = fma(W[a], m[q][a], U[q][a]);
    };
    int s = 0;
    unsigned ph = 0, xin = 0, xout = 0;
    const int ncl = op.st_ncls;
    const int i = warp;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t f = tile / tiles_per_face;
      const th_face* fp = faces + f;
      FaceRef fr;
      decode_face_restrict(fp, op, fr);
      Tile t;
      if (!tile_of(grp, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const int ng = t.gB - t.gA;
      const bool active = i <= ng, hasOwn = i < ng, hasPrev = active && i >= 1;
      const int gO = t.gA + (hasOwn ? i : ng - 1), gP = t.gA + (hasPrev ? i - 1 : 0);
      const int wO = grp[gO].x, wP = grp[gP].x, wl = grp[t.gB - 1].x;
      const int la = i < ng ? wO : wl + 3;
      const int lb = i < ng - 1 ? grp[gO + 1].x : i == ng - 1 ? wl + 3 : wl + L;
      const int nl = active ? lb - la : 0;  // <= 3 (stage_geometry)
      const int ly = la - t.y0;
      bool ownS[3], prevS[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        ownS[k] = hasOwn && la + k < wO + L;
        prevS[k] = hasPrev && la + k < wP + L;
      }
      const int yo = (la - wO) * 4, yp = (la - wP) * 4;  // first line's row in the own / previous window
      const double* const wrowO = wtab + cls[gO] * ncl * 100;
      const double* const wrowP = wtab + cls[gP] * ncl * 100;
      bool ok[NU];
#pragma unroll
      for (int q = 0; q < NU; ++q) ok[q] = hasOwn && lane + 32 * q < u;
      double UA[NU][D], UB[NU][D], PA[NU][D], PB[NU][D];
#pragma unroll
      for (int q = 0; q < NU; ++q)
#pragma unroll
        for (int a = 0; a < D; ++a) UA[q][a] = UB[q][a] = PA[q][a] = PB[q][a] = 0.0;
      int j = 0;
      int wA = grp[0].x;
      int wB = G1 > 1 ? grp[1].x : INT_MAX / 2;
      int cA = cls[0], cB = G1 > 1 ? cls[1] : 0;
      bool bad = false;
      for (int a2 = t.z0; a2 < t.z1; ++a2) {
        const int zA = a2 - wA, zB = a2 - wB;
        const bool inA = zA >= 0 && zA < L, inB = zB >= 0 && zB < L;
        mbar_wait(&full[s], ph);
        if (nl > 0) {
          const int4 h = *reinterpret_cast<const int4*>(hdr + s * 4);
          const int XS = h.x, YS = h.y, BASE = h.z;
          const double* st = stages + size_t(s) * stage_d + BASE + lane;
          const unsigned* el = eline + s * ny_max + ly;
          const int oA = cA * 100 + zA * 20, oB = cB * 100 + zB * 20;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (k >= nl) break;
            const unsigned e = el[k];
            const double* ln = st + (ly + k) * YS;
            double m[NU][D];
#pragma unroll
            for (int q = 0; q < NU; ++q) {
              double v[L];
#pragma unroll
              for (int x = 0; x < L; ++x) v[x] = ln[x * XS + int((e >> (6 * x)) & 63u) + 32 * q];
              gram_moments<L, D>(v, m[q]);
            }
            static_assert(D == 4, "order3: four degrees");
            if (ownS[k]) {
              if (inA) accumulate(wrowO + oA + yo + k * 4, m, UA);
              if (inB) accumulate(wrowO + oB + yo + k * 4, m, UB);
            }
            if (prevS[k]) {
              if (inA) accumulate(wrowP + oA + yp + k * 4, m, PA);
              if (inB) accumulate(wrowP + oB + yp + k * 4, m, PB);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
        if (!active) continue;
        if (zA == L - 1) {
          // ---- window j complete ----
          if (hasPrev) {  // the partial of group i - 1 to its warp
            double* xs = xch + (i - 1) * XSLOT + lane;
            mbar_wait(&xempty[i - 1], xout ^ 1);
#pragma unroll
            for (int q = 0; q < NU; ++q)
#pragma unroll
              for (int a = 0; a < D; ++a) xs[(q * D + a) * 32] = PA[q][a];
            __syncwarp();
            if (lane == 0) mbar_arrive(&xfull[i - 1]);
            xout ^= 1;
          }
          if (hasOwn) {
            const double* xs = xch + i * XSLOT + lane;
            mbar_wait(&xfull[i], xin);
#pragma unroll
            for (int q = 0; q < NU; ++q)
#pragma unroll
              for (int a = 0; a < D; ++a) UA[q][a] += xs[(q * D + a) * 32];
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[i]);
            xin ^= 1;
            // its normal children, store
            const int t1 = grp[gO].z, t2 = grp[j].z;
            if (t1 >= fr.lo1 && t1 < fr.lo1 + p && t2 >= fr.lo2 && t2 < fr.lo2 + p) {
              const int4 G0 = fr.g0 == 0 ? G0c : __ldg(&op.grp0[fr.g0]);
              const double* s0 = (s0sm ? s0_s : op.synth0) + fr.g0 * 12;
              double* const ob = dst + fr.dst + int64_t(t1 - fr.lo1) * fr.d1 + int64_t(t2 - fr.lo2) * fr.d2 + lane;
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const int t0 = G0.z + c;
                if (c < G0.w && t0 >= fr.lo0 && t0 < fr.hi0) {
                  double S0[D];
#pragma unroll
                  for (int a = 0; a < D; ++a) S0[a] = s0[c * 4 + a];
#pragma unroll
                  for (int q = 0; q < NU; ++q) {
                    double o = 0.0;
#pragma unroll
                    for (int a = 0; a < D; ++a) o = fma(S0[a], UA[q][a], o);
                    if (ok[q]) {
                      ob[int64_t(t0 - fr.lo0) * fr.dn + 32 * q] = o;
                      bad |= !isfinite(o);
                    }
                  }
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < NU; ++q)
#pragma unroll
            for (int a = 0; a < D; ++a) {
              UA[q][a] = UB[q][a];
              UB[q][a] = 0.0;
              PA[q][a] = PB[q][a];
              PB[q][a] = 0.0;
            }
          ++j;
          wA = wB;
          cA = cB;
          wB = j + 1 < G1 ? grp[j + 1].x : INT_MAX / 2;
          cB = j + 1 < G1 ? cls[j + 1] : 0;
        }
      }
      if (hasOwn) raise_flag(flag, bad);
    }
    } else if constexpr (ROLE == 1) {
    // warp w owns t1 group gA + w / nch and unknowns [cb, cb + 32 NU) of the tile;
    // lane q-th unknown = cb + lane + 32 q.  Per slice and t1 line: the normal Gram moments
    // m_a (gram_moments), then U_a += W_a(y, z) m_a for the <= 2 open t2 windows (A = j,
    // B = j + 1); a window is complete after its 5th slice: out_i = sum_a S0_i[a] U_a.
    int s = 0;
    unsigned ph = 0;
    const int gi = warp / nch, chunk = warp - gi * nch;
    const int ncl = op.st_ncls;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t f = tile / tiles_per_face;
      const th_face* fp = faces + f;
      FaceRef fr;
      decode_face_restrict(fp, op, fr);
      Tile t;
      if (!tile_of(grp, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const bool active = gi < t.gB - t.gA && warp < tg * nch;
      const int g1 = t.gA + (active ? gi : 0);
      const int ly = grp[g1].x - t.y0;
      const double* const wrow = wtab + cls[g1] * ncl * 100;  // + c2 * 100 per window
      const int cb = chunk * 32 * NU;
      bool ok[NU];
#pragma unroll
      for (int q = 0; q < NU; ++q) ok[q] = active && cb + lane + 32 * q < u;
      double UA[NU][D], UB[NU][D];
#pragma unroll
      for (int q = 0; q < NU; ++q)
#pragma unroll
        for (int i = 0; i < D; ++i) UA[q][i] = UB[q][i] = 0.0;
      int j = 0;
      int wA = grp[0].x;
      int wB = G1 > 1 ? grp[1].x : INT_MAX / 2;
      int cA = cls[0], cB = G1 > 1 ? cls[1] : 0;
      bool bad = false;
      for (int a2 = t.z0; a2 < t.z1; ++a2) {
        const int zA = a2 - wA, zB = a2 - wB;
        const bool inA = zA >= 0 && zA < L, inB = zB >= 0 && zB < L;
        mbar_wait(&full[s], ph);
#ifdef TH_AB_NOCOMPUTE  // diagnosis build: the producer's stream alone (consumers only hand slices back)
        if (false) {
#else
        if (active) {
#endif
          const int4 h = *reinterpret_cast<const int4*>(hdr + s * 4);  // (16-byte aligned: one load)
          const int XS = h.x, YS = h.y, BASE = h.z;
          const double* st = stages + size_t(s) * stage_d + BASE + cb + lane;
          const unsigned* el = eline + s * ny_max + ly;
          // a window the slice does not reach reads the zero block; lanes past u read whatever
          // follows their cell in the stage (finite or not: those results are never stored or
          // checked, and the reads stay inside the shared allocation)
          const double* wa = inA ? wrow + cA * 100 + zA * 20 : wzero;
          const double* wb = inB ? wrow + cB * 100 + zB * 20 : wzero;
#pragma unroll
          for (int y = 0; y < L; ++y) {
            const unsigned e = el[y];
            const double* ln = st + (ly + y) * YS;
            // the line's 4 + 4 folded weights through four 16-byte broadcast loads (the tables sit on
            // 32-byte boundaries: stage_d is even and every table offset a multiple of 4 doubles)
            double WA[D], WB[D];
            static_assert(D == 4, "order3: four degrees");
            {
              const double2 a0 = *reinterpret_cast<const double2*>(wa + y * 4),
                            a1 = *reinterpret_cast<const double2*>(wa + y * 4 + 2),
                            b0 = *reinterpret_cast<const double2*>(wb + y * 4),
                            b1 = *reinterpret_cast<const double2*>(wb + y * 4 + 2);
              WA[0] = a0.x, WA[1] = a0.y, WA[2] = a1.x, WA[3] = a1.y;
              WB[0] = b0.x, WB[1] = b0.y, WB[2] = b1.x, WB[3] = b1.y;
            }
#pragma unroll
            for (int q = 0; q < NU; ++q) {
              double v[L], m[D];
#pragma unroll
              for (int x = 0; x < L; ++x) v[x] = ln[x * XS + int((e >> (6 * x)) & 63u) + 32 * q];
              gram_moments<L, D>(v, m);
#pragma unroll
              for (int i = 0; i < D; ++i) {
                UA[q][i] = fma(WA[i], m[i], UA[q][i]);
                UB[q][i] = fma(WB[i], m[i], UB[q][i]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
        if (!active) continue;
        if (zA == L - 1) {
          // ---- window j complete: its normal children, store ----
          const int t1 = grp[g1].z, t2 = grp[j].z;
          if (t1 >= fr.lo1 && t1 < fr.lo1 + p && t2 >= fr.lo2 && t2 < fr.lo2 + p) {
            const int4 G0 = fr.g0 == 0 ? G0c : __ldg(&op.grp0[fr.g0]);
            const double* s0 = op.synth0 + fr.g0 * 12;
            double* const ob = dst + fr.dst + int64_t(t1 - fr.lo1) * fr.d1 + int64_t(t2 - fr.lo2) * fr.d2 + cb + lane;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const int t0 = G0.z + i;
              if (i < G0.w && t0 >= fr.lo0 && t0 < fr.hi0) {
                double S0[D];
#pragma unroll
                for (int a = 0; a < D; ++a) S0[a] = __ldg(s0 + i * 4 + a);
#pragma unroll
                for (int q = 0; q < NU; ++q) {
                  double o = 0.0;
#pragma unroll
                  for (int a = 0; a < D; ++a) o = fma(S0[a], UA[q][a], o);
                  if (ok[q]) {
                    ob[int64_t(t0 - fr.lo0) * fr.dn + 32 * q] = o;
                    bad |= !isfinite(o);
                  }
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < NU; ++q)
#pragma unroll
            for (int i = 0; i < D; ++i) {
              UA[q][i] = UB[q][i];
              UB[q][i] = 0.0;
            }
          ++j;
          wA = wB;
          cA = cB;
          wB = j + 1 < G1 ? grp[j + 1].x : INT_MAX / 2;
          cB = j + 1 < G1 ? cls[j + 1] : 0;
        }
      }
      if (active) raise_flag(flag, bad);
    }
    }
  }
}
