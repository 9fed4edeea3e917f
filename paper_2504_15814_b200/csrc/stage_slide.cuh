// Slice-staged fixed-window kernels (included by trihalo.cu after gram_slide.cuh):
// order3 restriction, and order2 / order3 / tensor_linear interpolation.
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
//   ROLE 0 (interpolation): t2 windows step by 1, so every slice's x/y moments go
//     into a lane-private ring of L slices in shared memory (as gram_slide.cuh)
//     and each completed block does its z-pass and synthesis from the ring.
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
__device__ __forceinline__ bool tile_of(const DevOp& op, const FaceRef& fr, int ti, int tg, int L, Tile& t) {
  t.gA = fr.g1 + ti * tg;
  t.gB = min(fr.g1 + fr.n1, t.gA + tg);
  if (fr.n0 != 1 || t.gA >= t.gB || fr.n2 < 1) return false;
  t.y0 = __ldg(&op.grp1[t.gA]).x;
  t.ny = __ldg(&op.grp1[t.gB - 1]).x + L - t.y0;
  t.z0 = __ldg(&op.grp1[fr.g2]).x;
  t.z1 = __ldg(&op.grp1[fr.g2 + fr.n2 - 1]).x + L;
  return true;
}

__device__ __forceinline__ int round_even(int v) { return (v + 1) & ~1; }

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Output staging of one interpolation block row (ROLE 0): the region normal children x
// the tile's t1 children x this block's t2 children, laid out in shared memory as the
// contiguous RUNS it forms in the target (the unit-stride axis, merged with the next axes
// while contiguous), each run slot shifted by the run's 8-byte alignment so that its
// 16-byte-aligned interior leaves with one cp.async.bulk store.
struct OutPlan {
  // target cell (a0 + i0, a1 + i1, a2 + i2) of the region lands in run  i . rm  at position
  // pos0 + i . pm  (cells), and run r starts (lowest cell) at element  rs0 + i_outer . st_outer
  int a0, a1, a2;
  int pm0, pm1, pm2, pos0;
  int rm0, rm1, rm2;
  int64_t rsm0, rsm1, rsm2, rs0;
  int n_o0;            // extent of the first outer axis (run-index decode)
  int64_t st_o0, st_o1;
  int R, nruns, rslot;

  __device__ bool make(const int lo[3], const int hi[3], const FaceRef& fr, int u, int out_d) {
    const int lob[3] = {fr.lo0, fr.lo1, fr.lo2};
    const int64_t st[3] = {fr.dn, fr.d1, fr.d2};
    int n[3];
    int64_t base = fr.dst;
    int merged = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      n[d] = hi[d] - lo[d];
      base += int64_t(lo[d] - lob[d]) * st[d];
      if (n[d] == 1) merged |= 1 << d;
    }
    if (n[0] <= 0 || n[1] <= 0 || n[2] <= 0) return false;
    a0 = lo[0], a1 = lo[1], a2 = lo[2];
    int inner = -1;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (inner < 0 && n[d] > 1 && (st[d] == u || st[d] == -u)) inner = d;
    if (inner < 0) return false;
    merged |= 1 << inner;
    int64_t span = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d == inner) span = int64_t(n[d]) * u;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (!(merged >> d & 1) && (st[d] == span || st[d] == -span)) {
          merged |= 1 << d;
          span *= n[d];
        }
    R = int(span / u);
    int pm[3], rm[3];
    int64_t rsm[3];
    pos0 = 0;
    rs0 = base;
    nruns = 1;
    n_o0 = 1;
    st_o0 = st_o1 = 0;
    int nouter = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      pm[d] = 0, rm[d] = 0, rsm[d] = 0;
      if (merged >> d & 1) {
        if (n[d] > 1) {
          const int w = int((st[d] > 0 ? st[d] : -st[d]) / u);
          pm[d] = st[d] > 0 ? w : -w;
          if (st[d] < 0) {
            pos0 += (n[d] - 1) * w;
            rs0 += int64_t(n[d] - 1) * st[d];
          }
        }
      } else {
        rsm[d] = st[d];
        rm[d] = nouter == 0 ? 1 : n_o0;
        if (nouter == 0) {
          n_o0 = n[d];
          st_o0 = st[d];
        } else {
          st_o1 = st[d];
        }
        nruns *= n[d];
        ++nouter;
      }
    }
    pm0 = pm[0], pm1 = pm[1], pm2 = pm[2];
    rm0 = rm[0], rm1 = rm[1], rm2 = rm[2];
    rsm0 = rsm[0], rsm1 = rsm[1], rsm2 = rsm[2];
    rslot = round_even(R * u + 2);
    return R * u * 8 >= 1024 && nruns * rslot <= out_d;
  }
  // shared-memory index (doubles, unknown 0) of target cell (t0, t1, t2)
  __device__ __forceinline__ int index(const double* dst, int t0, int t1, int t2, int u) const {
    const int i0 = t0 - a0, i1 = t1 - a1, i2 = t2 - a2;
    const int r = i0 * rm0 + i1 * rm1 + i2 * rm2;
    const int64_t start = rs0 + i0 * rsm0 + i1 * rsm1 + i2 * rsm2;
    const int sh = int((reinterpret_cast<uintptr_t>(dst + start) & 15) >> 3);
    return r * rslot + sh + (pos0 + i0 * pm0 + i1 * pm1 + i2 * pm2) * u;
  }
  // issue the bulk store of run r (16-byte-aligned interior) and its <= 2 edge doubles
  __device__ void store(double* dst, const double* out, int r, int u) const {
    const int64_t s0 = rs0 + int64_t(r % n_o0) * st_o0 + int64_t(r / n_o0) * st_o1;
    double* g = dst + s0;
    const uintptr_t ga = reinterpret_cast<uintptr_t>(g), gend = ga + uintptr_t(R) * u * 8;
    const uintptr_t lo = (ga + 15) & ~uintptr_t(15), hi = gend & ~uintptr_t(15);
    const double* sm = out + r * rslot + int((ga & 15) >> 3);
    if (hi > lo)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(lo),
                   "r"(smem_u32(sm + (lo - ga) / 8)), "r"(unsigned(hi - lo))
                   : "memory");
    if (lo > ga) g[0] = sm[0];
    if (gend > hi) g[R * u - 1] = sm[R * u - 1];
  }
};

}  // namespace stage

template <int ROLE, int ORDER, bool TENSOR, int NCW, int NST, int NU, int MINB>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB)
    stage_slide_kernel(DevOp op, const double* __restrict__ src, double* __restrict__ dst,
                       const th_face* __restrict__ faces, int64_t n_faces, int u, int32_t* flag, int stage_d,
                       int ny_max, int tg, int tiles_per_face, int out_d) {
  using namespace stage;
  constexpr int L = ORDER == 2 ? 3 : 5;
  constexpr int D = ORDER + 1;
  constexpr int NT = TENSOR ? 9 : (ORDER == 2 ? 6 : 10);  // per-slice values: pairs a + b <= ORDER
  constexpr int NM = ORDER == 2 ? 10 : 20;                // triples a + b + c <= ORDER
  static_assert(ROLE == 0 || (ORDER == 3 && !TENSOR), "restriction: order3 Gram only");
  static_assert(ROLE == 1 || NU == 1, "interpolation: one unknown per lane");
  extern __shared__ __align__(128) double sm[];
  double* const stages = sm;                                                      // [NST][stage_d]
  double* const wtab = sm + NST * stage_d;                  // ROLE 1: [class pair][z][y][a] folded weights
  // ROLE 1: 20 zeros after the table, the weights of a t2 window a slice does not reach
  double* const wzero = wtab + op.st_ncls * op.st_ncls * 100;
  double* const rings = wtab + (ROLE == 1 ? op.st_ncls * op.st_ncls * 100 + 20 : 0);  // ROLE 0: [NCW][L][NT][32]
  double* const outbuf = rings + (ROLE == 0 ? NCW * L * NT * 32 : 0);             // ROLE 0: [out_d] output runs
  int* const hdr = reinterpret_cast<int*>(outbuf + (ROLE == 0 ? out_d : 0));      // [NST][4]
  unsigned* const eline = reinterpret_cast<unsigned*>(hdr + NST * 4);             // [NST][ny_max]
  unsigned char* const shr = reinterpret_cast<unsigned char*>(eline + NST * ny_max);  // producer scratch
  __shared__ __align__(8) uint64_t full[NST], empty[NST];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = op.p, G1 = op.G1;
  const int nch = (u + 32 * NU - 1) / (32 * NU);
  const int64_t total = n_faces * tiles_per_face;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NCW);
    }
    mbar_fence_init();
  }
  if constexpr (ROLE == 1) {
    // W_a(y, z) of every (t1, t2) synthesis-row class pair (host-built, trihalo.cu prepare_stage)
    for (int i = threadIdx.x; i < op.st_ncls * op.st_ncls * 100; i += blockDim.x) wtab[i] = __ldg(op.st_w + i);
    for (int i = threadIdx.x; i < 20; i += blockDim.x) wzero[i] = 0.0;
  }
  __syncthreads();

  if (warp == NCW) {
    // ===================== producer =====================
    int s = 0;
    unsigned ph = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t f = tile / tiles_per_face;
      const th_face* fp = faces + f;
      FaceRef fr;
      decode_face(fp, op, fr);
      Tile t;
      if (!tile_of(op, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const int4 G0 = __ldg(&op.grp0[fr.g0]);
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
    if constexpr (ROLE == 1) {
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
      decode_face(fp, op, fr);
      Tile t;
      if (!tile_of(op, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const bool active = gi < t.gB - t.gA && warp < tg * nch;
      const int g1 = t.gA + (active ? gi : 0);
      const int ly = __ldg(&op.grp1[g1]).x - t.y0;
      const double* const wrow = wtab + __ldg(&op.st_cls[g1]) * ncl * 100;  // + c2 * 100 per window
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
      int wA = __ldg(&op.grp1[0]).x;
      int wB = G1 > 1 ? __ldg(&op.grp1[1]).x : INT_MAX / 2;
      int cA = __ldg(&op.st_cls[0]), cB = G1 > 1 ? __ldg(&op.st_cls[1]) : 0;
      bool bad = false;
      for (int a2 = t.z0; a2 < t.z1; ++a2) {
        const int zA = a2 - wA, zB = a2 - wB;
        const bool inA = zA >= 0 && zA < L, inB = zB >= 0 && zB < L;
        mbar_wait(&full[s], ph);
        if (active) {
          const int* h = hdr + s * 4;
          const int XS = h[0], YS = h[1], BASE = h[2];
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
            double WA[D], WB[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
              WA[i] = wa[y * 4 + i];
              WB[i] = wb[y * 4 + i];
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
          const int t1 = __ldg(&op.grp1[g1]).z, t2 = __ldg(&op.grp1[j]).z;
          if (t1 >= fr.lo1 && t1 < fr.lo1 + p && t2 >= fr.lo2 && t2 < fr.lo2 + p) {
            const int4 G0 = __ldg(&op.grp0[fr.g0]);
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
          wB = j + 1 < G1 ? __ldg(&op.grp1[j + 1]).x : INT_MAX / 2;
          cB = j + 1 < G1 ? __ldg(&op.st_cls[j + 1]) : 0;
        }
      }
      if (active) raise_flag(flag, bad);
    }
    } else {
    // warp w owns t1 group gA + w / nch and unknowns [cb, cb + 32) of the tile
    int s = 0;
    unsigned ph = 0;
    const int gi = warp / nch, chunk = warp - gi * nch;
    double* const ring = rings + warp * (L * NT * 32) + lane;  // [slot][t] x 32 lanes, lane-private
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t f = tile / tiles_per_face;
      const th_face* fp = faces + f;
      FaceRef fr;
      decode_face(fp, op, fr);
      Tile t;
      if (!tile_of(op, fr, int(tile - f * tiles_per_face), tg, L, t)) continue;
      const bool active = gi < t.gB - t.gA;
      const int g1 = t.gA + (active ? gi : 0);
      const int4 G0 = __ldg(&op.grp0[fr.g0]), Gy = __ldg(&op.grp1[g1]);
      const int ly = Gy.x - t.y0;
      const int cb = chunk * 32;
      const bool ok = active && cb + lane < u;
      double R0[TENSOR ? 3 : 1][TENSOR ? L : 1], R1[TENSOR ? 3 : 1][TENSOR ? L : 1];
      if constexpr (TENSOR) {
        const double* r0 = op.rows0 + __ldg(&op.row_off0[fr.g0]);
        const double* r1 = op.rows1 + __ldg(&op.row_off1[g1]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int x = 0; x < L; ++x) {
            R0[c][x] = c < G0.w ? __ldg(r0 + c * L + x) : 0.0;
            R1[c][x] = c < Gy.w ? __ldg(r1 + c * L + x) : 0.0;
          }
      }
      int gz = fr.g2;  // next t2 block to complete
      const int gz_end = fr.g2 + fr.n2;
      int wend = __ldg(&op.grp1[gz]).x + L - 1;
      bool bad = false;
      for (int a2 = t.z0; a2 < t.z1; ++a2) {
        mbar_wait(&full[s], ph);
        if (active) {
          const int* h = hdr + s * 4;
          const int XS = h[0], YS = h[1], BASE = h[2];
          const double* st = stages + size_t(s) * stage_d + BASE + cb + lane;
          const unsigned* el = eline + s * ny_max + ly;
          double T[NT];
#pragma unroll
          for (int i = 0; i < NT; ++i) T[i] = 0.0;
#pragma unroll
          for (int y = 0; y < L; ++y) {
            const unsigned e = el[y];
            const double* ln = st + (ly + y) * YS;
            double v[L];
#pragma unroll
            for (int x = 0; x < L; ++x) v[x] = ok ? ln[x * XS + int((e >> (6 * x)) & 63u)] : 0.0;
            if constexpr (TENSOR) {
#pragma unroll
              for (int c0 = 0; c0 < 3; ++c0) {
                double tx = 0.0;
#pragma unroll
                for (int x = 0; x < L; ++x) tx = fma(R0[c0][x], v[x], tx);
#pragma unroll
                for (int c1 = 0; c1 < 3; ++c1) T[c0 + 3 * c1] = fma(R1[c1][y], tx, T[c0 + 3 * c1]);
              }
            } else {
              double m[D];
              gram_moments<L, D>(v, m);
              int tt = 0;
#pragma unroll
              for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b + a < D; ++b, ++tt) gacc(T[tt], Gram<L>::P(b, y), m[a]);
            }
          }
          double* slot = ring + (a2 % L) * (NT * 32);
#pragma unroll
          for (int i = 0; i < NT; ++i) slot[i * 32] = T[i];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
        // ---- blocks whose window ends at this slice: z-pass + synthesis, store ----
        // (uniform over the consumer warps: all of them take part in the output staging)
        while (gz < gz_end && wend <= a2) {
          const int4 Gz = __ldg(&op.grp1[gz]);
          const int slot0 = Gz.x % L;
          double* const dbase = dst + fr.dst + cb + lane;
          OutPlan pl;
          bool staged = false;
          if (out_d > 0) {
            const int4 Gl = __ldg(&op.grp1[t.gB - 1]), Gf = __ldg(&op.grp1[t.gA]);
            const int lo[3] = {max(G0.z, fr.lo0), max(Gf.z, fr.lo1), max(Gz.z, fr.lo2)};
            const int hi[3] = {min(G0.z + G0.w, fr.hi0), min(Gl.z + Gl.w, fr.lo1 + p), min(Gz.z + Gz.w, fr.lo2 + p)};
            staged = pl.make(lo, hi, fr, u, out_d);
          }
          if (staged) {
            // the previous row's bulk stores have finished reading the buffer
            if (warp == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            named_bar(1, NCW * 32);
          }
          auto emit = [&](int t0, int t1, int t2, double o) {
            if (!ok) return;
            bad |= !isfinite(o);
            if (staged)
              outbuf[pl.index(dst, t0, t1, t2, u) + cb + lane] = o;
            else
              dbase[int64_t(t0 - fr.lo0) * fr.dn + int64_t(t1 - fr.lo1) * fr.d1 + int64_t(t2 - fr.lo2) * fr.d2] = o;
          };
          if (!active) {
          } else if constexpr (TENSOR) {
            const double* r2 = op.rows1 + __ldg(&op.row_off1[gz]);
#pragma unroll
            for (int l = 0; l < 3; ++l) {
              const int tz = Gz.z + l;
              if (!(l < Gz.w && tz >= fr.lo2 && tz < fr.lo2 + p)) continue;
              double o[NT];
#pragma unroll
              for (int i = 0; i < NT; ++i) o[i] = 0.0;
#pragma unroll
              for (int z = 0; z < L; ++z) {
                const double w = ldg_slice(r2 + l * L + z);
                const int sl = slot0 + z >= L ? slot0 + z - L : slot0 + z;
                const double* slot = ring + sl * (NT * 32);
#pragma unroll
                for (int i = 0; i < NT; ++i) o[i] = fma(w, slot[i * 32], o[i]);
              }
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                const int t1 = Gy.z + j;
                if (!(j < Gy.w && t1 >= fr.lo1 && t1 < fr.lo1 + p)) continue;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                  const int t0 = G0.z + i;
                  if (i < G0.w && t0 >= fr.lo0 && t0 < fr.hi0) emit(t0, t1, tz, o[i + 3 * j]);
                }
              }
            }
          } else {
            double M[NM];
#pragma unroll
            for (int i = 0; i < NM; ++i) M[i] = 0.0;
#pragma unroll
            for (int z = 0; z < L; ++z) {
              const int sl = slot0 + z >= L ? slot0 + z - L : slot0 + z;
              const double* slot = ring + sl * (NT * 32);
              int tt = 0, mi = 0;
#pragma unroll
              for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b + a < D; ++b, ++tt) {
                  const double Tz = slot[tt * 32];
#pragma unroll
                  for (int c = 0; c + b + a < D; ++c, ++mi) gacc(M[mi], Gram<L>::P(c, z), Tz);
                }
            }
            const double* s0 = op.synth0 + fr.g0 * 12;
            const double* s1 = op.synth1 + g1 * 12;
            const double* s2 = op.synth1 + gz * 12;
#pragma unroll
            for (int l = 0; l < 3; ++l) {
              const int tz = Gz.z + l;
              if (!(l < Gz.w && tz >= fr.lo2 && tz < fr.lo2 + p)) continue;
              double Q[NT];
              int tt = 0, mi = 0;
#pragma unroll
              for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b + a < D; ++b, ++tt) {
                  Q[tt] = 0.0;
#pragma unroll
                  for (int c = 0; c + b + a < D; ++c, ++mi) Q[tt] = fma(__ldg(s2 + l * 4 + c), M[mi], Q[tt]);
                }
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                const int t1 = Gy.z + j;
                if (!(j < Gy.w && t1 >= fr.lo1 && t1 < fr.lo1 + p)) continue;
                double R[D];
                int t3 = 0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                  R[a] = 0.0;
#pragma unroll
                  for (int b = 0; b + a < D; ++b, ++t3) R[a] = fma(__ldg(s1 + j * 4 + b), Q[t3], R[a]);
                }
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                  const int t0 = G0.z + i;
                  if (!(i < G0.w && t0 >= fr.lo0 && t0 < fr.hi0)) continue;
                  double o = 0.0;
#pragma unroll
                  for (int a = 0; a < D; ++a) o = fma(__ldg(s0 + i * 4 + a), R[a], o);
                  emit(t0, t1, tz, o);
                }
              }
            }
          }
          if (staged) {
            // generic-proxy writes -> visible to the bulk (async-proxy) reads, then one warp stores
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_bar(1, NCW * 32);
            if (warp == 0) {
              for (int r = lane; r < pl.nruns; r += 32) pl.store(dst, outbuf, r, u);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
          ++gz;
          if (gz < gz_end) wend = __ldg(&op.grp1[gz]).x + L - 1;
        }
      }
      if (active) raise_flag(flag, bad);
    }
    if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
}
