// Pipelined restriction (included by trihalo.cu).
//
// Restriction streams ~9x more fine-source bytes than it writes (SURVEY
// §8a A1, 1.15 MB per p=9 face), so the kernel is organised around keeping
// HBM busy: each warp walks a contiguous range of (face, column) work items
// and runs an NST-deep ring of shared-memory slices filled with cp.async
// (8-byte LDGSTS: the unpadded u = 59 AoS cells are only 8-byte aligned, which
// rules out TMA bulk copies).  A slice is one z-plane of a block's window
// (LT x L0 cells x up to 64 unknowns); slice s+NST-1 is issued before slice s
// is consumed, so ~NST-1 slices per warp are always in flight without
// holding registers.  Weights (dense blocks, <= 4 children) sit in shared
// memory and are read as warp-wide broadcasts; 2 unknowns per lane.
//   MODE 1  dense  out[c] = sum_cell W[cell][c] v[cell]          (order2/3, matrix_linear)
//   MODE 2  tensor normal, then t1, then t2 1-D rows              (tensor_linear, linear.py:115-151)
#pragma once

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct ItemRef {  // decoded (face, block) work item of a restriction warp
  FaceRef fr;
  int4 G0, G1, G2;
  int g0, g1, g2;
  bool valid;
};

__device__ __forceinline__ void decode_restrict_item(const DevOp& op, const th_face* __restrict__ faces,
                                                     int64_t item, ItemRef& r) {
  const int64_t f = item / op.max_items;
  const int it = int(item - f * op.max_items);
  decode_face(faces + f, op, r.fr);
  r.valid = decode_item(op, r.fr, it, r.g0, r.g1, r.g2);
  if (r.valid) {
    r.G0 = __ldg(&op.grp0[r.g0]);
    r.G1 = __ldg(&op.grp1[r.g1]);
    r.G2 = __ldg(&op.grp1[r.g2]);
  }
}

template <int MODE, int L0, int LT, int NST, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) restrict_pipe_kernel(DevOp op, const double* __restrict__ src,
                                                                   double* __restrict__ dst,
                                                                   const th_face* __restrict__ faces,
                                                                   int64_t n_faces, int u, int32_t* flag) {
  constexpr int SL = L0 * LT;     // cells per slice
  constexpr int S = L0 * LT * LT;  // cells per window
  constexpr int C0 = 3;            // normal children (k = 3), t1 / t2 children 1
  extern __shared__ double4 smem4[];
  double4* sw4 = smem4;                                             // dense weights [blk][cell] (MODE 1)
  const int n_w4 = MODE == 1 ? op.n_blocks * S : 0;
  double* ring = reinterpret_cast<double*>(smem4 + n_w4);           // [WARPS][NST][SL][64]
  if constexpr (MODE == 1) {
    const double4* gw = reinterpret_cast<const double4*>(op.weights);
    for (int i = threadIdx.x; i < n_w4; i += blockDim.x) sw4[i] = gw[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my_ring = ring + size_t(warp) * NST * SL * 64;
  // contiguous range of (face, block) items for this warp
  const int64_t total = n_faces * op.max_items;
  const int64_t nw = int64_t(gridDim.x) * WARPS;
  const int64_t gw_id = int64_t(blockIdx.x) * WARPS + warp;
  const int64_t per = (total + nw - 1) / nw;
  const int64_t i_begin = min(total, gw_id * per), i_end = min(total, i_begin + per);
  const int n_chunks = (u + 63) / 64;
  // slice counter space: (item, chunk, z)
  const int64_t n_slices = (i_end - i_begin) * n_chunks * LT;

  ItemRef iss, con;  // issue-side and consume-side decoded items
  int64_t iss_item = -1, con_item = -1;

  auto issue = [&](int64_t s) {
    if (s < n_slices) {
      const int64_t ic = s / LT;
      const int z = int(s - ic * LT);
      const int64_t item = i_begin + ic / n_chunks;
      const int cb = int(ic % n_chunks) * 64;
      if (item != iss_item) {
        decode_restrict_item(op, faces, item, iss);
        iss_item = item;
      }
      if (iss.valid) {
        double* slot = my_ring + size_t(s % NST) * SL * 64;
        const th_face* fp = faces + item / op.max_items;
        const int a2 = iss.G2.x + z;
        const int b2 = (a2 >= op.p) + (a2 >= 2 * op.p);
        const int64_t adj = iss.fr.src0 - __ldg(&fp->src[0]);
        const int64_t zo = int64_t(a2 - b2 * op.p) * iss.fr.s2 + adj + cb + lane;
        const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
#pragma unroll
        for (int y = 0; y < LT; ++y) {
          const int a1 = iss.G1.x + y;
          const int b1 = (a1 >= op.p) + (a1 >= 2 * op.p);
          const int64_t row = __ldg(&fp->src[b1 + 3 * b2]) + zo + int64_t(a1 - b1 * op.p) * iss.fr.s1 +
                              int64_t(iss.G0.x) * iss.fr.sn;
#pragma unroll
          for (int x = 0; x < L0; ++x) {
            const double* g = src + row + int64_t(x) * iss.fr.sn;
            double* d = slot + (y * L0 + x) * 64 + lane;
            if (ok0) cp_async8(d, g);
            if (ok1) cp_async8(d + 32, g + 32);
          }
        }
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < NST - 1; ++s) issue(s);

  double acc[C0][2];
  double T[C0][2];
  double R0[C0][L0], R1[LT], R2[LT];
  for (int64_t s = 0; s < n_slices; ++s) {
    issue(s + NST - 1);
    cp_async_wait<NST - 1>();
    __syncwarp();
    const int64_t ic = s / LT;
    const int z = int(s - ic * LT);
    const int64_t item = i_begin + ic / n_chunks;
    const int cb = int(ic % n_chunks) * 64;
    if (item != con_item) {
      decode_restrict_item(op, faces, item, con);
      con_item = item;
      if (MODE == 2 && con.valid) {
        const double* r0 = op.rows0 + __ldg(&op.row_off0[con.g0]);
        const double* r1 = op.rows1 + __ldg(&op.row_off1[con.g1]);
        const double* r2 = op.rows1 + __ldg(&op.row_off1[con.g2]);
#pragma unroll
        for (int c = 0; c < C0; ++c)
#pragma unroll
          for (int x = 0; x < L0; ++x) R0[c][x] = c < con.G0.w ? __ldg(r0 + c * L0 + x) : 0.0;
#pragma unroll
        for (int y = 0; y < LT; ++y) {
          R1[y] = __ldg(r1 + y);
          R2[y] = __ldg(r2 + y);
        }
      }
    }
    if (con.valid) {
      if (z == 0) {
#pragma unroll
        for (int c = 0; c < C0; ++c) acc[c][0] = acc[c][1] = 0.0;
      }
      const double* slot = my_ring + size_t(s % NST) * SL * 64 + lane;
      if constexpr (MODE == 1) {
        const int bid = __ldg(&op.block_id[(con.g0 * op.G1 + con.g1) * op.G1 + con.g2]);
        const double4* Ws = sw4 + bid * S + z * SL;
#pragma unroll
        for (int c = 0; c < SL; ++c) {
          const double v0 = slot[c * 64], v1 = slot[c * 64 + 32];
          const double4 w = Ws[c];
          acc[0][0] = fma(w.x, v0, acc[0][0]);
          acc[0][1] = fma(w.x, v1, acc[0][1]);
          acc[1][0] = fma(w.y, v0, acc[1][0]);
          acc[1][1] = fma(w.y, v1, acc[1][1]);
          acc[2][0] = fma(w.z, v0, acc[2][0]);
          acc[2][1] = fma(w.z, v1, acc[2][1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < C0; ++c) T[c][0] = T[c][1] = 0.0;
#pragma unroll
        for (int y = 0; y < LT; ++y)
#pragma unroll
          for (int c = 0; c < C0; ++c) {
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int x = 0; x < L0; ++x) {
              t0 = fma(R0[c][x], slot[(y * L0 + x) * 64], t0);
              t1 = fma(R0[c][x], slot[(y * L0 + x) * 64 + 32], t1);
            }
            T[c][0] = fma(R1[y], t0, T[c][0]);
            T[c][1] = fma(R1[y], t1, T[c][1]);
          }
        double r2 = 0.0;
#pragma unroll
        for (int zz = 0; zz < LT; ++zz)
          if (zz == z) r2 = R2[zz];
#pragma unroll
        for (int c = 0; c < C0; ++c) {
          acc[c][0] = fma(r2, T[c][0], acc[c][0]);
          acc[c][1] = fma(r2, T[c][1], acc[c][1]);
        }
      }
      if (z == LT - 1) {  // window complete: store the children inside the face's box
        const FaceRef& fr = con.fr;
        const int t1 = con.G1.z, t2 = con.G2.z;
        bool bad = false;
        if (t1 >= fr.lo1 && t1 < fr.lo1 + op.p && t2 >= fr.lo2 && t2 < fr.lo2 + op.p) {
          double* base = dst + fr.dst + (t1 - fr.lo1) * fr.d1 + (t2 - fr.lo2) * fr.d2 + cb + lane;
          const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
#pragma unroll
          for (int c = 0; c < C0; ++c) {
            const int t0 = con.G0.z + c;
            if (c < con.G0.w && t0 >= fr.lo0 && t0 < fr.hi0) {
              double* dp = base + (t0 - fr.lo0) * fr.dn;
              if (ok0) { dp[0] = acc[c][0]; bad |= !isfinite(acc[c][0]); }
              if (ok1) { dp[32] = acc[c][1]; bad |= !isfinite(acc[c][1]); }
            }
          }
        }
        raise_flag(flag, bad);
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}
