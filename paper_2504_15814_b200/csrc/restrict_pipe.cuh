// Pipelined restriction (included by trihalo.cu).
//
// Restriction streams ~9x more fine-source bytes than it writes (SURVEY
// §8a A1, 1.15 MB per p=9 face), so the kernel is organised around keeping
// HBM busy: each warp walks a contiguous range of (face, column) work items
// and runs an NST-deep ring of shared-memory slices filled with cp.async
// (8-byte LDGSTS: the unpadded u = 59 AoS cells are only 8-byte aligned, which
// rules out TMA bulk copies).  A slice is one z-plane of a block's window
// (LT x L0 cells x up to 64 unknowns); slice s+NST-1 is issued before slice s
// is consumed, so NST-1 slices per warp are in flight without holding
// registers.  Address work is hoisted: faces are decoded only when the face
// changes (the nine fine-block bases go to a per-warp shared cache), per-face
// normal offsets and per-item row offsets are precomputed, so one cp.async
// pair costs one 64-bit add.  Dense weights (<= 4 children) sit in shared
// memory and are read as broadcasts; 2 unknowns per lane.
//   MODE 1  dense  out[c] = sum_cell W[cell][c] v[cell]          (order2/3, matrix_linear)
//   MODE 2  tensor normal, then t1, then t2 1-D rows              (tensor_linear, linear.py:115-151)
#pragma once

__device__ __forceinline__ void cp_async8(unsigned smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_dst), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int MODE, int L0, int LT, int NST, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) restrict_pipe_kernel(DevOp op, const double* __restrict__ src,
                                                                   double* __restrict__ dst,
                                                                   const th_face* __restrict__ faces,
                                                                   int64_t n_faces, int u, int32_t* flag) {
  constexpr int SL = L0 * LT;      // cells per slice
  constexpr int S = L0 * LT * LT;  // cells per window
  constexpr int C0 = 3;            // normal children (k = 3); t1 / t2 children 1
  constexpr int SLOT = SL * 64;    // doubles per ring slot
  extern __shared__ double4 smem4[];
  __shared__ int64_t face_base[WARPS][9];
  double4* sw4 = smem4;  // dense weights [blk][cell] (MODE 1)
  const int n_w4 = MODE == 1 ? op.n_blocks * S : 0;
  double* ring = reinterpret_cast<double*>(smem4 + n_w4);
  if constexpr (MODE == 1) {
    const double4* gw = reinterpret_cast<const double4*>(op.weights);
    for (int i = threadIdx.x; i < n_w4; i += blockDim.x) sw4[i] = gw[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my_ring = ring + size_t(warp) * NST * SLOT;
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(my_ring)) + lane * 8u;
  const int64_t total = n_faces * op.max_items;
  const int64_t nw = int64_t(gridDim.x) * WARPS;
  const int64_t gid = int64_t(blockIdx.x) * WARPS + warp;
  const int64_t per = (total + nw - 1) / nw;
  const int64_t i_begin = min(total, gid * per), i_end = min(total, i_begin + per);
  const int n_chunks = (u + 63) / 64;
  const int64_t n_slices = (i_end - i_begin) * n_chunks * LT;
  const int p = op.p;

  // ---- issuer state --------------------------------------------------------
  int64_t i_face = -1, i_item = -1;
  FaceRef ifr;
  int64_t ixo[L0], iyo[LT];
  int iyb[LT];
  int4 iG2;
  bool i_valid = false;
  // ---- consumer state ------------------------------------------------------
  int64_t c_face = -1, c_item = -1;
  FaceRef cfr;
  int4 cG0, cG1, cG2;
  int cg0 = 0, cg1 = 0, cg2 = 0;
  bool c_valid = false;

  auto issue = [&](int64_t s) {
    if (s < n_slices) {
      const int64_t ic = s / LT;
      const int z = int(s - ic * LT);
      const int64_t item = i_begin + ic / n_chunks;
      const int cb = int(ic - (ic / n_chunks) * n_chunks) * 64;
      if (item != i_item) {
        i_item = item;
        const int64_t f = item / op.max_items;
        if (f != i_face) {
          i_face = f;
          decode_face(faces + f, op, ifr);
          const int64_t adj = ifr.src0 - __ldg(&faces[f].src[0]);
          __syncwarp();
          if (lane < 9) face_base[warp][lane] = __ldg(&faces[f].src[lane]) + adj;
          __syncwarp();
#pragma unroll
          for (int x = 0; x < L0; ++x) ixo[x] = int64_t(x) * ifr.sn;
        }
        int g0, g1, g2;
        i_valid = decode_item(op, ifr, int(item - f * op.max_items), g0, g1, g2);
        if (i_valid) {
          const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]);
          iG2 = __ldg(&op.grp1[g2]);
#pragma unroll
          for (int y = 0; y < LT; ++y) {
            const int a1 = G1.x + y;
            iyb[y] = (a1 >= p) + (a1 >= 2 * p);
            iyo[y] = int64_t(a1 - iyb[y] * p) * ifr.s1 + int64_t(G0.x) * ifr.sn;
          }
        }
      }
      if (i_valid) {
        const int a2 = iG2.x + z;
        const int b2 = (a2 >= p) + (a2 >= 2 * p);
        const int64_t zo = int64_t(a2 - b2 * p) * ifr.s2 + cb + lane;
        const unsigned slot = ring_s + unsigned((s % NST) * SLOT) * 8u;
        const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
#pragma unroll
        for (int y = 0; y < LT; ++y) {
          const double* row = src + (face_base[warp][iyb[y] + 3 * b2] + iyo[y] + zo);
#pragma unroll
          for (int x = 0; x < L0; ++x) {
            const double* g = row + ixo[x];
            const unsigned d = slot + unsigned((y * L0 + x) * 64 * 8);
            if (ok0) cp_async8(d, g);
            if (ok1) cp_async8(d + 256u, g + 32);
          }
        }
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < NST - 1; ++s) issue(s);

  double acc[C0][2];
  double R0[MODE == 2 ? C0 : 1][MODE == 2 ? L0 : 1], R1[MODE == 2 ? LT : 1], R2[MODE == 2 ? LT : 1];
  const double4* Ws = sw4;
  int64_t obase = 0;
  bool store_ok = false;
  for (int64_t s = 0; s < n_slices; ++s) {
    issue(s + NST - 1);
    const int64_t ic = s / LT;
    const int z = int(s - ic * LT);
    const int64_t item = i_begin + ic / n_chunks;
    const int cb = int(ic - (ic / n_chunks) * n_chunks) * 64;
    if (item != c_item) {
      c_item = item;
      const int64_t f = item / op.max_items;
      if (f != c_face) {
        c_face = f;
        decode_face(faces + f, op, cfr);
      }
      c_valid = decode_item(op, cfr, int(item - f * op.max_items), cg0, cg1, cg2);
      if (c_valid) {
        cG0 = __ldg(&op.grp0[cg0]);
        cG1 = __ldg(&op.grp1[cg1]);
        cG2 = __ldg(&op.grp1[cg2]);
        if constexpr (MODE == 1) {
          Ws = sw4 + __ldg(&op.block_id[(cg0 * op.G1 + cg1) * op.G1 + cg2]) * S;
        } else {
          const double* r0 = op.rows0 + __ldg(&op.row_off0[cg0]);
          const double* r1 = op.rows1 + __ldg(&op.row_off1[cg1]);
          const double* r2 = op.rows1 + __ldg(&op.row_off1[cg2]);
#pragma unroll
          for (int c = 0; c < C0; ++c)
#pragma unroll
            for (int x = 0; x < L0; ++x) R0[c][x] = c < cG0.w ? __ldg(r0 + c * L0 + x) : 0.0;
#pragma unroll
          for (int y = 0; y < LT; ++y) {
            R1[y] = __ldg(r1 + y);
            R2[y] = __ldg(r2 + y);
          }
        }
        const int t1 = cG1.z, t2 = cG2.z;
        store_ok = t1 >= cfr.lo1 && t1 < cfr.lo1 + p && t2 >= cfr.lo2 && t2 < cfr.lo2 + p;
        obase = cfr.dst + (t1 - cfr.lo1) * cfr.d1 + (t2 - cfr.lo2) * cfr.d2 + lane;
      }
    }
    cp_async_wait<NST - 1>();
    __syncwarp();
    if (c_valid) {
      if (z == 0) {
#pragma unroll
        for (int c = 0; c < C0; ++c) acc[c][0] = acc[c][1] = 0.0;
      }
      const double* slot = my_ring + size_t(s % NST) * SLOT + lane;
      if constexpr (MODE == 1) {
        const double4* W = Ws + z * SL;
#pragma unroll
        for (int c = 0; c < SL; ++c) {
          const double v0 = slot[c * 64], v1 = slot[c * 64 + 32];
          const double4 w = W[c];
          acc[0][0] = fma(w.x, v0, acc[0][0]);
          acc[0][1] = fma(w.x, v1, acc[0][1]);
          acc[1][0] = fma(w.y, v0, acc[1][0]);
          acc[1][1] = fma(w.y, v1, acc[1][1]);
          acc[2][0] = fma(w.z, v0, acc[2][0]);
          acc[2][1] = fma(w.z, v1, acc[2][1]);
        }
      } else {
        double T[C0][2];
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
        double r2 = R2[0];
#pragma unroll
        for (int zz = 1; zz < LT; ++zz)
          if (zz == z) r2 = R2[zz];
#pragma unroll
        for (int c = 0; c < C0; ++c) {
          acc[c][0] = fma(r2, T[c][0], acc[c][0]);
          acc[c][1] = fma(r2, T[c][1], acc[c][1]);
        }
      }
      if (z == LT - 1) {  // window complete: store the children inside the face's box
        bool bad = false;
        if (store_ok) {
          const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
#pragma unroll
          for (int c = 0; c < C0; ++c) {
            const int t0 = cG0.z + c;
            if (c < cG0.w && t0 >= cfr.lo0 && t0 < cfr.hi0) {
              double* dp = dst + obase + cb + (t0 - cfr.lo0) * cfr.dn;
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
