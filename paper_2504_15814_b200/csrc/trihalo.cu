// B200 (sm_100a) kernels and the C ABI of include/trihalo_b200.h.
//
// Data model: AoS cells (u unknowns contiguous, the reference HaloBuffer
// layout, geometry.py:272-303) addressed through per-face offsets/strides.
// Each warp owns one (face, block) work item: a block is the tensor product
// of one normal group and two tangential groups of the operator (see
// builder.hpp) — a source window of <= 5x5x5 cells feeding <= 27 target
// cells.  Lanes run over unknowns (lane, lane+32), so every weight is
// warp-uniform (one broadcast load feeds 2 unknowns x 2 children) and every
// source/target cell access is a contiguous 8*u-byte run (coalesced for all
// six face orientations; the orientation only changes strides).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/trihalo_b200.h"
#include "builder.hpp"

namespace {

thread_local std::string g_last_error;
thread_local int g_last_column = -1;

int32_t fail(int32_t code, const std::string& msg, int col = -1) {
  g_last_error = msg;
  g_last_column = col;
  return code;
}

#define TH_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return fail(TH_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// device view of an operator (passed by value)
// ---------------------------------------------------------------------------
struct DevOp {
  int32_t role, scheme, p, k;
  int32_t prefetch;    // L2 bulk prefetch of block windows (TH_PREFETCH=0 disables; tuning)
  int32_t ns0;         // source extent along the normal (2k)
  int32_t G0, G1;      // groups along normal / tangential
  int32_t max_items;   // work items per face (upper bound)
  const int4* grp0;    // (win0, winL, tgt0, tgtN)
  const int4* grp1;
  const int32_t* block_id;
  const int64_t* block_off;
  const int32_t* block_cp;
  const double* weights;
  const int64_t* row_off0;  // 1-D rows (tensor_linear)
  const double* rows0;
  const int64_t* row_off1;
  const double* rows1;
  const double* synth0;     // Gram synthesis tables [group][3][4]
  const double* synth1;
  int32_t n_blocks;
  int32_t units_per_face;   // (normal group, t1 group) columns per face, fixed-window kernels
  int32_t ns_t;             // source extent along a tangential axis
  int32_t seg_g[3][2];
  int32_t half_g[3][2];
  int32_t half_t[3][2];
  // staged order3 restriction (stage_slide.cuh): synthesis-row class of every tangential
  // group and the folded tangential weights W[c1][c2][z][y][a] of every class pair
  const int32_t* st_cls;
  const double* st_w;
  int32_t st_ncls;
};

// one face, rewritten in reference-frame terms: source cell (a0, a1, a2) of
// block b lives at src[b] + a0*sn + (a1 - b1*p)*s1 + (a2 - b2*p)*s2 and target
// cell (t0, t1, t2) at dst + (t0-lo0)*dn + (t1-lo1)*d1 + (t2-lo2)*d2; the
// normal flip of geometry.py:180-190 is folded into the signed strides.
struct FaceRef {
  int64_t src0;   // block 0 (interpolation)
  int64_t sn, s1, s2;
  int64_t dst, dn, d1, d2;
  int lo0, lo1, lo2, hi0;
  int g0, n0, g1, n1, g2, n2;
};

// Every field of the record is loaded unconditionally and the axis-dependent ones selected
// afterwards: one global-memory latency per decode (loading normal / side first and then the
// strides they select is a chain of dependent loads, which the persistent tile kernels -- one
// decoding thread per tile, whose warp the others wait for -- and the per-warp restriction
// kernel had on their critical paths; profiles/r02_ab_ring.txt).
// interpolation faces (role 0):
__device__ __forceinline__ void decode_face_interp(const th_face* __restrict__ fp, const DevOp& op, FaceRef& r) {
  const int64_t src0 = __ldg(&fp->src[0]), dst0 = __ldg(&fp->dst);
  const int64_t ss0 = __ldg(&fp->src_stride[0]), ss1 = __ldg(&fp->src_stride[1]), ss2 = __ldg(&fp->src_stride[2]);
  const int64_t ds0 = __ldg(&fp->dst_stride[0]), ds1 = __ldg(&fp->dst_stride[1]), ds2 = __ldg(&fp->dst_stride[2]);
  const int n = __ldg(&fp->normal), side = __ldg(&fp->side), s = __ldg(&fp->segment);
  const int64_t ssn = n == 0 ? ss0 : n == 1 ? ss1 : ss2, dsn = n == 0 ? ds0 : n == 1 ? ds1 : ds2;
  r.s1 = n == 0 ? ss1 : ss0;
  r.s2 = n == 2 ? ss1 : ss2;
  r.d1 = n == 0 ? ds1 : ds0;
  r.d2 = n == 2 ? ds1 : ds2;
  r.sn = side ? -ssn : ssn;
  r.dn = side ? -dsn : dsn;
  r.src0 = src0 + (side ? int64_t(op.ns0 - 1) * ssn : 0);
  r.dst = dst0 + (side ? int64_t(op.k - 1) * dsn : 0);
  r.lo0 = 0;
  r.hi0 = op.k;
  r.lo1 = (s % 3) * op.p;
  r.lo2 = (s / 3) * op.p;
  r.g0 = 0;
  r.n0 = op.G0;
  r.g1 = op.seg_g[s % 3][0];
  r.n1 = op.seg_g[s % 3][1] - r.g1;
  r.g2 = op.seg_g[s / 3][0];
  r.n2 = op.seg_g[s / 3][1] - r.g2;
}

// decode_face for restriction faces (role 1), every field loaded unconditionally (one latency)
__device__ __forceinline__ void decode_face_restrict(const th_face* __restrict__ fp, const DevOp& op, FaceRef& r) {
  const int64_t src0 = __ldg(&fp->src[0]), dst0 = __ldg(&fp->dst);
  const int64_t ss0 = __ldg(&fp->src_stride[0]), ss1 = __ldg(&fp->src_stride[1]), ss2 = __ldg(&fp->src_stride[2]);
  const int64_t ds0 = __ldg(&fp->dst_stride[0]), ds1 = __ldg(&fp->dst_stride[1]), ds2 = __ldg(&fp->dst_stride[2]);
  const int n = __ldg(&fp->normal), side = __ldg(&fp->side), h = __ldg(&fp->half);
  const int64_t ssn = n == 0 ? ss0 : n == 1 ? ss1 : ss2, dsn = n == 0 ? ds0 : n == 1 ? ds1 : ds2;
  r.s1 = n == 0 ? ss1 : ss0;
  r.s2 = n == 2 ? ss1 : ss2;
  r.d1 = n == 0 ? ds1 : ds0;
  r.d2 = n == 2 ? ds1 : ds2;
  r.sn = side ? -ssn : ssn;
  r.dn = side ? -dsn : dsn;
  r.src0 = src0 + (side ? int64_t(op.ns0 - 1) * ssn : 0);
  r.lo0 = op.half_t[h][0];
  r.hi0 = op.half_t[h][1];
  r.lo1 = r.lo2 = 0;
  r.g0 = op.half_g[h][0];
  r.n0 = op.half_g[h][1] - r.g0;
  r.g1 = r.g2 = 0;
  r.n1 = r.n2 = op.G1;
  r.dst = dst0 + (side ? int64_t(r.hi0 - r.lo0 - 1) * dsn : 0);
}

__device__ __forceinline__ void decode_face(const th_face* __restrict__ fp, const DevOp& op, FaceRef& r) {
  if (op.role == 0) decode_face_interp(fp, op, r);
  else decode_face_restrict(fp, op, r);
}

// source address of reference source cell (a0, a1, a2) (relative to lane 0)
__device__ __forceinline__ int64_t src_addr(const th_face* __restrict__ fp, const DevOp& op, const FaceRef& r,
                                            int a0, int a1, int a2) {
  if (op.role == 0) return r.src0 + a0 * r.sn + a1 * r.s1 + a2 * r.s2;
  const int b1 = a1 / op.p, b2 = a2 / op.p;
  const int64_t base = __ldg(&fp->src[b1 + 3 * b2]) + (r.src0 - __ldg(&fp->src[0]));
  return base + a0 * r.sn + (a1 - b1 * op.p) * r.s1 + (a2 - b2 * op.p) * r.s2;
}

__device__ __forceinline__ bool decode_item(const DevOp& op, const FaceRef& fr, int it, int& g0, int& g1, int& g2) {
  const int n12 = fr.n1 * fr.n2;
  if (it >= fr.n0 * n12) return false;
  g1 = fr.g1 + it % fr.n1;
  const int r = it / fr.n1;
  g2 = fr.g2 + r % fr.n2;
  g0 = fr.g0 + r / fr.n2;
  return true;
}

__device__ __forceinline__ void raise_flag(int32_t* flag, bool bad) {
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// generic dense-block apply: out[child] = sum_cell W[cell][child] * v[cell]
// ---------------------------------------------------------------------------
template <int MAXC>
__global__ void __launch_bounds__(128) dense_apply_kernel(DevOp op, const double* __restrict__ src,
                                                          double* __restrict__ dst,
                                                          const th_face* __restrict__ faces, int64_t n_faces,
                                                          int u, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = n_faces * op.max_items;
  for (int64_t item = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; item < total; item += nwarps) {
    const int64_t f = item / op.max_items;
    const int it = int(item - f * op.max_items);
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face(fp, op, fr);
    int g0, g1, g2;
    if (!decode_item(op, fr, it, g0, g1, g2)) continue;
    const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]), G2 = __ldg(&op.grp1[g2]);
    const int bid = __ldg(&op.block_id[(g0 * op.G1 + g1) * op.G1 + g2]);
    const double* __restrict__ W = op.weights + __ldg(&op.block_off[bid]);
    const int CP = __ldg(&op.block_cp[bid]);
    const int C0 = G0.w, C1 = G1.w, C = G0.w * G1.w * G2.w;
    for (int cb = 0; cb < u; cb += 64) {
      const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
      double acc[MAXC][2];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) acc[c][0] = acc[c][1] = 0.0;
      int cell = 0;
      for (int z = 0; z < G2.y; ++z)
        for (int y = 0; y < G1.y; ++y) {
          const int64_t row = src_addr(fp, op, fr, G0.x, G1.x + y, G2.x + z) + cb + lane;
          for (int x = 0; x < G0.y; ++x, ++cell) {
            const double* sp = src + row + int64_t(x) * fr.sn;
            const double v0 = ok0 ? __ldg(sp) : 0.0;
            const double v1 = ok1 ? __ldg(sp + 32) : 0.0;
            const double2* wc = reinterpret_cast<const double2*>(W + int64_t(cell) * CP);
#pragma unroll
            for (int c = 0; c < MAXC; c += 2) {
              if (c < C) {
                const double2 w = __ldg(wc + c / 2);
                acc[c][0] = fma(w.x, v0, acc[c][0]);
                acc[c][1] = fma(w.x, v1, acc[c][1]);
                acc[c + 1][0] = fma(w.y, v0, acc[c + 1][0]);
                acc[c + 1][1] = fma(w.y, v1, acc[c + 1][1]);
              }
            }
          }
        }
      bool bad = false;
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if (c < C) {
          const int i0 = c % C0, i1 = (c / C0) % C1, i2 = c / (C0 * C1);
          const int t0 = G0.z + i0, t1 = G1.z + i1, t2 = G2.z + i2;
          if (t0 >= fr.lo0 && t0 < fr.hi0 && t1 >= fr.lo1 && t1 < fr.lo1 + op.p && t2 >= fr.lo2 &&
              t2 < fr.lo2 + op.p) {
            double* dp = dst + fr.dst + (t0 - fr.lo0) * fr.dn + (t1 - fr.lo1) * fr.d1 + (t2 - fr.lo2) * fr.d2 +
                         cb + lane;
            if (ok0) { dp[0] = acc[c][0]; bad |= !isfinite(acc[c][0]); }
            if (ok1) { dp[32] = acc[c][1]; bad |= !isfinite(acc[c][1]); }
          }
        }
      }
      raise_flag(flag, bad);
    }
  }
}

// ---------------------------------------------------------------------------
// d-linear tensor product: three per-axis passes (normal, t1, t2) over the
// block window, in the reference's contraction order (linear.py:115-151)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) tensor_apply_kernel(DevOp op, const double* __restrict__ src,
                                                           double* __restrict__ dst,
                                                           const th_face* __restrict__ faces, int64_t n_faces,
                                                           int u, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = n_faces * op.max_items;
  for (int64_t item = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; item < total; item += nwarps) {
    const int64_t f = item / op.max_items;
    const int it = int(item - f * op.max_items);
    const th_face* fp = faces + f;
    FaceRef fr;
    decode_face(fp, op, fr);
    int g0, g1, g2;
    if (!decode_item(op, fr, it, g0, g1, g2)) continue;
    const int4 G0 = __ldg(&op.grp0[g0]), G1 = __ldg(&op.grp1[g1]), G2 = __ldg(&op.grp1[g2]);
    const double* __restrict__ R0 = op.rows0 + __ldg(&op.row_off0[g0]);  // [C0][L0]
    const double* __restrict__ R1 = op.rows1 + __ldg(&op.row_off1[g1]);  // [C1][L1]
    const double* __restrict__ R2 = op.rows1 + __ldg(&op.row_off1[g2]);  // [C2][L2]
    for (int cb = 0; cb < u; cb += 64) {
      const bool ok0 = cb + lane < u, ok1 = cb + lane + 32 < u;
      double out[3][3][3][2];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < 3; ++c) out[a][b][c][0] = out[a][b][c][1] = 0.0;
      for (int z = 0; z < G2.y; ++z) {
        double tyz[3][3][2];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) tyz[a][b][0] = tyz[a][b][1] = 0.0;
        for (int y = 0; y < G1.y; ++y) {
          const int64_t row = src_addr(fp, op, fr, G0.x, G1.x + y, G2.x + z) + cb + lane;
          double tx[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          for (int x = 0; x < G0.y; ++x) {
            const double* sp = src + row + int64_t(x) * fr.sn;
            const double v0 = ok0 ? __ldg(sp) : 0.0;
            const double v1 = ok1 ? __ldg(sp + 32) : 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
              if (a < G0.w) {
                const double w = __ldg(R0 + a * G0.y + x);
                tx[a][0] = fma(w, v0, tx[a][0]);
                tx[a][1] = fma(w, v1, tx[a][1]);
              }
          }
#pragma unroll
          for (int b = 0; b < 3; ++b)
            if (b < G1.w) {
              const double w = __ldg(R1 + b * G1.y + y);
#pragma unroll
              for (int a = 0; a < 3; ++a) {
                tyz[a][b][0] = fma(w, tx[a][0], tyz[a][b][0]);
                tyz[a][b][1] = fma(w, tx[a][1], tyz[a][b][1]);
              }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < G2.w) {
            const double w = __ldg(R2 + c * G2.y + z);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                out[a][b][c][0] = fma(w, tyz[a][b][0], out[a][b][c][0]);
                out[a][b][c][1] = fma(w, tyz[a][b][1], out[a][b][c][1]);
              }
          }
      }
      bool bad = false;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (a < G0.w && b < G1.w && c < G2.w) {
              const int t0 = G0.z + a, t1 = G1.z + b, t2 = G2.z + c;
              if (t0 >= fr.lo0 && t0 < fr.hi0 && t1 >= fr.lo1 && t1 < fr.lo1 + op.p && t2 >= fr.lo2 &&
                  t2 < fr.lo2 + op.p) {
                double* dp = dst + fr.dst + (t0 - fr.lo0) * fr.dn + (t1 - fr.lo1) * fr.d1 +
                             (t2 - fr.lo2) * fr.d2 + cb + lane;
                if (ok0) { dp[0] = out[a][b][c][0]; bad |= !isfinite(out[a][b][c][0]); }
                if (ok1) { dp[32] = out[a][b][c][1]; bad |= !isfinite(out[a][b][c][1]); }
              }
            }
          }
      raise_flag(flag, bad);
    }
  }
}

#include "helpers.cuh"
#include "window.cuh"
#include "restrict_pipe.cuh"
#include "gram_slide.cuh"
#include "stage_slide.cuh"
#include "tile_interp.cuh"
#include "tile_interp3.cuh"
#include "ring_interp.cuh"

__global__ void finite_kernel(const double* __restrict__ v, int64_t n, int32_t* flag) {
  bool bad = false;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(__ldg(v + i));
  raise_flag(flag, bad);
}

// csr._apply_kernel (csr.py:143-156): one warp per row, lanes over unknowns
__global__ void csr_apply_kernel(const int64_t* __restrict__ ro, const int64_t* __restrict__ ci,
                                 const double* __restrict__ val, int64_t n_rows, const double* __restrict__ src,
                                 double* __restrict__ out, int u) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nwarps) {
    const int64_t lo = __ldg(ro + r), hi = __ldg(ro + r + 1);
    for (int cb = 0; cb < u; cb += 32) {
      if (cb + lane >= u) break;
      double acc = 0.0;
      for (int64_t t = lo; t < hi; ++t) acc = fma(__ldg(val + t), __ldg(src + __ldg(ci + t) * u + cb + lane), acc);
      out[r * u + cb + lane] = acc;
    }
  }
}

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct th_operator {
  th::HostOperator host;
  DevOp dev;
  std::vector<void*> allocs;
  int64_t bytes = 0;
  int max_children = 0;
  bool on_device = false;
  bool smem_ok = false;
  size_t smem_bytes = 0;
  // restriction register kernel: mode (0 = not eligible), window, classes, params blob
  int r_mode = 0, r_L = 0, r_ncls = 0;
  std::vector<unsigned char> r_params;
  // staged order3 restriction (stage_slide.cuh) eligibility and its folded weights
  bool st_ok = false;
  std::vector<int32_t> st_cls;
  std::vector<double> st_w;
  // staged tile interpolation (tile_interp.cuh): mode (0 = not eligible, 1 = tensor_linear,
  // 2 = order2 Gram) and tiles per face axis
  int ti_mode = 0, ti_nt = 0;
  // staged order3 tile interpolation (tile_interp3.cuh) eligibility
  bool t3_ok = false;
  int t3_nt = 1;
  // slice-ring interpolation (ring_interp.cuh): window length (0 = not eligible), t1 parts per
  // face, and the largest line / window-start / slice counts of a tile
  int rg_L = 0, rg_ntp = 1, rg_nymax = 0, rg_nsmax = 0, rg_nzmax = 0;
  bool rg_tensor = false;  // d-linear 1-D rows (tensor_linear, matrix_linear in factored form) instead of Gram moments
};

namespace {

template <int MODE, int L, int NCLS>
bool fill_restrict_params(const th::HostOperator& h, std::vector<unsigned char>& blob) {
  using PT = RestrictParams<MODE, L, NCLS>;
  PT prm;
  std::memset(&prm, 0, sizeof(prm));
  constexpr int S = L * L * L;
  if (MODE == 1) {
    if ((int)h.block_off.size() > NCLS) return false;
    for (size_t b = 0; b < h.block_off.size(); ++b) {
      if (h.block_cp[b] != 4) return false;
      for (int cell = 0; cell < S; ++cell)
        for (int c = 0; c < 3; ++c) prm.w[b][cell][c] = h.weights[h.block_off[b] + size_t(cell) * 4 + c];
    }
  } else {
    if (h.groups[0].size() != 1 || h.rows[0].size() != size_t(3 * L)) return false;
    for (int c = 0; c < 3; ++c)
      for (int x = 0; x < L; ++x) prm.r0[c][x] = h.rows[0][c * L + x];
    for (size_t g = 0; g < h.groups[1].size(); ++g)
      for (int y = 0; y < L; ++y) {
        const double v = h.rows[1][h.row_off[1][g] + y];
        if (g == 0) prm.rt[y] = v;
        else if (v != prm.rt[y]) return false;
      }
  }
  blob.resize(sizeof(PT));
  std::memcpy(blob.data(), &prm, sizeof(PT));
  return true;
}

// eligibility of the register restriction kernel (restrict_pipe.cuh)
void prepare_restrict(th_operator* op) {
  const th::HostOperator& h = op->host;
  op->r_mode = 0;
  if (h.role != 1 || h.k != 3 || h.fast_C0 != 3 || h.fast_CT != 1 || h.groups[0].size() != 1 ||
      h.groups[0][0].tgtN != 3)
    return;
  for (const auto& g : h.groups[1])
    if (g.tgtN != 1) return;
  bool ok = false;
  if (h.fast_mode == 1 && h.fast_L0 == 3) ok = fill_restrict_params<1, 3, 1>(h, op->r_params), op->r_ncls = 1;
  else if (h.fast_mode == 1 && h.fast_L0 == 5) ok = fill_restrict_params<1, 5, 9>(h, op->r_params), op->r_ncls = 9;
  else if (h.fast_mode == 2 && h.fast_L0 == 3) ok = fill_restrict_params<2, 3, 1>(h, op->r_params), op->r_ncls = 1;
  if (ok) {
    op->r_mode = h.fast_mode;
    op->r_L = h.fast_L0;
  }
}

// eligibility of the staged order3 restriction (stage_slide.cuh): every face
// half has one normal group (5-cell window, <= 3 children); tangential groups
// have 5-cell windows and one child, starts non-decreasing, and window j + 2
// starts after window j ends (a fine slice feeds at most two coarse columns)
void prepare_stage(th_operator* op) {
  const th::HostOperator& h = op->host;
  op->st_ok = false;
  if (h.role != 1 || h.scheme != TH_SCHEME_ORDER3 || !h.gram_ok || h.synth[0].empty() || h.synth[1].empty()) return;
  for (int a = 0; a < 3; ++a)
    if (h.half_g[a][1] - h.half_g[a][0] > 1) return;
  for (const auto& g : h.groups[0])
    if (g.winL != 5 || g.tgtN < 1 || g.tgtN > 3) return;
  const auto& g1 = h.groups[1];
  if (g1.empty()) return;
  for (size_t j = 0; j < g1.size(); ++j) {
    if (g1[j].winL != 5 || g1[j].tgtN != 1) return;
    if (j > 0 && g1[j].win0 < g1[j - 1].win0) return;
    if (j + 2 < g1.size() && g1[j + 2].win0 < g1[j].win0 + 5) return;
  }
  // Fold the tangential synthesis into per-window weights.  With one t1 child and one t2
  // child per window the order3 LS value is
  //   out_i = sum_a S0_i[a] U_a,   U_a = sum_{y,z} W_a(y, z) m_a(y, z),
  //   W_a(y, z) = sum_{b + c <= 3 - a} S1[b] P_b(y) S2[c] P_c(z)
  // (m_a = normal Gram moment of source line (y, z)); W depends only on the windows' synthesis
  // rows, i.e. on the (t1, t2) pair of row classes: interior windows share one row, clipped edge
  // windows have their own.
  const int G = (int)g1.size();
  std::vector<int> rep;  // first group of each class
  op->st_cls.assign(G, 0);
  for (int g = 0; g < G; ++g) {
    int c = 0;
    for (; c < (int)rep.size(); ++c)
      if (std::equal(h.synth[1].begin() + g * 12, h.synth[1].begin() + g * 12 + 4,
                     h.synth[1].begin() + rep[c] * 12))
        break;
    if (c == (int)rep.size()) rep.push_back(g);
    op->st_cls[g] = c;
  }
  const int nc = (int)rep.size();
  if (nc > 6) return;  // > 29 KB of weights: keep the generic slide
  auto P = [](int d, int x) -> double {  // 5-point Gram polynomials (window.cuh Gram<5>)
    const int t = x - 2;
    return d == 0 ? 1.0 : d == 1 ? double(t) : d == 2 ? double(t * t - 2) : double(5 * t * t * t - 17 * t) / 6.0;
  };
  op->st_w.assign(size_t(nc) * nc * 100, 0.0);
  for (int c1 = 0; c1 < nc; ++c1)
    for (int c2 = 0; c2 < nc; ++c2) {
      const double* S1 = &h.synth[1][rep[c1] * 12];
      const double* S2 = &h.synth[1][rep[c2] * 12];
      for (int z = 0; z < 5; ++z)
        for (int y = 0; y < 5; ++y)
          for (int a = 0; a < 4; ++a) {
            double w = 0.0;
            for (int b = 0; a + b < 4; ++b)
              for (int c = 0; a + b + c < 4; ++c) w += S1[b] * P(b, y) * S2[c] * P(c, z);
            op->st_w[(size_t(c1 * nc + c2) * 25 + z * 5 + y) * 4 + a] = w;
          }
    }
  op->st_ok = true;
}

// Staged tile interpolation eligibility (tile_interp.cuh): one normal group with a 3-cell
// window and <= 3 children; tangential groups with 3-cell windows, <= 3 children and
// non-decreasing starts.  A face axis splits into ti_nt balanced tiles of <= 3 groups whose
// windows span <= TNY cells (the shared-memory box).
void prepare_tile(th_operator* op) {
  const th::HostOperator& h = op->host;
  op->ti_mode = 0;
  if (h.role != 0 || h.groups[0].size() != 1 || h.groups[1].empty()) return;
  int mode = 0;
  // tensor_linear, and matrix_linear: its operator is the collapsed product of the same 1-D
  // rows (linear.py:202-245), evaluated here in factored form (weights equal up to rounding)
  const bool linear_rows = h.fast_mode == 2 || (h.fast_mode == 1 && h.scheme == TH_SCHEME_MATRIX_LINEAR);
  if (linear_rows && h.fast_L0 == 3 && h.fast_C0 == 3 && h.fast_CT == 3) mode = 1;
  else if (h.gram_ok && h.fast_C0 == 3 && h.scheme == TH_SCHEME_ORDER2 && !h.synth[1].empty()) mode = 2;
  if (!mode) return;
  const th::Group& g0 = h.groups[0][0];
  if (g0.winL != 3 || g0.tgtN < 1 || g0.tgtN > 3) return;
  const auto& g1 = h.groups[1];
  for (size_t j = 0; j < g1.size(); ++j) {
    if (g1[j].winL != 3 || g1[j].tgtN < 1 || g1[j].tgtN > 3) return;
    if (j > 0 && g1[j].win0 < g1[j - 1].win0) return;
  }
  int nmax = 0;
  for (int c = 0; c < 3; ++c) nmax = std::max(nmax, h.seg_g[c][1] - h.seg_g[c][0]);
  if (nmax < 1) return;
  const int nt = (nmax + 2) / 3;
  for (int c = 0; c < 3; ++c) {
    const int n = h.seg_g[c][1] - h.seg_g[c][0];
    for (int t = 0; t < nt; ++t) {
      const int a = t * n / nt, b = (t + 1) * n / nt;
      if (b - a > 3) return;
      if (b > a && g1[h.seg_g[c][0] + b - 1].win0 + 3 - g1[h.seg_g[c][0] + a].win0 > TNY) return;
    }
  }
  // one tile per face only: at p = 17 (3 x 3 tiles of partial blocks) the per-warp slide is
  // faster (config 4 order2 interpolation 0.56 vs 0.43-0.49 of HBM, profiles/r01_ab_tile.txt)
  if (nt > 1) return;
  op->ti_mode = mode;
  op->ti_nt = nt;
}

// Staged order3 tile interpolation eligibility (tile_interp3.cuh): one normal group with a
// 5-cell window and <= 3 children; tangential groups with 5-cell windows, <= 3 children and
// non-decreasing starts; every segment axis splits into t3_nt balanced runs of <= 3 groups
// whose windows span <= T3Y cells (one run at p <= 9, three at p = 17).
void prepare_tile3(th_operator* op) {
  const th::HostOperator& h = op->host;
  op->t3_ok = false;
  if (h.role != 0 || h.scheme != TH_SCHEME_ORDER3 || !h.gram_ok || h.fast_C0 != 3 || h.synth[0].empty() ||
      h.synth[1].empty() || h.groups[0].size() != 1 || h.groups[1].empty())
    return;
  const th::Group& g0 = h.groups[0][0];
  if (g0.winL != 5 || g0.tgtN < 1 || g0.tgtN > 3) return;
  const auto& g1 = h.groups[1];
  for (size_t j = 0; j < g1.size(); ++j) {
    if (g1[j].winL != 5 || g1[j].tgtN < 1 || g1[j].tgtN > 3) return;
    if (j > 0 && g1[j].win0 < g1[j - 1].win0) return;
  }
  int nmax = 0;
  for (int c = 0; c < 3; ++c) nmax = std::max(nmax, h.seg_g[c][1] - h.seg_g[c][0]);
  if (nmax < 1) return;
  const int nt = (nmax + 2) / 3;  // spatial tiles per face axis: <= 3 groups each
  for (int c = 0; c < 3; ++c) {
    const int a0 = h.seg_g[c][0], n = h.seg_g[c][1] - a0;
    for (int t = 0; t < nt; ++t) {
      const int a = a0 + t * n / nt, b = a0 + (t + 1) * n / nt;
      if (b - a > 3) return;
      if (b > a && g1[b - 1].win0 + 5 - g1[a].win0 > T3Y) return;
    }
  }
  op->t3_nt = nt;
  op->t3_ok = true;
}

// Slice-ring interpolation (ring_interp.cuh): Gram least squares with one normal group of
// 3 children, full windows of L = 3 / 5 cells on every tangential group, window starts
// non-decreasing in steps of <= 1 (so every source slice lies in some row's window).  A
// segment's blocks along t1 split into rg_ntp balanced parts of <= RG_NS blocks whose lines
// span <= L + 3 cells.
void prepare_ring(th_operator* op) {
  const th::HostOperator& h = op->host;
  op->rg_L = 0;
  op->rg_tensor = false;
  if (h.role != 0 || h.groups[0].size() != 1 || h.groups[1].empty()) return;
  // tensor_linear, and matrix_linear in factored form (the collapsed operator is the product of
  // the same 1-D rows, linear.py:202-245; cf. prepare_tile)
  const bool linear_rows = (h.fast_mode == 2 || (h.fast_mode == 1 && h.scheme == TH_SCHEME_MATRIX_LINEAR)) &&
                           h.fast_L0 == 3 && h.fast_C0 == 3 && h.fast_CT == 3 && !h.rows[0].empty() &&
                           !h.rows[1].empty();
  const bool gram = (h.scheme == TH_SCHEME_ORDER2 || h.scheme == TH_SCHEME_ORDER3) && h.gram_ok && h.fast_C0 == 3 &&
                    h.synth[0].size() >= 12 && !h.synth[1].empty();
  if (!linear_rows && !gram) return;
  const int L = linear_rows ? 3 : h.scheme == TH_SCHEME_ORDER2 ? 3 : 5;
  const th::Group& g0 = h.groups[0][0];
  if (g0.winL != L || g0.tgtN < 1 || g0.tgtN > 3) return;
  const auto& g1 = h.groups[1];
  for (size_t j = 0; j < g1.size(); ++j) {
    if (g1[j].winL != L || g1[j].tgtN < 1 || g1[j].tgtN > 3) return;
    if (j > 0 && (g1[j].win0 < g1[j - 1].win0 || g1[j].win0 > g1[j - 1].win0 + 1)) return;
  }
  int nmax = 0;
  for (int c = 0; c < 3; ++c) nmax = std::max(nmax, h.seg_g[c][1] - h.seg_g[c][0]);
  if (nmax < 1) return;
  for (int ntp = (nmax + RG_NS - 1) / RG_NS; ntp <= nmax; ++ntp) {
    bool ok = true;
    int nymax = 0, nsmax = 0, nzmax = 0;
    for (int c = 0; c < 3 && ok; ++c) {
      const int a0 = h.seg_g[c][0], n = h.seg_g[c][1] - a0;
      if (n < 1) continue;
      nzmax = std::max(nzmax, g1[a0 + n - 1].win0 + L - g1[a0].win0);
      for (int t = 0; t < ntp && ok; ++t) {
        const int a = a0 + t * n / ntp, b = a0 + (t + 1) * n / ntp;
        if (b <= a) continue;
        const int ny = g1[b - 1].win0 + L - g1[a].win0;
        ok = b - a <= RG_NS && ny <= L + 3;
        nymax = std::max(nymax, ny);
        nsmax = std::max(nsmax, linear_rows ? b - a : ny - L + 1);  // T entries per slice: blocks / window starts
      }
    }
    if (ok) {
      op->rg_L = L;
      op->rg_tensor = linear_rows;
      op->rg_ntp = ntp;
      op->rg_nymax = nymax;
      op->rg_nsmax = nsmax;
      op->rg_nzmax = nzmax;
      return;
    }
  }
}

// launch geometry of the slice-staged kernels (stage_slide.cuh) for u unknowns;
// false = the operator / u does not fit them
struct StageGeom {
  int nst = 0, stage_d = 0, ny_max = 0, tg = 0, tiles_per_face = 0, out_d = 0;
  size_t smem = 0;
  bool own = false;  // line-owner consumers (stage_slide.cuh, OWN): ncw + 1 consumer warps
};
// restriction: one consumer warp per t1 group at u <= 64, two unknowns per lane (18 warps with one
// unknown per lane measured 0.76 against 0.845 of the copy peak: profiles/r02_ab_restriction.txt)
constexpr int kRestrictNCW = 9, kRestrictNU = 2;

bool stage_geometry(const th_operator* op, int u, int minb, StageGeom& g) {
  const th::HostOperator& h = op->host;
  if (h.role != 1 || !op->st_ok) return false;
  const int L = h.fast_L0 > 0 ? h.fast_L0 : 5;
  const int ncw = kRestrictNCW, nu = kRestrictNU;
  const int nch = (u + 32 * nu - 1) / (32 * nu);
  if (nch > ncw) return false;
  const auto& g1 = h.groups[1];
  const int max_n = (int)g1.size();
  if (max_n == 0) return false;
  const int tiles = (max_n + ncw / nch - 1) / (ncw / nch);
  g.tg = (max_n + tiles - 1) / tiles;
  g.tiles_per_face = tiles;
  g.ny_max = 0;
  for (int ga = 0; ga < max_n; ga += g.tg) {
    const int gb = std::min(max_n, ga + g.tg);
    g.ny_max = std::max(g.ny_max, g1[gb - 1].win0 + L - g1[ga].win0);
  }
  // stage rows hold runs of u-double cells widened to 16-byte boundaries; lanes past u read up to
  // 63 - u doubles beyond a cell (never stored), covered by the regions that follow the stages
  g.stage_d = (L * g.ny_max * ((u + 3) & ~1) + 1) & ~1;  // cell slots of round_even(u + 2) doubles
  const size_t extra = op->st_w.size() * 8 + 20 * 8;
  // (dynamic shared memory: the opt-in maximum less the kernels' static tables)
  const size_t budget = size_t(227 * 1024) / size_t(minb) - 3072;
  // Line-owner consumers: every line of a slice projected once (u <= 64; every warp owns <= 3 lines
  // of a tile: window starts step by <= 3, the last group's window starts >= 2 after its
  // neighbour's) where the hand-over slots fit beside a 3-stage ring (p = 9; at p = 17 they do not).
  //   TH_ROWN=0                  one consumer warp per t1 group (5 lines each) instead (A/B, tests)
  static const int use_own = [] { const char* e = std::getenv("TH_ROWN"); return e ? std::atoi(e) : 1; }();
  bool own = use_own && nch == 1 && nu == 2 && L == 5 && g.tg <= ncw;
  for (int ga = 0; own && ga < max_n; ga += g.tg) {
    const int gb = std::min(max_n, ga + g.tg);
    for (int i = ga; i + 1 < gb; ++i) own &= g1[i + 1].win0 - g1[i].win0 <= 3;
    if (gb - ga >= 2) own &= g1[gb - 1].win0 - g1[gb - 2].win0 >= 2;
  }
  const size_t xch = size_t(ncw) * nu * 4 * 32 * 8;
  for (int nst = 3; nst >= 2; --nst) {
    const size_t smem = size_t(nst) * g.stage_d * 8 + extra + size_t(nst) * 16 + size_t(nst) * g.ny_max * 4 +
                        size_t(L) * g.ny_max + 64 * 8;
    if (nst == 3 && own && smem + xch <= budget) {
      g.nst = nst;
      g.smem = smem + xch;
      g.own = true;
      return true;
    }
    if (smem <= budget) {
      g.nst = nst;
      g.smem = smem;
      g.out_d = 0;
      return true;
    }
  }
  return false;
}

template <class T>
int32_t upload(th_operator* op, const std::vector<T>& v, const T** out) {
  if (v.empty()) { *out = nullptr; return TH_OK; }
  void* p = nullptr;
  TH_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
  op->allocs.push_back(p);
  TH_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  op->bytes += int64_t(v.size() * sizeof(T));
  *out = static_cast<const T*>(p);
  return TH_OK;
}

int32_t map_error(const th::Error& e) {
  return fail(int32_t(e.code), e.what(), e.column);
}

}  // namespace

extern "C" {

int32_t th_abi_version(void) { return 1; }

const char* th_last_error(void) { return g_last_error.c_str(); }

int32_t th_last_error_column(void) { return g_last_column; }

int32_t th_scheme_feasible(int32_t role, int32_t scheme, int32_t p, int32_t k) {
  try {
    th::check_feasible(role, scheme, p, k);
  } catch (const th::Error& e) {
    return map_error(e);
  }
  return TH_OK;
}

void th_operator_destroy(th_operator* op) {
  if (!op) return;
  for (void* p : op->allocs) cudaFree(p);
  delete op;
}

static int32_t operator_create(int32_t role, int32_t scheme, int32_t p, int32_t k, th_operator** out,
                               bool upload_to_device) {
  if (!out) return fail(TH_ERR_CONFIG, "out pointer is NULL");
  *out = nullptr;
  th_operator* op = new th_operator();
  try {
    op->host = th::build_operator(role, scheme, p, k);
  } catch (const th::Error& e) {
    delete op;
    return map_error(e);
  } catch (const std::exception& e) {
    delete op;
    return fail(TH_ERR_CONFIG, e.what());
  }
  const th::HostOperator& h = op->host;
  DevOp& d = op->dev;
  std::memset(&d, 0, sizeof(d));
  d.role = h.role;
  d.scheme = h.scheme;
  d.p = h.p;
  d.k = h.k;
  d.ns0 = h.ax[0].ns;
  d.G0 = (int)h.groups[0].size();
  d.G1 = (int)h.groups[1].size();
  d.max_items = h.max_items;
  std::memcpy(d.seg_g, h.seg_g, sizeof(d.seg_g));
  std::memcpy(d.half_g, h.half_g, sizeof(d.half_g));
  std::memcpy(d.half_t, h.half_t, sizeof(d.half_t));
  std::vector<int4> g0, g1;
  for (const auto& g : h.groups[0]) {
    g0.push_back(make_int4(g.win0, g.winL, g.tgt0, g.tgtN));
    op->max_children = std::max(op->max_children, g.tgtN);
  }
  int mc1 = 0;
  for (const auto& g : h.groups[1]) {
    g1.push_back(make_int4(g.win0, g.winL, g.tgt0, g.tgtN));
    mc1 = std::max(mc1, g.tgtN);
  }
  op->max_children *= mc1 * mc1;
  op->on_device = upload_to_device;
  d.n_blocks = (int32_t)h.block_off.size();
  {
    const char* e = std::getenv("TH_PREFETCH");
    // bit 1: restriction window bulk prefetch, bit 8: interp unit windows, bit 16: staged tile
    // interpolation prefetches the tile after next (profiles/r01_ab_tile3.txt)
    d.prefetch = e ? std::atoi(e) : 25;
  }
  d.units_per_face = 0;
  d.ns_t = h.ax[1].ns;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      d.units_per_face = std::max(d.units_per_face, (h.half_g[a][1] - h.half_g[a][0]) * (h.seg_g[b][1] - h.seg_g[b][0]));
  op->smem_ok = h.fast_mode == 1 && h.fast_C0 * h.fast_CT * h.fast_CT <= 4;
  for (size_t b = 0; b < h.block_cp.size() && op->smem_ok; ++b)
    op->smem_ok = h.block_cp[b] == 4 &&
                  h.block_off[b] == int64_t(b) * 4 * h.fast_L0 * h.fast_LT * h.fast_LT;
  op->smem_bytes = op->smem_ok ? size_t(d.n_blocks) * h.fast_L0 * h.fast_LT * h.fast_LT * 32 : 0;
  if (op->smem_bytes > 200 * 1024) op->smem_ok = false;
  prepare_restrict(op);
  prepare_stage(op);
  prepare_tile(op);
  prepare_tile3(op);
  prepare_ring(op);
  if (!upload_to_device) {
    *out = op;
    return TH_OK;
  }
  int32_t rc;
  if ((rc = upload(op, g0, &d.grp0)) || (rc = upload(op, g1, &d.grp1)) || (rc = upload(op, h.block_id, &d.block_id)) ||
      (rc = upload(op, h.block_off, &d.block_off)) || (rc = upload(op, h.block_cp, &d.block_cp)) ||
      (rc = upload(op, h.weights, &d.weights)) || (rc = upload(op, h.row_off[0], &d.row_off0)) ||
      (rc = upload(op, h.rows[0], &d.rows0)) || (rc = upload(op, h.row_off[1], &d.row_off1)) ||
      (rc = upload(op, h.rows[1], &d.rows1)) || (rc = upload(op, h.synth[0], &d.synth0)) ||
      (rc = upload(op, h.synth[1], &d.synth1)) || (rc = upload(op, op->st_cls, &d.st_cls)) ||
      (rc = upload(op, op->st_w, &d.st_w))) {
    th_operator_destroy(op);
    return rc;
  }
  d.st_ncls = op->st_ok ? (int32_t)std::lround(std::sqrt(double(op->st_w.size() / 100))) : 0;
  *out = op;
  return TH_OK;
}

int32_t th_operator_create(int32_t role, int32_t scheme, int32_t p, int32_t k, th_operator** out) {
  return operator_create(role, scheme, p, k, out, true);
}

int32_t th_operator_create_host(int32_t role, int32_t scheme, int32_t p, int32_t k, th_operator** out) {
  return operator_create(role, scheme, p, k, out, false);
}

int32_t th_operator_info_get(const th_operator* op, th_operator_info* info) {
  if (!op || !info) return fail(TH_ERR_CONFIG, "NULL operator or info");
  const th::HostOperator& h = op->host;
  info->role = h.role;
  info->scheme = h.scheme;
  info->p = h.p;
  info->k = h.k;
  info->n_src_cells = h.n_src_cells();
  info->n_tgt_cells_full = h.n_tgt_cells();
  info->n_blocks = (int32_t)h.block_off.size();
  info->max_items_per_face = h.max_items;
  info->device_bytes = op->bytes;
  info->max_condition = h.max_condition;
  info->n_condition_warnings = h.n_condition_warnings;
  info->kernel = h.scheme == TH_SCHEME_TENSOR_LINEAR ? 1 : 0;
  return TH_OK;
}

int32_t th_operator_export_rows(const th_operator* op, int32_t selector, int64_t* n_rows, int64_t* nnz,
                                int64_t* row_offsets, int64_t* col_indices, double* values) {
  if (!op || !n_rows || !nnz) return fail(TH_ERR_CONFIG, "NULL argument");
  std::vector<int64_t> ro, ci;
  std::vector<double> v;
  try {
    th::export_rows(op->host, selector, ro, ci, v);
  } catch (const th::Error& e) {
    return map_error(e);
  }
  *n_rows = int64_t(ro.size()) - 1;
  *nnz = int64_t(ci.size());
  if (row_offsets) std::memcpy(row_offsets, ro.data(), ro.size() * sizeof(int64_t));
  if (col_indices) std::memcpy(col_indices, ci.data(), ci.size() * sizeof(int64_t));
  if (values) std::memcpy(values, v.data(), v.size() * sizeof(double));
  return TH_OK;
}

// Resident CTAs per SM of a kernel at a dynamic shared-memory size, computed once per
// (device, kernel, size): launches stay cheap and concurrent callers share the cache.  The
// kernel's dynamic-smem limit is raised to the device's opt-in maximum the first time the
// kernel is seen on a device (a limit raised only to the first size seen would reject a later,
// larger launch of the same kernel).
static cudaError_t resident_ctas(const void* kfn, int nth, size_t smem, int* per_sm) {
  struct Entry {
    int dev;
    const void* fn;
    size_t smem;
    int per_sm;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  static std::vector<std::pair<int, const void*>> raised;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& c : cache)
    if (c.dev == dev && c.fn == kfn && c.smem == smem) {
      *per_sm = c.per_sm;
      return cudaSuccess;
    }
  if (std::find(raised.begin(), raised.end(), std::make_pair(dev, kfn)) == raised.end()) {
    int optin = 0;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, kfn)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - int(fa.sharedSizeBytes))) != cudaSuccess)
      return e;
    raised.emplace_back(dev, kfn);
  }
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kfn, nth, smem)) != cudaSuccess) return e;
  cache.push_back({dev, kfn, smem, *per_sm});
  return cudaSuccess;
}

int32_t th_apply_faces(const th_operator* op, const double* src, double* dst, const th_face* faces, int64_t n_faces,
                       int32_t u, int32_t* flag, void* stream) {
  if (!op) return fail(TH_ERR_CONFIG, "NULL operator");
  if (!op->on_device) return fail(TH_ERR_CONTRACT, "operator was built host-only (th_operator_create_host)");
  if (u < 1) return fail(TH_ERR_CONFIG, "u must be >= 1, got " + std::to_string(u));
  if (n_faces < 0) return fail(TH_ERR_CONFIG, "n_faces must be >= 0");
  if (n_faces == 0) return TH_OK;
  if (!src || !dst || !faces) return fail(TH_ERR_CONTRACT, "NULL source, target or face pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t items = n_faces * int64_t(op->dev.max_items);
  const int threads = 128;
  const int64_t want = (items + 3) / 4;
  const int blocks = int(std::min<int64_t>(want, int64_t(num_sms()) * 16));
  const th::HostOperator& h = op->host;
  const bool interp = h.role == 0;
  bool done = true;
#define TH_WIN(MODE, L, CT, ORDER, NU, SMEM, MINB)                                                     \
  do {                                                                                                 \
    auto kfn = window_kernel<MODE, L, L, 3, CT, ORDER, NU, MINB>;                                    \
    if (SMEM > 48 * 1024) TH_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM))); \
    const int64_t units = n_faces * int64_t(op->dev.units_per_face);                                  \
    const int wblocks = int(std::min<int64_t>((units + 3) / 4, int64_t(num_sms()) * 16));              \
    kfn<<<wblocks, threads, SMEM, s>>>(op->dev, src, dst, faces, n_faces, u, flag);                    \
  } while (0)
#define TH_RREG(MODE, L, NCLS, NU, MINB, CTAS)                                                        \
  do {                                                                                                 \
    using PT = RestrictParams<MODE, L, NCLS>;                                                          \
    const PT* prm = reinterpret_cast<const PT*>(op->r_params.data());                                 \
    const int64_t warps_needed = n_faces * int64_t(op->dev.max_items);                                \
    const int rblocks = int(std::min<int64_t>((warps_needed + 3) / 4, int64_t(num_sms()) * CTAS));    \
    restrict_reg_kernel<MODE, L, NCLS, NU, MINB><<<rblocks, 128, 0, s>>>(op->dev, *prm, src, dst, faces, n_faces, u, flag); \
  } while (0)
#define TH_GRAM(ORDER, ROLE, MINB)                                                                     \
  do {                                                                                                 \
    auto kfn = gram_slide_kernel<ORDER, ROLE, MINB>;                                                   \
    const size_t smem = size_t(4) * (ORDER == 2 ? 3 * 6 : 5 * 10) * 32 * 8 +                           \
                        size_t(op->dev.G0 + op->dev.G1) * 12 * 8;                                      \
    if (smem > 48 * 1024) TH_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); \
    const int64_t units = n_faces * int64_t(op->dev.units_per_face) * ((u + 31) / 32);                 \
    const int gblocks = int(std::min<int64_t>((units + 3) / 4, int64_t(num_sms()) * MINB * 2));       \
    kfn<<<gblocks, 128, smem, s>>>(op->dev, src, dst, faces, n_faces, u, flag);                        \
  } while (0)
#define TH_SLIDE(ROLE, ORDER, TENSOR, NCW, NU, MINB)                                                          \
  do {                                                                                                        \
    auto kfn = sg.own       ? stage_slide_kernel<ROLE, ORDER, TENSOR, NCW + 1, 3, NU, MINB, true>             \
               : sg.nst == 3 ? stage_slide_kernel<ROLE, ORDER, TENSOR, NCW, 3, NU, MINB>                      \
                             : stage_slide_kernel<ROLE, ORDER, TENSOR, NCW, 2, NU, MINB>;                     \
    TH_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sg.smem)));           \
    const int64_t tiles = n_faces * sg.tiles_per_face;                                                       \
    const int sblocks = int(std::min<int64_t>(tiles, int64_t(num_sms()) * MINB));                             \
    kfn<<<sblocks, (NCW + (sg.own ? 2 : 1)) * 32, sg.smem, s>>>(op->dev, src, dst, faces, n_faces, u, flag,   \
                                                                sg.stage_d, sg.ny_max, sg.tg,                 \
                                                                sg.tiles_per_face, sg.out_d);                 \
  } while (0)
  // Kernel choice: the measured defaults (profiles/r01_ab_*.txt, r02_*); register budgets are the
  // largest occupancies at which the hot kernels do not spill.  Environment switches, read once
  // per process, select the fallbacks for A/B runs and are exercised by the GPU tests:
  //   TH_GRAM bits (default 15)  1: Gram slide for order2 / order3 interpolation
  //                              2: Gram slide for order3 restriction (fallback of bit 4)
  //                              4: slice-staged order3 restriction (stage_slide.cuh)
  //                              8: tensor_linear interpolation through the slice ring
  //   TH_TILE=0                  per-warp slide (gram_slide.cuh) instead of the tile-parallel
  //                              interpolation kernel (tile_interp.cuh)
  //   TH_TILE3=0                 order3 interpolation through the per-warp slide instead of the
  //                              staged two-phase tiles (tile_interp3.cuh)
  // (Round 1's TH_STAGE_INTERP, TH_TILE_CFG, TH_TILE_MULTI and TH_TILE3=2 variants lost their
  // A/Bs and were removed.)
  static const int use_gram = [] { const char* e = std::getenv("TH_GRAM"); return e ? std::atoi(e) : 15; }();
  const bool gram = h.gram_ok && h.fast_C0 == 3;
  const bool tensor_fast = h.fast_mode == 2 && h.fast_L0 == 3 && h.fast_C0 == 3 && h.fast_CT == 3;
  static const int use_tile = [] { const char* e = std::getenv("TH_TILE"); return e ? std::atoi(e) : 1; }();
  //   TH_RING bits (default 11)  1: order3 interpolation through the slice ring (ring_interp.cuh)
  //                                 where the order3 tiles do not fit (p = 17)
  //                              2: order2 interpolation likewise, where the 3-cell tiles do not fit
  //                              8: tensor_linear / matrix_linear interpolation likewise
  //                              4: the slice ring instead of the tile kernels wherever it fits
  //   TH_RING_NA, TH_RING_R      A warps / ring slots of the slice ring (defaults: Gram 7 A warps for
  //                              rows of <= 3 blocks, 5 otherwise, d-linear 8; as many slots as fit)
  static const int use_ring = [] { const char* e = std::getenv("TH_RING"); return e ? std::atoi(e) : 11; }();
  static const int ring_na = [] { const char* e = std::getenv("TH_RING_NA"); return e ? std::atoi(e) : 0; }();
  auto ring_launch = [&]() -> int32_t {
    const int L = op->rg_L, NP = (L == 5 || op->rg_tensor) ? 10 : 6;
    const int nch = (u + 31) / 32;
    int cmax = 0;
    for (int c = 0; c < nch; ++c) cmax = std::max(cmax, int(int64_t(c + 1) * u / nch - int64_t(c) * u / nch));
    // (measured defaults, profiles/r02_ab_ring.txt: the d-linear rows leave the B warps little to do)
    const int na_default = op->rg_tensor ? 8 : op->rg_nsmax <= 3 ? 7 : 5;
    const int NA = std::min(std::max(ring_na > 0 ? ring_na : na_default, 1), RG_NW - RG_NS);
    const int bpitch = (L * op->rg_nymax) | 1;
    int tpitch = op->rg_nsmax * NP;
    while (tpitch % 4 != 2) ++tpitch;  // 16-byte accesses of consecutive lanes conflict-free
    const int64_t boxd = (int64_t(cmax) * bpitch + 1) & ~int64_t(1), trd = int64_t(cmax) * tpitch;
    const void* kfn = op->rg_tensor ? reinterpret_cast<const void*>(ring_interp_kernel<1>)
                      : L == 5      ? reinterpret_cast<const void*>(ring_interp_kernel<3>)
                                    : reinterpret_cast<const void*>(ring_interp_kernel<2>);
    int per_sm = 0;
    const size_t fixed = 8 * (size_t(ring_fixed_doubles(op->dev.G1)) + (RG_DIRECT ? 0 : size_t(NA) * 2 * boxd));
    TH_CUDA(resident_ctas(kfn, RG_NTH, fixed + 8 * size_t(trd) * (L + 1), &per_sm));
    cudaFuncAttributes fa;
    TH_CUDA(cudaFuncGetAttributes(&fa, kfn));
    const int64_t avail = int64_t(fa.maxDynamicSharedSizeBytes) - int64_t(fixed);
    static const int ring_r = [] { const char* e = std::getenv("TH_RING_R"); return e ? std::atoi(e) : RG_RMAX; }();
    // the header ring (RG_NH entries, decoded RG_HAHEAD tiles ahead) must outlast the skew between
    // the leading A iterator and the slowest warp: (R + (RG_PFD + 1) NA) / L + 2 tiles of >= L slices
    const int r_hdr = (RG_NH - RG_HAHEAD - 2) * L - (RG_PFD + 1) * NA;
    const int R = int(std::min<int64_t>(std::min(std::min(ring_r, RG_RMAX), r_hdr), avail / (8 * trd)));
    // a row's L slices resident plus one being produced; a tile's slices counted by the lanes of a warp
    if (per_sm >= 1 && R >= L + 1 && op->rg_nzmax <= 32) {
      const size_t smem = fixed + 8 * size_t(trd) * R;
      const int64_t tiles = n_faces * int64_t(op->rg_ntp) * nch;
      const int tblocks = int(std::min<int64_t>(tiles, int64_t(num_sms())));
      T3Syn0 syn0;
      if (op->rg_tensor) {  // the normal rows [child][3] in slots of 4, absent children zero
        std::fill(syn0.v, syn0.v + 12, 0.0);
        const th::Group& g0 = h.groups[0][0];
        for (int c = 0; c < g0.tgtN && c < 3; ++c)
          for (int x = 0; x < 3; ++x) syn0.v[c * 4 + x] = h.rows[0][size_t(h.row_off[0][0]) + c * 3 + x];
      } else {
        std::copy(h.synth[0].begin(), h.synth[0].begin() + 12, syn0.v);
      }
      if (op->rg_tensor)
        ring_interp_kernel<1><<<tblocks, RG_NTH, smem, s>>>(op->dev, syn0, src, dst, faces, tiles, op->rg_ntp, nch,
                                                            cmax, u, NA, R, bpitch, tpitch, flag);
      else if (L == 5)
        ring_interp_kernel<3><<<tblocks, RG_NTH, smem, s>>>(op->dev, syn0, src, dst, faces, tiles, op->rg_ntp, nch,
                                                            cmax, u, NA, R, bpitch, tpitch, flag);
      else
        ring_interp_kernel<2><<<tblocks, RG_NTH, smem, s>>>(op->dev, syn0, src, dst, faces, tiles, op->rg_ntp, nch,
                                                            cmax, u, NA, R, bpitch, tpitch, flag);
      TH_CUDA(cudaGetLastError());
      return TH_OK;
    }
    return -1;  // does not fit: the caller falls through to the next kernel
  };
  const bool ring_ok = interp && op->rg_L && (use_ring & (op->rg_tensor ? 8 : op->rg_L == 5 ? 1 : 2));
  if (ring_ok && (use_ring & 4)) {
    const int32_t rc = ring_launch();
    if (rc >= 0) return rc;
  }
  if (use_tile && interp && op->ti_mode) {
    const int nt = op->ti_nt;
    const int pitch = TBOX | 1;
    const int TW = op->ti_mode == 1 ? 9 : 12;
    const size_t smem = 8 * (size_t(tile_box_offset(TW, op->dev.G0, op->dev.G1)) + size_t(2) * u * pitch);
    // exact unknown split of the flattened item index (idx < 9 u) through a 32-bit reciprocal
    const bool exact = uint64_t(9) * u * uint64_t(u) < (uint64_t(1) << 32);
    if (smem <= 220 * 1024 && exact) {
      const unsigned umag = u > 1 ? unsigned((uint64_t(1) << 32) / unsigned(u) + 1) : 0u;  // u = 1: unused
      const int64_t tiles = n_faces * int64_t(nt) * nt;
#define TH_TILEK(TENSOR, NTH, MINB)                                                                         \
  do {                                                                                                      \
    auto kfn = tile_interp_kernel<TENSOR, NTH, MINB>;                                                       \
    int per_sm = 0;                                                                                         \
    TH_CUDA(resident_ctas(reinterpret_cast<const void*>(kfn), NTH, smem, &per_sm));                        \
    const int tblocks = int(std::min<int64_t>(tiles, int64_t(num_sms()) * std::max(per_sm, 1)));          \
    kfn<<<tblocks, NTH, smem, s>>>(op->dev, src, dst, faces, tiles, nt, pitch, u, umag, flag);              \
  } while (0)
      if (op->ti_mode == 1) TH_TILEK(true, 192, 2);
      else TH_TILEK(false, 192, 2);
#undef TH_TILEK
      TH_CUDA(cudaGetLastError());
      return TH_OK;
    }
  }
  static const int use_tile3 = [] { const char* e = std::getenv("TH_TILE3"); return e ? std::atoi(e) : 1; }();
  // one spatial tile per face only: at p = 17 (3 x 3 tiles per face, overlapping boxes) the
  // warp-specialised tiles run 0.27 of the copy peak against the per-warp slide's 0.40
  if (use_tile3 && interp && op->t3_ok && op->t3_nt == 1) {
    const int nch = (u + T3PCMAX - 1) / T3PCMAX;
    int cmax = 0;
    for (int c = 0; c < nch; ++c) cmax = std::max(cmax, (c + 1) * u / nch - c * u / nch);
    const size_t smem = 8 * (size_t(tile_box_offset(12, op->dev.G0, op->dev.G1)) +
                             T3P_NBOX * size_t((cmax * T3BOX + 1) & ~1) + T3P_NT * size_t(cmax) * T3TP);
    if (smem <= 227 * 1024) {
      auto kfn = tile3p_interp_kernel;
      int per_sm = 0;
      TH_CUDA(resident_ctas(reinterpret_cast<const void*>(kfn), T3P_NTH, smem, &per_sm));
      const int nt = op->t3_nt;
      const int64_t tiles = n_faces * int64_t(nt * nt * nch);
      const int tblocks = int(std::min<int64_t>(tiles, int64_t(num_sms()) * std::max(per_sm, 1)));
      T3Syn0 syn0;
      std::copy(h.synth[0].begin(), h.synth[0].begin() + 12, syn0.v);
      kfn<<<tblocks, T3P_NTH, smem, s>>>(op->dev, syn0, src, dst, faces, tiles, nt, nch, 0, cmax, u, flag);
      TH_CUDA(cudaGetLastError());
      return TH_OK;
    }
  }
  if (ring_ok) {
    const int32_t rc = ring_launch();
    if (rc >= 0) return rc;
  }
  StageGeom sg;
  if ((use_gram & 8) && interp && tensor_fast) {
    // tensor_linear interpolation through the slice ring (gram_slide.cuh, TENSOR = true)
    auto kfn = gram_slide_kernel<2, 0, 4, true>;
    const size_t smem = size_t(4) * 3 * 9 * 32 * 8;
    const int64_t units = n_faces * int64_t(op->dev.units_per_face) * ((u + 31) / 32);
    const int gblocks = int(std::min<int64_t>((units + 3) / 4, int64_t(num_sms()) * 8));
    kfn<<<gblocks, 128, smem, s>>>(op->dev, src, dst, faces, n_faces, u, flag);
  }
  else if (gram && (use_gram & 1) && interp && h.scheme == TH_SCHEME_ORDER2) TH_GRAM(2, 0, 4);
  else if (gram && (use_gram & 1) && interp && h.scheme == TH_SCHEME_ORDER3) TH_GRAM(3, 0, 3);
  else if (gram && (use_gram & 4) && !interp && h.scheme == TH_SCHEME_ORDER3 && stage_geometry(op, u, 1, sg))
    TH_SLIDE(1, 3, false, kRestrictNCW, kRestrictNU, 1);  // persistent, one CTA per SM
  else if (gram && (use_gram & 2) && !interp && h.scheme == TH_SCHEME_ORDER3) TH_GRAM(3, 1, 3);
#undef TH_GRAM
#undef TH_SLIDE
  else if (op->r_mode == 1 && op->r_L == 3) TH_RREG(1, 3, 1, 2, 4, 8);
  else if (op->r_mode == 2 && op->r_L == 3) TH_RREG(2, 3, 1, 2, 4, 8);
  else if (op->r_mode == 1 && op->r_L == 5) TH_RREG(1, 5, 9, 2, 4, 8);
#undef TH_RREG
  // (occupancies: the largest at which each instantiation does not spill, ptxas.log)
  else if (h.fast_mode == 3 && h.fast_L0 == 3 && interp) TH_WIN(3, 3, 3, 2, 1, 0, 2);
  else if (h.fast_mode == 3 && h.fast_L0 == 5 && interp) TH_WIN(3, 5, 3, 3, 1, 0, 2);
  else if ((h.fast_mode == 2 || (h.fast_mode == 1 && h.scheme == TH_SCHEME_MATRIX_LINEAR)) && h.fast_L0 == 3 &&
           interp)
    TH_WIN(2, 3, 3, 0, 1, 0, 2);  // d-linear rows (tensor_linear; matrix_linear in factored form)
  else if (h.fast_mode == 2 && h.fast_L0 == 3 && !interp) TH_WIN(2, 3, 1, 0, 2, 0, 2);
  else if (h.fast_mode == 1 && h.fast_L0 == 3 && !interp && op->smem_ok) TH_WIN(1, 3, 1, 0, 2, op->smem_bytes, 2);
  else if (h.fast_mode == 1 && h.fast_L0 == 5 && !interp && op->smem_ok) TH_WIN(1, 5, 1, 0, 2, op->smem_bytes, 2);
  else done = false;
#undef TH_WIN
  if (done) {
  } else if (op->dev.scheme == TH_SCHEME_TENSOR_LINEAR) {
    tensor_apply_kernel<<<blocks, threads, 0, s>>>(op->dev, src, dst, faces, n_faces, u, flag);
  } else if (op->max_children <= 4) {
    dense_apply_kernel<4><<<blocks, threads, 0, s>>>(op->dev, src, dst, faces, n_faces, u, flag);
  } else if (op->max_children <= 10) {
    dense_apply_kernel<10><<<blocks, threads, 0, s>>>(op->dev, src, dst, faces, n_faces, u, flag);
  } else {
    dense_apply_kernel<28><<<blocks, threads, 0, s>>>(op->dev, src, dst, faces, n_faces, u, flag);
  }
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

int32_t th_check_finite(const double* values, int64_t n, int32_t* flag, void* stream) {
  if (n <= 0) return TH_OK;
  if (!values || !flag) return fail(TH_ERR_CONTRACT, "NULL pointer");
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
  finite_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(values, n, flag);
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

// Same-level halo copy: each face record moves an n_ext x t_ext x t_ext
// world box of cells from src[0] to dst, both addressed through their world strides.  Work
// unit = one warp per (face, eighth of the box's values); the warp reads the face record once
// and streams its eighth as x-runs (n_ext cells when the normal is x, t_ext otherwise), which
// with the pool's strides are contiguous spans of cells * u doubles in source and target.
// Four 8-byte loads in flight per lane, positions advanced incrementally (no divisions per
// value).  The first version (warp per x-run, record re-read per run) was latency bound at
// 0.77-0.80 of the copy peak: three dependent record loads per 4 KB moved.
constexpr int kCopyChunks = 8;

__global__ void __launch_bounds__(256) box_copy_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                       const th_face* __restrict__ faces, int64_t n_faces,
                                                       int n_ext, int t_ext, int u) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t units = n_faces * kCopyChunks;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < units; w += nw) {
    const th_face* fp = faces + w / kCopyChunks;
    const int c = int(w % kCopyChunks);
    const int normal = __ldg(&fp->normal);
    const int ext_x = normal == 0 ? n_ext : t_ext;
    const int ext_y = normal == 1 ? n_ext : t_ext;
    const int ext_z = normal == 2 ? n_ext : t_ext;
    const int64_t s0 = __ldg(&fp->src[0]), d0 = __ldg(&fp->dst);
    const int64_t sx = __ldg(&fp->src_stride[0]), sy = __ldg(&fp->src_stride[1]), sz = __ldg(&fp->src_stride[2]);
    const int64_t dx = __ldg(&fp->dst_stride[0]), dy = __ldg(&fp->dst_stride[1]), dz = __ldg(&fp->dst_stride[2]);
    const int n = ext_x * u;                       // values per x-run
    const int64_t total = int64_t(n) * ext_y * ext_z;
    const int64_t beg = total * c / kCopyChunks, end = total * (c + 1) / kCopyChunks;
    if (sx == u && dx == u) {
      // position of value e = beg + lane as (run r, offset j); runs are (y, z) with y fastest
      int64_t e = beg + lane;
      int64_t r = e / n;
      int j = int(e - r * n);
      int y = int(r % ext_y), z = int(r / ext_y);
      while (e < end) {
        double v[4];
        int64_t so[4], dof[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          so[i] = s0 + y * sy + z * sz + j;
          dof[i] = d0 + y * dy + z * dz + j;
          if (e + 32 * i < end) v[i] = __ldg(src + so[i]);
          j += 32;  // advance to this lane's next value
          while (j >= n) {
            j -= n;
            if (++y == ext_y) { y = 0; ++z; }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (e + 32 * i < end) dst[dof[i]] = v[i];
        e += 128;
      }
    } else {  // general strides: value e -> (run, cell, unknown)
      for (int64_t e = beg + lane; e < end; e += 32) {
        const int64_t r = e / n;
        const int j = int(e - r * n), cell = j / u, q = j - cell * u;
        const int y = int(r % ext_y), z = int(r / ext_y);
        dst[d0 + y * dy + z * dz + cell * dx + q] = __ldg(src + s0 + y * sy + z * sz + cell * sx + q);
      }
    }
  }
}

int32_t th_copy_faces(const double* src, double* dst, const th_face* faces, int64_t n_faces, int32_t n_ext,
                      int32_t t_ext, int32_t u, void* stream) {
  if (n_faces < 0) return fail(TH_ERR_CONFIG, "n_faces must be >= 0");
  if (n_faces == 0) return TH_OK;
  if (!src || !dst || !faces) return fail(TH_ERR_CONTRACT, "NULL source, target or face pointer");
  if (n_ext < 1 || t_ext < 1 || u < 1) return fail(TH_ERR_CONFIG, "box extents and u must be >= 1");
  const int64_t units = n_faces * kCopyChunks;  // one warp each
  const int blocks = int(std::min<int64_t>((units + 7) / 8, int64_t(num_sms()) * 8));
  box_copy_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, faces, n_faces, n_ext, t_ext, u);
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

// Strided box copy (multi-GPU packing / unpacking of cross-face source boxes): box b moves
// ext[0] x ext[1] x ext[2] cells (world x, y, z) of u unknowns from src + boxes[b].src to
// dst + boxes[b].dst, each side addressed through its own world strides.  Warp per (box,
// eighth of its values); when both sides keep the cells of an x-run contiguous (x stride == u)
// the run is copied as ext[0] * u consecutive doubles.
__global__ void __launch_bounds__(256) strided_box_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                          const th_box* __restrict__ boxes, int64_t n_boxes, int u) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t units = n_boxes * kCopyChunks;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < units; w += nw) {
    const th_box* bp = boxes + w / kCopyChunks;
    const int c = int(w % kCopyChunks);
    const int ex = __ldg(&bp->ext[0]), ey = __ldg(&bp->ext[1]), ez = __ldg(&bp->ext[2]);
    const int64_t s0 = __ldg(&bp->src), d0 = __ldg(&bp->dst);
    const int64_t sx = __ldg(&bp->src_stride[0]), sy = __ldg(&bp->src_stride[1]), sz = __ldg(&bp->src_stride[2]);
    const int64_t dx = __ldg(&bp->dst_stride[0]), dy = __ldg(&bp->dst_stride[1]), dz = __ldg(&bp->dst_stride[2]);
    const int64_t n = int64_t(ex) * u;  // values per x-run
    const int64_t total = n * ey * ez;
    const int64_t beg = total * c / kCopyChunks, end = total * (c + 1) / kCopyChunks;
    const bool runs = sx == u && dx == u;
    for (int64_t e = beg + lane; e < end; e += 32) {
      const int64_t r = e / n;
      const int64_t j = e - r * n;
      const int y = int(r % ey), z = int(r / ey);
      int64_t so = s0 + y * sy + z * sz, dof = d0 + y * dy + z * dz;
      if (runs) {
        so += j;
        dof += j;
      } else {
        const int64_t cell = j / u, q = j - cell * u;
        so += cell * sx + q;
        dof += cell * dx + q;
      }
      dst[dof] = __ldg(src + so);
    }
  }
}

int32_t th_copy_boxes(const double* src, double* dst, const th_box* boxes, int64_t n_boxes, int32_t u, void* stream) {
  if (n_boxes < 0) return fail(TH_ERR_CONFIG, "n_boxes must be >= 0");
  if (n_boxes == 0) return TH_OK;
  if (!src || !dst || !boxes) return fail(TH_ERR_CONTRACT, "NULL source, target or box pointer");
  if (u < 1) return fail(TH_ERR_CONFIG, "u must be >= 1");
  const int64_t units = n_boxes * kCopyChunks;
  const int blocks = int(std::min<int64_t>((units + 7) / 8, int64_t(num_sms()) * 8));
  strided_box_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, boxes, n_boxes, u);
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

int32_t th_operator_source_box(const th_operator* op, int32_t selector, int32_t* box) {
  if (!op || !box) return fail(TH_ERR_CONFIG, "NULL argument");
  const th::HostOperator& h = op->host;
  int g0a, g0b, ga[2], gb[2];
  if (h.role == 0) {
    if (selector < 0 || selector > 8) return fail(TH_ERR_CONFIG, "segment must be in [0, 8]");
    g0a = 0;
    g0b = int(h.groups[0].size());
    ga[0] = h.seg_g[selector % 3][0], gb[0] = h.seg_g[selector % 3][1];
    ga[1] = h.seg_g[selector / 3][0], gb[1] = h.seg_g[selector / 3][1];
  } else {
    if (selector < 0 || selector > 2) return fail(TH_ERR_CONFIG, "half must be TH_HALF_FULL, _INNER or _OUTER");
    g0a = h.half_g[selector][0];
    g0b = h.half_g[selector][1];
    ga[0] = ga[1] = 0;
    gb[0] = gb[1] = int(h.groups[1].size());
  }
  auto span = [](const std::vector<th::Group>& g, int a, int b, int32_t* out) {
    int lo = 1 << 30, hi = -1;
    for (int i = a; i < b; ++i) {
      lo = std::min(lo, g[i].win0);
      hi = std::max(hi, g[i].win0 + g[i].winL);
    }
    out[0] = hi > lo ? lo : 0;
    out[1] = hi > lo ? hi - lo : 0;
  };
  span(h.groups[0], g0a, g0b, box);
  span(h.groups[1], ga[0], gb[0], box + 2);
  span(h.groups[1], ga[1], gb[1], box + 4);
  return TH_OK;
}

int32_t th_memcpy_async(void* dst, const void* src, int64_t bytes, int32_t kind, void* stream) {
  if (bytes < 0) return fail(TH_ERR_CONFIG, "bytes must be >= 0");
  if (bytes == 0) return TH_OK;
  if (!src || !dst) return fail(TH_ERR_CONTRACT, "NULL pointer");
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  TH_CUDA(cudaMemcpyAsync(dst, src, size_t(bytes), k, static_cast<cudaStream_t>(stream)));
  return TH_OK;
}

int32_t th_pseudoinverse_rows(const double* a, int32_t s, int32_t n, double* w, double* cond) {
  if (!a || !w || !cond) return fail(TH_ERR_CONFIG, "NULL argument");
  if (n < 1 || s < n)
    return fail(TH_ERR_CONTRACT, "system must have rows >= cols, got (" + std::to_string(s) + ", " + std::to_string(n) + ")");
  for (int64_t i = 0; i < int64_t(s) * n; ++i)
    if (!std::isfinite(a[i])) return fail(TH_ERR_CONTRACT, "matrix entries must be finite");
  try {
    double c = 0.0;
    const std::vector<double> out = th::fit_pseudo_inverse(std::vector<double>(a, a + int64_t(s) * n), s, n, c);
    std::copy(out.begin(), out.end(), w);
    *cond = c;
  } catch (const th::Error& e) {
    return fail(map_error(e), e.what(), e.column);
  }
  return TH_OK;
}

int32_t th_copy_patch_blocks(void* dst, const void* src, int64_t n_patches, int64_t patch_elems, int64_t row_elems,
                             const int32_t* blocks, int32_t n_blocks, int32_t kind, void* stream) {
  if (n_patches <= 0 || n_blocks <= 0) return TH_OK;
  if (!dst || !src || !blocks) return fail(TH_ERR_CONTRACT, "NULL pointer");
  if (patch_elems <= 0 || row_elems <= 0 || patch_elems % row_elems)
    return fail(TH_ERR_CONFIG, "patch_elems must be a positive multiple of row_elems");
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  const size_t pitch = size_t(row_elems) * 8, rows_per_patch = size_t(patch_elems / row_elems);
  for (int b = 0; b < n_blocks; ++b) {
    const int32_t row0 = blocks[4 * b], nrows = blocks[4 * b + 1], x0 = blocks[4 * b + 2], w = blocks[4 * b + 3];
    if (row0 < 0 || nrows <= 0 || x0 < 0 || w <= 0 || x0 + w > row_elems || size_t(row0 + nrows) > rows_per_patch)
      return fail(TH_ERR_CONFIG, "block outside the patch");
    cudaMemcpy3DParms prm;
    std::memset(&prm, 0, sizeof(prm));
    prm.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), pitch, pitch, rows_per_patch);
    prm.dstPtr = make_cudaPitchedPtr(dst, pitch, pitch, rows_per_patch);
    prm.srcPos = make_cudaPos(size_t(x0) * 8, size_t(row0), 0);
    prm.dstPos = prm.srcPos;
    prm.extent = make_cudaExtent(size_t(w) * 8, size_t(nrows), size_t(n_patches));
    prm.kind = k;
    TH_CUDA(cudaMemcpy3DAsync(&prm, static_cast<cudaStream_t>(stream)));
  }
  return TH_OK;
}

// Pack / unpack the same blocks of every patch between a patch pool and a compact layout
// (per patch: the blocks back to back, each rows x width elements).  Warp per (patch, block).
__global__ void __launch_bounds__(256) patch_blocks_kernel(double* __restrict__ pool, double* __restrict__ compact,
                                                           int64_t n_patches, int64_t patch_elems, int64_t row_elems,
                                                           const int4* __restrict__ blocks, const int64_t* __restrict__ boff,
                                                           int n_blocks, int64_t compact_elems, int pack) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t units = n_patches * n_blocks;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < units; w += nw) {
    const int64_t pt = w / n_blocks;
    const int b = int(w - pt * n_blocks);
    const int4 B = __ldg(&blocks[b]);  // (row0, rows, x0, width)
    double* const pp = pool + pt * patch_elems + int64_t(B.x) * row_elems + B.z;
    double* const cp = compact + pt * compact_elems + __ldg(&boff[b]);
    const int n = B.y * B.w;
    for (int e = lane; e < n; e += 32) {
      const int r = e / B.w, c = e - r * B.w;
      if (pack) cp[e] = pp[int64_t(r) * row_elems + c];
      else pp[int64_t(r) * row_elems + c] = cp[e];
    }
  }
}

int32_t th_pool_blocks(double* pool, double* compact, int64_t n_patches, int64_t patch_elems, int64_t row_elems,
                       const int32_t* blocks, const int64_t* block_offsets, int32_t n_blocks, int64_t compact_elems,
                       int32_t pack, void* stream) {
  if (n_patches <= 0 || n_blocks <= 0) return TH_OK;
  if (!pool || !compact || !blocks || !block_offsets) return fail(TH_ERR_CONTRACT, "NULL pointer");
  const int64_t units = n_patches * n_blocks;
  const int grid = int(std::min<int64_t>((units + 7) / 8, int64_t(num_sms()) * 8));
  patch_blocks_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pool, compact, n_patches, patch_elems, row_elems, reinterpret_cast<const int4*>(blocks), block_offsets, n_blocks,
      compact_elems, pack);
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

int32_t th_operator_support_layers(const th_operator* op, int32_t* lo, int32_t* count) {
  if (!op || !lo || !count) return fail(TH_ERR_CONFIG, "NULL argument");
  int a = op->host.ax[0].ns, b = 0;
  for (const auto& g : op->host.groups[0]) {
    a = std::min(a, g.win0);
    b = std::max(b, g.win0 + g.winL);
  }
  *lo = a;
  *count = b - a;
  return TH_OK;
}

int32_t th_copy_box_layers(const double* src, double* dst, int64_t n_faces, int32_t normal, int32_t n_ext,
                           int32_t t_ext, int32_t u, int32_t lo, int32_t count, int32_t kind, void* stream) {
  if (n_faces <= 0 || count <= 0) return TH_OK;
  if (!src || !dst) return fail(TH_ERR_CONTRACT, "NULL pointer");
  if (normal < 0 || normal > 2 || lo < 0 || lo + count > n_ext || u < 1 || t_ext < 1)
    return fail(TH_ERR_CONFIG, "bad box layer selection");
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t cell = size_t(u) * sizeof(double);
  const size_t box = cell * size_t(n_ext) * t_ext * t_ext;
  if (normal == 2) {  // z slowest: the layers are one contiguous run per face
    const size_t plane = cell * size_t(t_ext) * t_ext;
    TH_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(dst) + lo * plane, box,
                              reinterpret_cast<const char*>(src) + lo * plane, box, count * plane, size_t(n_faces), k, s));
    return TH_OK;
  }
  // normal y: per face, t_ext z-planes each holding `count` contiguous rows of t_ext cells;
  // normal x: per face, t_ext^2 rows of n_ext cells of which `count` are taken
  const size_t row = normal == 1 ? cell * t_ext * n_ext : cell * n_ext;       // pitch between runs
  const size_t width = normal == 1 ? cell * t_ext * count : cell * count;     // bytes per run
  const size_t runs = normal == 1 ? size_t(t_ext) : size_t(t_ext) * t_ext;    // runs per face
  const size_t off = normal == 1 ? cell * t_ext * lo : cell * lo;
  cudaMemcpy3DParms prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.srcPtr = make_cudaPitchedPtr(const_cast<char*>(reinterpret_cast<const char*>(src)) + off, row, row, runs);
  prm.dstPtr = make_cudaPitchedPtr(reinterpret_cast<char*>(dst) + off, row, row, runs);
  prm.extent = make_cudaExtent(width, runs, size_t(n_faces));
  prm.kind = k;
  (void)box;
  TH_CUDA(cudaMemcpy3DAsync(&prm, s));
  return TH_OK;
}

int32_t th_csr_apply(const int64_t* row_offsets, const int64_t* col_indices, const double* values, int64_t n_rows,
                     const double* src, double* out, int32_t u, void* stream) {
  if (u < 1) return fail(TH_ERR_CONFIG, "u must be >= 1");
  if (n_rows <= 0) return TH_OK;
  const int blocks = int(std::min<int64_t>((n_rows + 3) / 4, int64_t(num_sms()) * 16));
  csr_apply_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(row_offsets, col_indices, values, n_rows,
                                                                         src, out, u);
  TH_CUDA(cudaGetLastError());
  return TH_OK;
}

}  // extern "C"
