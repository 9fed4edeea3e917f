// Host-side operator construction for the B200 halo path.
//
// Builds, once per (role, scheme, p, k), the "compressed block layout" the
// kernels consume:
//   * per reference axis, the target indices are grouped into runs that
//     share one source window (the stencil of taylor.py:114-140, or the
//     3-cell window holding the d-linear rows of linear.py:28-112);
//   * each (normal group, t1 group, t2 group) triple owns one dense weight
//     block  W[window cell][child];  identical blocks are stored once
//     (interior blocks repeat across the face);
//   * tensor_linear keeps the per-axis 1-D rows instead (linear.py:115-151).
// Weights are computed exactly as the reference does (Householder QR
// pseudo-inverse of the factorial-normalised design matrix, rows
// basis(delta) @ A+), so dense blocks reproduce the reference CSR rows.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace th {

enum class Err { Config = 1, Infeasible = 2, Contract = 3, Singular = 4, Cuda = 5 };

struct Error : std::runtime_error {
  Err code;
  int column;
  Error(Err c, const std::string& m, int col = -1) : std::runtime_error(m), code(c), column(col) {}
};

struct Group {
  int32_t win0, winL, tgt0, tgtN;
};

struct AxisGeom {
  int ns, nt;
  double s_org, s_sp, t_org, t_sp;
  double src_level(int i) const { return s_org + (i + 0.5) * s_sp; }
  double tgt_level(int j) const { return t_org + (j + 0.5) * t_sp; }
};

struct OneDRow {
  std::vector<int> idx;
  std::vector<double> w;
};

struct HostOperator {
  int role = 0, scheme = 0, p = 0, k = 0;
  AxisGeom ax[3];
  std::vector<Group> groups[2];  // [0] normal axis, [1] both tangential axes
  // dense blocks
  std::vector<int32_t> block_id;   // [g0][g1][g2]
  std::vector<int64_t> block_off;  // per unique block, into weights
  std::vector<int32_t> block_cp;   // child stride of the block
  std::vector<double> weights;
  // tensor_linear / matrix_linear 1-D rows (child-major over the group window)
  std::vector<int64_t> row_off[2];  // per group: offset into rows[a]
  std::vector<double> rows[2];
  // face selections
  int seg_g[3][2] = {};   // tangential group range covering segment column c
  int half_g[3][2] = {};  // normal group range of half h (interpolation: all)
  int half_t[3][2] = {};  // normal target index range of half h
  int max_items = 0;
  // fast fixed-window kernels (trihalo.cu window_kernel): every normal group
  // has window fast_L0 and <= fast_C0 children, every tangential group
  // window fast_LT and <= fast_CT children
  int fast_mode = 0;  // 0 none, 1 dense blocks, 2 tensor rows, 3 Gram-separable least squares
  int fast_L0 = 0, fast_LT = 0, fast_C0 = 0, fast_CT = 0;
  // Gram synthesis values per group: [child < 3][degree < 4] = P_a(e_child) / |P_a|^2
  // (filled for every Taylor operator whose windows are all full: gram_ok)
  std::vector<double> synth[2];
  bool gram_ok = false;
  double max_condition = 0.0;
  int n_condition_warnings = 0;
  std::vector<std::string> condition_warnings;

  int n_src_cells() const { return ax[0].ns * ax[1].ns * ax[2].ns; }
  int n_tgt_cells() const { return ax[0].nt * ax[1].nt * ax[2].nt; }
};

// schemes.py:23-47; throws Error(Infeasible) / Error(Config)
void check_feasible(int role, int scheme, int p, int k);

HostOperator build_operator(int role, int scheme, int p, int k);

// Householder QR least-squares pseudo-inverse of a full-rank tall s x n matrix (row-major),
// rank test 1e-12 (linalg.py:40-112); returns n x s row-major, throws Error(Singular).
std::vector<double> fit_pseudo_inverse(const std::vector<double>& a, int s, int n, double& cond);

// CSR-style export of a row block (segment for interpolation: -1 = full
// face; half for restriction), reference row order and column numbering.
void export_rows(const HostOperator& op, int selector, std::vector<int64_t>& row_offsets,
                 std::vector<int64_t>& cols, std::vector<double>& vals);

}  // namespace th
