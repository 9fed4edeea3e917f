// Host-side operator construction (see builder.hpp).  Reference behaviour
// followed, per function:
//   geometry of the reference face ......... geometry.py:202-228
//   nearest source cell (ties -> lower) .... taylor.py:92-111
//   stencil window translated inward ....... taylor.py:114-140
//   graded-lex factorial-normalised basis .. taylor.py:33-64
//   Householder QR pseudo-inverse .......... linalg.py:40-112
//   Taylor rows basis(delta) @ A+ .......... taylor.py:171-219
//   d-linear 1-D rows ...................... linear.py:28-112, collapse linear.py:202-240
//   feasibility rules + messages ........... schemes.py:23-47, taylor.py:80-89
#include "builder.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>

namespace th {

namespace {

const char* scheme_name(int s) {
  switch (s) {
    case 0: return "tensor_linear";
    case 1: return "matrix_linear";
    case 2: return "order2";
    case 3: return "order3";
  }
  return "?";
}

const char* role_name(int r) { return r == 0 ? "interpolate" : "restrict"; }

constexpr int kMaxChildren = 3;

int stencil_block(int order) { return order == 2 ? 3 : 5; }

int basis_size(int order) { return order == 2 ? 10 : 20; }

void validate_pk(int p, int k) {
  if (p < 1) throw Error(Err::Config, "p must be >= 1, got " + std::to_string(p));
  if (k < 1 || k > p)
    throw Error(Err::Config,
                "k must satisfy 1 <= k <= p, got k=" + std::to_string(k) + ", p=" + std::to_string(p));
}

std::string axis_note(int order) {
  int k_min = (order + 2) / 2;  // ceil((order + 1) / 2)
  std::ostringstream os;
  os << "order " << order << " needs at least " << order + 1
     << " source levels per axis (interpolation: p >= " << order + 1
     << " tangentially; either role: k >= " << k_min << ")";
  return os.str();
}

AxisGeom make_axis(int role, int axis, int p, int k) {
  AxisGeom g;
  if (role == 0) {  // interpolation: coarse source (2k, p, p) spacing 3, fine target (k, 3p, 3p)
    if (axis == 0) g = {2 * k, k, -3.0 * k, 3.0, 0.0, 1.0};
    else g = {p, 3 * p, 0.0, 3.0, 0.0, 1.0};
  } else {  // restriction: fine source (2k, 3p, 3p), coarse target (k, p, p) spacing 3
    if (axis == 0) g = {2 * k, k, -double(k), 1.0, 0.0, 3.0};
    else g = {3 * p, p, 0.0, 1.0, 0.0, 3.0};
  }
  return g;
}

int nearest(const AxisGeom& g, int j) {
  double c = g.tgt_level(j);
  int best = 0;
  double bd = std::fabs(g.src_level(0) - c);
  for (int i = 1; i < g.ns; ++i) {
    double d = std::fabs(g.src_level(i) - c);
    if (d < bd) { bd = d; best = i; }
  }
  return best;
}

// d-linear two-point row, constant slope beyond the ends (linear.py:28-47)
OneDRow lin_row(const std::vector<double>& lv, double x) {
  OneDRow r;
  int n = (int)lv.size();
  if (n == 1) { r.idx = {0}; r.w = {1.0}; return r; }
  int hi = int(std::lower_bound(lv.begin(), lv.end(), x) - lv.begin());
  int a, b;
  if (hi <= 0) { a = 0; b = 1; }
  else if (hi >= n) { a = n - 2; b = n - 1; }
  else { a = hi - 1; b = hi; }
  double t = (x - lv[a]) / (lv[b] - lv[a]);
  r.idx = {a, b};
  r.w = {1.0 - t, t};
  return r;
}

// per-axis 1-D rows of the d-linear operators, one per target index
std::vector<OneDRow> linear_rows(int role, int axis, int p, int k) {
  std::vector<OneDRow> rows;
  if (role == 0) {
    if (axis == 0) {
      std::vector<double> lv(2 * k);
      for (int i = 0; i < 2 * k; ++i) lv[i] = ((i + 0.5) - k) * 3.0;
      for (int i = 0; i < k; ++i) rows.push_back(lin_row(lv, i + 0.5));
    } else {
      std::vector<double> lv(p);
      for (int i = 0; i < p; ++i) lv[i] = (i + 0.5) * 3.0;
      for (int m = 0; m < 3 * p; ++m) rows.push_back(lin_row(lv, m + 0.5));
    }
  } else {
    if (axis == 0) {
      std::vector<double> lv(2 * k);
      for (int i = 0; i < 2 * k; ++i) lv[i] = (i + 0.5) - k;
      for (int j = 0; j < k; ++j) {
        int lo = k + 3 * j;
        if (lo + 2 < 2 * k) {
          OneDRow r;
          r.idx = {lo, lo + 1, lo + 2};
          r.w = {1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0};
          rows.push_back(r);
        } else {
          rows.push_back(lin_row(lv, (j + 0.5) * 3.0));
        }
      }
    } else {
      for (int j = 0; j < p; ++j) {
        OneDRow r;
        r.idx = {3 * j, 3 * j + 1, 3 * j + 2};
        r.w = {1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0};
        rows.push_back(r);
      }
    }
  }
  // the reference drops exact-zero partners only at CSR assembly; keep the
  // row as is (a zero weight contributes nothing to the dense block either)
  return rows;
}

struct Exps {
  std::vector<int> a, b, c;
  std::vector<double> norm;
};

Exps basis(int order) {
  Exps e;
  auto fact = [](int n) { double f = 1; for (int i = 2; i <= n; ++i) f *= i; return f; };
  for (int deg = 0; deg <= order; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b) {
        e.a.push_back(a);
        e.b.push_back(b);
        e.c.push_back(deg - a - b);
        e.norm.push_back(fact(a) * fact(b) * fact(deg - a - b));
      }
  return e;
}

inline double pw(double x, int e) {
  switch (e) {
    case 0: return 1.0;
    case 1: return x;
    case 2: return x * x;
  }
  return std::pow(x, double(e));
}

inline double phi(const Exps& e, int q, const double* pt) {
  return pw(pt[0], e.a[q]) * pw(pt[1], e.b[q]) * pw(pt[2], e.c[q]) / e.norm[q];
}

// Householder QR without pivoting, rank test 1e-12, A+ = R^-1 Q^T
// (linalg.py:40-112).  a is s x n row-major; returns n x s row-major.
std::vector<double> pseudo_inverse(const std::vector<double>& a, int s, int n, double& cond) {
  std::vector<double> r(a), vs(size_t(s) * n, 0.0), v(s);
  for (int j = 0; j < n; ++j) {
    double nx = 0;
    for (int i = j; i < s; ++i) nx += r[size_t(i) * n + j] * r[size_t(i) * n + j];
    nx = std::sqrt(nx);
    if (nx == 0.0) continue;
    for (int i = j; i < s; ++i) v[i] = r[size_t(i) * n + j];
    v[j] += std::copysign(nx, r[size_t(j) * n + j]);
    double nv = 0;
    for (int i = j; i < s; ++i) nv += v[i] * v[i];
    nv = std::sqrt(nv);
    for (int i = j; i < s; ++i) v[i] /= nv;
    for (int c = j; c < n; ++c) {
      double d = 0;
      for (int i = j; i < s; ++i) d += v[i] * r[size_t(i) * n + c];
      for (int i = j; i < s; ++i) r[size_t(i) * n + c] -= 2.0 * v[i] * d;
    }
    for (int i = j; i < s; ++i) vs[size_t(i) * n + j] = v[i];
  }
  double top = 0;
  for (int i = 0; i < n; ++i) top = std::max(top, std::fabs(r[size_t(i) * n + i]));
  double lo = top;
  for (int i = 0; i < n; ++i) {
    double d = std::fabs(r[size_t(i) * n + i]);
    if (top == 0.0 || d < 1e-12 * top)
      throw Error(Err::Singular, "rank-deficient fit: column " + std::to_string(i) + " has negligible pivot", i);
    lo = std::min(lo, d);
  }
  cond = top / lo;
  // Q^T = H_{n-1} ... H_0 applied to the identity
  std::vector<double> qt(size_t(s) * s, 0.0);
  for (int i = 0; i < s; ++i) qt[size_t(i) * s + i] = 1.0;
  for (int j = 0; j < n; ++j) {
    for (int c = 0; c < s; ++c) {
      double d = 0;
      for (int i = j; i < s; ++i) d += vs[size_t(i) * n + j] * qt[size_t(i) * s + c];
      for (int i = j; i < s; ++i) qt[size_t(i) * s + c] -= 2.0 * vs[size_t(i) * n + j] * d;
    }
  }
  std::vector<double> w(size_t(n) * s, 0.0);
  for (int i = n - 1; i >= 0; --i) {
    for (int c = 0; c < s; ++c) {
      double acc = qt[size_t(i) * s + c];
      for (int j = i + 1; j < n; ++j) acc -= r[size_t(i) * n + j] * w[size_t(j) * s + c];
      w[size_t(i) * s + c] = acc / r[size_t(i) * n + i];
    }
  }
  return w;
}

// window of a target index along one axis
struct Win {
  int start, len;
};

Win taylor_window(int c, int ns, int block) {
  int L = std::min(block, ns);
  int st = std::max(0, std::min(c - block / 2, ns - L));
  return {st, L};
}

// Discrete orthogonal (Gram) polynomials on the centred window points
// {-1,0,1} / {-2,...,2}, integer-valued there: the least-squares fit of
// taylor.py over a full tensor window equals the orthogonal projection onto
// total degree <= order, whatever basis spans that space, so the kernels
// project with these (diagonal normal matrix) instead of applying A+.
double gram_value(int L, int a, double e) {
  switch (a) {
    case 0: return 1.0;
    case 1: return e;
    case 2: return L == 3 ? 3.0 * e * e - 2.0 : e * e - 2.0;
  }
  return (5.0 * e * e * e - 17.0 * e) / 6.0;
}

double gram_norm(int L, int a) {
  static const double n3[3] = {3.0, 2.0, 6.0};
  static const double n5[4] = {5.0, 10.0, 14.0, 10.0};
  return L == 3 ? n3[a] : n5[a];
}

void choose_fast_path(HostOperator& op) {
  const bool interp = op.role == 0;
  const int L = op.scheme == 3 ? 5 : 3;
  const int C0 = 3, CT = interp ? 3 : 1;
  auto axis_ok = [&](const std::vector<Group>& gr, int Lw, int Cmax) {
    for (const Group& g : gr)
      if (g.winL != Lw || g.tgtN > Cmax) return false;
    return true;
  };
  if (!axis_ok(op.groups[0], L, C0) || !axis_ok(op.groups[1], L, CT)) return;
  op.fast_L0 = op.fast_LT = L;
  op.fast_C0 = C0;
  op.fast_CT = CT;
  if (op.scheme == 0) {
    op.fast_mode = 2;
  }
  if (op.scheme >= 2) {  // Gram synthesis tables for both roles (full windows checked above)
    op.gram_ok = true;
    const int order = op.scheme;
    for (int a = 0; a < 2; ++a) {
      const AxisGeom& g = op.ax[a];
      for (const Group& gr : op.groups[a]) {
        const double mid = g.src_level(gr.win0 + (L - 1) / 2);
        for (int c = 0; c < 3; ++c)
          for (int d = 0; d < 4; ++d) {
            double v = 0.0;
            if (c < gr.tgtN && d <= order) v = gram_value(L, d, (g.tgt_level(gr.tgt0 + c) - mid) / g.s_sp) / gram_norm(L, d);
            op.synth[a].push_back(v);
          }
      }
    }
  }
  if (op.scheme == 0) {
  } else if (interp && op.scheme >= 2) {
    op.fast_mode = 3;
  } else {
    // dense blocks are laid out with the real child counts: the fixed-window
    // kernel indexes them as C0 x CT x CT, so every group must be full
    for (const Group& g : op.groups[0])
      if (g.tgtN != C0) return;
    for (const Group& g : op.groups[1])
      if (g.tgtN != CT) return;
    op.fast_mode = 1;
  }
}

}  // namespace

std::vector<double> fit_pseudo_inverse(const std::vector<double>& a, int s, int n, double& cond) {
  return pseudo_inverse(a, s, n, cond);
}

void check_feasible(int role, int scheme, int p, int k) {
  if (scheme < 0 || scheme > 3)
    throw Error(Err::Config, "unknown scheme " + std::to_string(scheme) +
                                 "; expected one of ('tensor_linear', 'matrix_linear', 'order2', 'order3')");
  if (role != 0 && role != 1)
    throw Error(Err::Config, "role must be 'interpolate' or 'restrict', got " + std::to_string(role));
  validate_pk(p, k);
  if (scheme < 2) return;
  int order = scheme;
  int block = stencil_block(order);
  int ext[3] = {2 * k, role == 0 ? p : 3 * p, role == 0 ? p : 3 * p};
  long s = 1;
  for (int d = 0; d < 3; ++d) {
    int levels = std::min(block, ext[d]);
    if (levels < order + 1) {
      std::ostringstream os;
      os << scheme_name(scheme) << " " << role_name(role) << " infeasible at p=" << p << ", k=" << k
         << ": an axis offers only " << ext[d] << " source cells; " << axis_note(order);
      throw Error(Err::Infeasible, os.str());
    }
    s *= levels;
  }
  long need = basis_size(order) + 3;
  if (s < need) {
    std::ostringstream os;
    os << scheme_name(scheme) << " " << role_name(role) << " infeasible at p=" << p << ", k=" << k
       << ": stencil " << s << " < " << need;
    throw Error(Err::Infeasible, os.str());
  }
}

HostOperator build_operator(int role, int scheme, int p, int k) {
  check_feasible(role, scheme, p, k);
  HostOperator op;
  op.role = role;
  op.scheme = scheme;
  op.p = p;
  op.k = k;
  for (int d = 0; d < 3; ++d) op.ax[d] = make_axis(role, d, p, k);

  const bool taylor = scheme >= 2;
  const int block = taylor ? stencil_block(scheme) : 3;

  // per axis (0 normal, 1 tangential): centre, window, 1-D linear rows
  std::vector<int> centre[2];
  std::vector<Win> win[2];
  std::vector<OneDRow> lrows[2];
  for (int a = 0; a < 2; ++a) {
    const AxisGeom& g = op.ax[a];
    if (!taylor) lrows[a] = linear_rows(role, a, p, k);
    for (int j = 0; j < g.nt; ++j) {
      int c = nearest(g, j);
      Win w = taylor_window(c, g.ns, block);
      if (!taylor) {  // stretch to hold the 1-D row support
        int lo = w.start, hi = w.start + w.len;
        for (int i : lrows[a][j].idx) { lo = std::min(lo, i); hi = std::max(hi, i + 1); }
        w = {lo, hi - lo};
      }
      centre[a].push_back(c);
      win[a].push_back(w);
    }
    // groups: runs of equal windows (window start is monotone in the target index),
    // at most kMaxChildren targets each so a block has <= 27 children
    std::vector<Group>& gr = op.groups[a];
    for (int j = 0; j < g.nt; ++j) {
      if (!gr.empty() && gr.back().win0 == win[a][j].start && gr.back().winL == win[a][j].len &&
          gr.back().tgtN < kMaxChildren) {
        gr.back().tgtN++;
      } else {
        gr.push_back({win[a][j].start, win[a][j].len, j, 1});
      }
    }
  }

  // face selections
  const int G0 = (int)op.groups[0].size(), G1 = (int)op.groups[1].size();
  auto range_of = [](const std::vector<Group>& gr, int lo, int hi, int* out) {
    int a = -1, b = -1;
    for (int g = 0; g < (int)gr.size(); ++g) {
      int t0 = gr[g].tgt0, t1 = gr[g].tgt0 + gr[g].tgtN;
      if (t1 > lo && t0 < hi) { if (a < 0) a = g; b = g + 1; }
    }
    if (a < 0) { a = 0; b = 0; }
    out[0] = a;
    out[1] = b;
  };
  if (role == 0) {
    for (int c = 0; c < 3; ++c) range_of(op.groups[1], c * p, (c + 1) * p, op.seg_g[c]);
    for (int h = 0; h < 3; ++h) {
      op.half_g[h][0] = 0; op.half_g[h][1] = G0;
      op.half_t[h][0] = 0; op.half_t[h][1] = k;
    }
    int m = 0;
    for (int c1 = 0; c1 < 3; ++c1)
      for (int c2 = 0; c2 < 3; ++c2)
        m = std::max(m, G0 * (op.seg_g[c1][1] - op.seg_g[c1][0]) * (op.seg_g[c2][1] - op.seg_g[c2][0]));
    op.max_items = m;
  } else {
    int inner = (k + 1) / 2;
    int lay[3][2] = {{0, k}, {0, inner}, {inner, k}};
    for (int h = 0; h < 3; ++h) {
      op.half_t[h][0] = lay[h][0];
      op.half_t[h][1] = lay[h][1];
      range_of(op.groups[0], lay[h][0], lay[h][1], op.half_g[h]);
    }
    for (int c = 0; c < 3; ++c) { op.seg_g[c][0] = 0; op.seg_g[c][1] = G1; }
    op.max_items = (op.half_g[0][1] - op.half_g[0][0]) * G1 * G1;
  }

  // 1-D rows over group windows (tensor_linear, and the matrix_linear blocks)
  if (!taylor) {
    for (int a = 0; a < 2; ++a) {
      for (const Group& g : op.groups[a]) {
        op.row_off[a].push_back((int64_t)op.rows[a].size());
        for (int i = 0; i < g.tgtN; ++i) {
          std::vector<double> r(g.winL, 0.0);
          const OneDRow& lr = lrows[a][g.tgt0 + i];
          for (size_t t = 0; t < lr.idx.size(); ++t) r[lr.idx[t] - g.win0] += lr.w[t];
          op.rows[a].insert(op.rows[a].end(), r.begin(), r.end());
        }
      }
    }
  }

  // dense blocks (matrix schemes; tensor_linear also gets them so rows can be exported)
  const Exps ex = taylor ? basis(scheme) : Exps();
  const int nb = taylor ? basis_size(scheme) : 0;
  struct Fit {
    std::vector<double> w;  // n x s
    double cond;
  };
  std::map<std::vector<int>, Fit> fits;  // key: per-axis (window start - centre, window length)
  std::map<std::string, int> uniq;
  op.block_id.assign(size_t(G0) * G1 * G1, -1);
  for (int g0 = 0; g0 < G0; ++g0)
    for (int g2 = 0; g2 < G1; ++g2)
      for (int g1 = 0; g1 < G1; ++g1) {
        const Group* gg[3] = {&op.groups[0][g0], &op.groups[1][g1], &op.groups[1][g2]};
        const int L0 = gg[0]->winL, L1 = gg[1]->winL, L2 = gg[2]->winL;
        const int C0 = gg[0]->tgtN, C1 = gg[1]->tgtN, C2 = gg[2]->tgtN;
        const int S = L0 * L1 * L2, C = C0 * C1 * C2, CP = (C + 1) & ~1;
        std::vector<double> W(size_t(S) * CP, 0.0);
        for (int i2 = 0; i2 < C2; ++i2)
          for (int i1 = 0; i1 < C1; ++i1)
            for (int i0 = 0; i0 < C0; ++i0) {
              const int child = i0 + C0 * (i1 + C1 * i2);
              const int t[3] = {gg[0]->tgt0 + i0, gg[1]->tgt0 + i1, gg[2]->tgt0 + i2};
              if (taylor) {
                int c[3] = {centre[0][t[0]], centre[1][t[1]], centre[1][t[2]]};
                std::vector<int> key = {gg[0]->win0 - c[0], L0, gg[1]->win0 - c[1], L1, gg[2]->win0 - c[2], L2};
                auto it = fits.find(key);
                if (it == fits.end()) {
                  std::vector<double> A(size_t(S) * nb);
                  for (int z = 0; z < L2; ++z)
                    for (int y = 0; y < L1; ++y)
                      for (int x = 0; x < L0; ++x) {
                        double off[3] = {double(gg[0]->win0 + x - c[0]), double(gg[1]->win0 + y - c[1]),
                                         double(gg[2]->win0 + z - c[2])};
                        int cell = x + L0 * (y + L1 * z);
                        for (int q = 0; q < nb; ++q) A[size_t(cell) * nb + q] = phi(ex, q, off);
                      }
                  Fit f;
                  f.w = pseudo_inverse(A, S, nb, f.cond);
                  it = fits.emplace(key, std::move(f)).first;
                }
                const Fit& f = it->second;
                double delta[3];
                for (int d = 0; d < 3; ++d) {
                  const AxisGeom& g = op.ax[d == 0 ? 0 : d];
                  delta[d] = (g.tgt_level(t[d]) - g.src_level(c[d])) / g.s_sp;
                }
                double ph[20];
                for (int q = 0; q < nb; ++q) ph[q] = phi(ex, q, delta);
                for (int cell = 0; cell < S; ++cell) {
                  double acc = 0;
                  for (int q = 0; q < nb; ++q) acc += ph[q] * f.w[size_t(q) * S + cell];
                  W[size_t(cell) * CP + child] = acc;
                }
              } else {
                const OneDRow* r[3] = {&lrows[0][t[0]], &lrows[1][t[1]], &lrows[1][t[2]]};
                for (size_t a0 = 0; a0 < r[0]->idx.size(); ++a0)
                  for (size_t a1 = 0; a1 < r[1]->idx.size(); ++a1) {
                    double wab = r[0]->w[a0] * r[1]->w[a1];
                    for (size_t a2 = 0; a2 < r[2]->idx.size(); ++a2) {
                      int x = r[0]->idx[a0] - gg[0]->win0, y = r[1]->idx[a1] - gg[1]->win0,
                          z = r[2]->idx[a2] - gg[2]->win0;
                      W[size_t(x + L0 * (y + L1 * z)) * CP + child] += wab * r[2]->w[a2];
                    }
                  }
              }
            }
        std::string key(reinterpret_cast<const char*>(W.data()), W.size() * sizeof(double));
        key += std::to_string(S) + "/" + std::to_string(CP);
        auto it = uniq.find(key);
        int id;
        if (it == uniq.end()) {
          id = (int)op.block_off.size();
          uniq.emplace(std::move(key), id);
          op.block_off.push_back((int64_t)op.weights.size());
          op.block_cp.push_back(CP);
          op.weights.insert(op.weights.end(), W.begin(), W.end());
        } else {
          id = it->second;
        }
        op.block_id[(size_t(g0) * G1 + g1) * G1 + g2] = id;
      }
  for (auto& kv : fits) {
    op.max_condition = std::max(op.max_condition, kv.second.cond);
    if (kv.second.cond > 1e12) {
      op.n_condition_warnings++;
      std::ostringstream os;
      os << "derivative fit condition_estimate " << kv.second.cond
         << " exceeds 1e+12; operator accuracy may floor well above machine precision";
      op.condition_warnings.push_back(os.str());
    }
  }
  if (!taylor) op.max_condition = std::nan("");
  choose_fast_path(op);
  return op;
}

void export_rows(const HostOperator& op, int selector, std::vector<int64_t>& row_offsets, std::vector<int64_t>& cols,
                 std::vector<double>& vals) {
  int lo[3], hi[3];
  if (op.role == 0) {
    lo[0] = 0;
    hi[0] = op.k;
    if (selector < 0) {
      lo[1] = lo[2] = 0;
      hi[1] = hi[2] = 3 * op.p;
    } else {
      if (selector > 8) throw Error(Err::Config, "segment must be in [0, 8], got " + std::to_string(selector));
      lo[1] = (selector % 3) * op.p;
      lo[2] = (selector / 3) * op.p;
      hi[1] = lo[1] + op.p;
      hi[2] = lo[2] + op.p;
    }
  } else {
    if (selector < 0 || selector > 2) throw Error(Err::Config, "half selector must be 0, 1 or 2");
    lo[0] = op.half_t[selector][0];
    hi[0] = op.half_t[selector][1];
    lo[1] = lo[2] = 0;
    hi[1] = hi[2] = op.p;
  }
  const int G1 = (int)op.groups[1].size();
  auto find = [](const std::vector<Group>& gr, int t) {
    for (int g = 0; g < (int)gr.size(); ++g)
      if (t >= gr[g].tgt0 && t < gr[g].tgt0 + gr[g].tgtN) return g;
    return -1;
  };
  const int ns0 = op.ax[0].ns, ns1 = op.ax[1].ns;
  row_offsets.assign(1, 0);
  cols.clear();
  vals.clear();
  for (int t2 = lo[2]; t2 < hi[2]; ++t2)
    for (int t1 = lo[1]; t1 < hi[1]; ++t1)
      for (int t0 = lo[0]; t0 < hi[0]; ++t0) {
        int g[3] = {find(op.groups[0], t0), find(op.groups[1], t1), find(op.groups[1], t2)};
        const Group* gg[3] = {&op.groups[0][g[0]], &op.groups[1][g[1]], &op.groups[1][g[2]]};
        int id = op.block_id[(size_t(g[0]) * G1 + g[1]) * G1 + g[2]];
        const double* W = op.weights.data() + op.block_off[id];
        int CP = op.block_cp[id];
        int C0 = gg[0]->tgtN, C1 = gg[1]->tgtN;
        int child = (t0 - gg[0]->tgt0) + C0 * ((t1 - gg[1]->tgt0) + C1 * (t2 - gg[2]->tgt0));
        int L0 = gg[0]->winL, L1 = gg[1]->winL, L2 = gg[2]->winL;
        for (int z = 0; z < L2; ++z)
          for (int y = 0; y < L1; ++y)
            for (int x = 0; x < L0; ++x) {
              double w = W[size_t(x + L0 * (y + L1 * z)) * CP + child];
              if (std::fabs(w) < 1e-14) continue;
              int a0 = gg[0]->win0 + x, a1 = gg[1]->win0 + y, a2 = gg[2]->win0 + z;
              cols.push_back(a0 + (int64_t)ns0 * (a1 + (int64_t)ns1 * a2));
              vals.push_back(w);
            }
        row_offsets.push_back((int64_t)cols.size());
      }
}

}  // namespace th
