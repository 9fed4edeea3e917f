"""Oracle restatement of reference operator construction (TEST INFRASTRUCTURE ONLY).

Each function follows the reference file:line named in its docstring.  The
arithmetic is performed with the same NumPy operations in the same order as
the reference so that, on one machine, the CSR arrays come out bit-identical
(checked against golden fixtures made by the real reference, see
tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import geometry as G

DROP_TOLERANCE = 1e-14          # csr.py:20
RANK_TOLERANCE = 1e-12          # linalg.py:18
STENCIL_BLOCK = {2: 3, 3: 5}    # taylor.py:28
STENCIL_MARGIN = 3              # taylor.py:29


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    scheme: str = ""
    max_condition: float = float("nan")
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d

    def take_rows(self, rows: np.ndarray) -> "Csr":
        """Row subset in the given order (csr.py:176-201)."""
        counts = self.row_offsets[rows + 1] - self.row_offsets[rows]
        off = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        take = (np.concatenate([np.arange(self.row_offsets[r], self.row_offsets[r + 1]) for r in rows])
                if rows.size else np.zeros(0, dtype=np.int64))
        return Csr(int(rows.size), self.n_cols, off, self.col_indices[take], self.values[take],
                   self.scheme, self.max_condition, dict(self.meta))


def canonical_csr(n_rows, n_cols, rows, cols, vals, scheme="", max_condition=float("nan")) -> Csr:
    """Canonical CSR from triplets: lexsort (row, col, value), merge in that
    order, drop |w| < 1e-14 (csr.py:79-140)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((vals, cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        first = np.ones(rows.size, dtype=bool)
        first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        grp = np.cumsum(first) - 1
        merged = np.zeros(int(grp[-1]) + 1)
        np.add.at(merged, grp, vals)
        rows, cols = rows[first], cols[first]
        keep = np.abs(merged) >= DROP_TOLERANCE
        rows, cols, merged = rows[keep], cols[keep], merged[keep]
    else:
        merged = vals
    off = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(off, rows + 1, 1)
    off = np.cumsum(off)
    return Csr(n_rows, n_cols, off, cols, merged, scheme, max_condition)


# ---------------------------------------------------------------------------
# d-linear pieces (linear.py)
# ---------------------------------------------------------------------------

def lin_row(levels: np.ndarray, x: float):
    """Two-point linear row with constant-slope extrapolation (linear.py:28-47)."""
    n = levels.size
    if n == 1:
        return np.array([0]), np.array([1.0])
    hi = int(np.searchsorted(levels, x))
    a, b = (0, 1) if hi <= 0 else ((n - 2, n - 1) if hi >= n else (hi - 1, hi))
    t = (x - levels[a]) / (levels[b] - levels[a])
    return np.array([a, b]), np.array([1.0 - t, t])


def _as_matrix(rows, ncols):
    m = np.zeros((len(rows), ncols))
    for r, (idx, w) in enumerate(rows):
        m[r, idx] += w
    return m


def coarse_tangential_levels(p):
    return (np.arange(p) + 0.5) * 3.0           # linear.py:50-51


def coarse_normal_levels(k):
    return (np.arange(2 * k) + 0.5 - k) * 3.0   # linear.py:54-55


def fine_normal_levels(k):
    return np.arange(2 * k) + 0.5 - k           # linear.py:58-59


def axis_tangential(p):
    """3p x p (linear.py:69-75)."""
    lv = coarse_tangential_levels(p)
    return _as_matrix([lin_row(lv, m + 0.5) for m in range(3 * p)], p)


def axis_normal(k):
    """k x 2k (linear.py:78-84)."""
    lv = coarse_normal_levels(k)
    return _as_matrix([lin_row(lv, i + 0.5) for i in range(k)], 2 * k)


def restrict_axis_tangential(p):
    """p x 3p child means (linear.py:87-92)."""
    m = np.zeros((p, 3 * p))
    for j in range(p):
        m[j, 3 * j:3 * j + 3] = 1.0 / 3.0
    return m


def restrict_axis_normal(k):
    """k x 2k: child mean where the three children exist, else linear
    continuation from the fine layers (linear.py:95-112)."""
    lv = fine_normal_levels(k)
    rows = []
    for j in range(k):
        lo = k + 3 * j
        if lo + 2 < 2 * k:
            rows.append((np.array([lo, lo + 1, lo + 2]), np.full(3, 1.0 / 3.0)))
        else:
            rows.append(lin_row(lv, (j + 0.5) * 3.0))
    return _as_matrix(rows, 2 * k)


def tensor_contract(mx, my, mz, grid):
    """Three per-axis matmuls with transposed copies (linear.py:115-151)."""
    nz, ny, nx, u = grid.shape
    ax, ay, az = mx.shape[0], my.shape[0], mz.shape[0]
    t1 = np.matmul(mx, grid.reshape(nz * ny, nx, u))
    t1c = np.ascontiguousarray(t1.reshape(nz, ny, ax, u).transpose(0, 2, 1, 3))
    t2 = np.matmul(my, t1c)
    t2c = np.ascontiguousarray(t2.transpose(1, 2, 0, 3))
    t3 = np.matmul(mz, t2c)
    return np.ascontiguousarray(t3.transpose(2, 1, 0, 3))


def segment_slices(p, s):
    sy, sz = (s % 3) * p, (s // 3) * p
    return slice(sy, sy + p), slice(sz, sz + p)


def half_slice(k, half):
    if half is None:
        return slice(0, k)
    lo = G.inner_layers(k)
    return slice(0, lo) if half == "inner" else slice(lo, k)


def collapse_linear(p, k, role) -> Csr:
    """matrix_linear: triple product of the 1-D rows (linear.py:202-240)."""
    if role == "interpolate":
        src, tgt = G.ref_interp_source(p, k), G.ref_interp_target_full(p, k)
        xr = [lin_row(coarse_normal_levels(k), i + 0.5) for i in range(k)]
        tr = [lin_row(coarse_tangential_levels(p), m + 0.5) for m in range(3 * p)]
    else:
        src, tgt = G.ref_restrict_source(p, k), G.ref_restrict_target(p, k, None)
        an = restrict_axis_normal(k)
        xr = [(np.flatnonzero(an[j]), an[j, np.flatnonzero(an[j])]) for j in range(k)]
        tr = [(np.arange(3 * j, 3 * j + 3), np.full(3, 1.0 / 3.0)) for j in range(p)]
    nx, ny, nz = tgt.extents
    R, C, V = [], [], []
    for k2 in range(nz):
        zi, zw = tr[k2]
        for j in range(ny):
            yi, yw = tr[j]
            for i in range(nx):
                xi, xw = xr[i]
                row = tgt.lin(i, j, k2)
                for a, wa in zip(xi, xw):
                    for b, wb in zip(yi, yw):
                        wab = wa * wb
                        for c, wc in zip(zi, zw):
                            R.append(row)
                            C.append(src.lin(a, b, c))
                            V.append(wab * wc)
    return canonical_csr(tgt.n, src.n, R, C, V, "matrix_linear")


# ---------------------------------------------------------------------------
# least squares (linalg.py)
# ---------------------------------------------------------------------------

class RankDeficient(Exception):
    def __init__(self, column):
        super().__init__(f"rank-deficient fit: column {column}")
        self.column = column


def householder(a: np.ndarray):
    """Householder QR without pivoting; vectors stored column-wise (linalg.py:40-56)."""
    r = np.array(a, dtype=np.float64, copy=True)
    s, n = r.shape
    vs = np.zeros((s, n))
    for j in range(n):
        x = r[j:, j]
        nx_ = np.linalg.norm(x)
        if nx_ == 0.0:
            continue
        v = x.copy()
        v[0] += np.copysign(nx_, x[0])
        v /= np.linalg.norm(v)
        r[j:, j:] -= 2.0 * np.outer(v, v @ r[j:, j:])
        vs[j:, j] = v
    return vs, np.triu(r[:n, :])


def apply_qt(vs, b):
    """Q^T b by successive reflections (linalg.py:59-70)."""
    out = np.array(b, dtype=np.float64, copy=True)
    sq = out.ndim == 1
    if sq:
        out = out[:, None]
    for j in range(vs.shape[1]):
        v = vs[j:, j]
        out[j:, :] -= 2.0 * np.outer(v, v @ out[j:, :])
    return out[:, 0] if sq else out


def rank_check(r) -> float:
    """Pivot test at 1e-12 * max|R_ii|; returns max/min |R_ii| (linalg.py:73-80)."""
    d = np.abs(np.diag(r))
    top = d.max(initial=0.0)
    bad = np.flatnonzero(d < RANK_TOLERANCE * top) if top > 0.0 else np.arange(d.size)
    if bad.size:
        raise RankDeficient(int(bad[0]))
    return float(top / d.min())


def back_substitute(r, b):
    """linalg.py:83-88"""
    n = r.shape[0]
    x = np.zeros_like(b)
    for i in range(n - 1, -1, -1):
        x[i] = (b[i] - r[i, i + 1:] @ x[i + 1:]) / r[i, i]
    return x


def pseudo_inverse(a):
    """A+ = R^-1 Q^T (n x s) from one factorisation (linalg.py:104-112)."""
    s, n = a.shape
    vs, r = householder(a)
    cond = rank_check(r)
    qt = apply_qt(vs, np.eye(s))
    return back_substitute(r, qt[:n, :]), cond


# ---------------------------------------------------------------------------
# Taylor / least-squares operators (taylor.py)
# ---------------------------------------------------------------------------

def basis_exponents(order):
    """Graded lexicographic (taylor.py:57-64)."""
    ex = []
    for deg in range(order + 1):
        for a in range(deg, -1, -1):
            for b in range(deg - a, -1, -1):
                ex.append((a, b, deg - a - b))
    return ex


def design(exps, pts):
    """Factorial-normalised monomials (taylor.py:42-50)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    cols = []
    for a, b, c in exps:
        norm = math.factorial(a) * math.factorial(b) * math.factorial(c)
        cols.append(pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c / norm)
    return np.stack(cols, axis=1)


def nearest_cell(t_idx, tgt: G.Region, src: G.Region):
    """Per-axis argmin, ties to the lower index (taylor.py:92-111)."""
    c = tgt.centre(t_idx)
    out = []
    for d in range(3):
        lv = src.origin[d] + (np.arange(src.extents[d]) + 0.5) * src.spacing
        out.append(int(np.argmin(np.abs(lv - c[d]))))
    return tuple(out)


def stencil_offsets(centre, src: G.Region, order):
    """Cube translated inward, clipped to the extent (taylor.py:114-140)."""
    block = STENCIL_BLOCK[order]
    ax = []
    for d in range(3):
        ext = src.extents[d]
        lv = min(block, ext)
        start = max(0, min(centre[d] - block // 2, ext - lv))
        ax.append(np.arange(start, start + lv) - centre[d])
    ox, oy, oz = np.meshgrid(ax[0], ax[1], ax[2], indexing="ij")
    return np.stack([ox, oy, oz], axis=-1).transpose(2, 1, 0, 3).reshape(-1, 3)


def taylor_full_face(p, k, order, role) -> Csr:
    """Full-face Taylor operator (taylor.py:171-219)."""
    if role == "interpolate":
        src, tgt = G.ref_interp_source(p, k), G.ref_interp_target_full(p, k)
    else:
        src, tgt = G.ref_restrict_source(p, k), G.ref_restrict_target(p, k, None)
    exps = basis_exponents(order)
    so, to = np.asarray(src.origin), np.asarray(tgt.origin)
    fits = {}
    R, C, V = [], [], []
    max_cond = 0.0
    for r in range(tgt.n):
        t_idx = tgt.unlin(r)
        c_idx = nearest_cell(t_idx, tgt, src)
        hit = fits.get(c_idx)
        if hit is None:
            offs = stencil_offsets(c_idx, src, order)
            w, cond = pseudo_inverse(design(exps, offs * 1.0))
            cells = offs + np.asarray(c_idx)
            cols = np.array([src.lin(*cell) for cell in cells], dtype=np.int64)
            hit = (w, cols, cond)
            fits[c_idx] = hit
        w, cols, cond = hit
        tc = to + (np.asarray(t_idx) + 0.5) * tgt.spacing
        cc = so + (np.asarray(c_idx) + 0.5) * src.spacing
        delta = (tc - cc) / src.spacing
        roww = design(exps, delta[None, :])[0] @ w
        R.append(np.full(cols.size, r, dtype=np.int64))
        C.append(cols)
        V.append(roww)
        max_cond = max(max_cond, cond)
    return canonical_csr(tgt.n, src.n, np.concatenate(R), np.concatenate(C), np.concatenate(V),
                         f"order{order}", max_cond)


_FULL_CACHE: dict = {}


def full_face_operator(scheme, role, p, k) -> Csr:
    key = (scheme, role, p, k)
    op = _FULL_CACHE.get(key)
    if op is None:
        if scheme == "matrix_linear":
            op = collapse_linear(p, k, role)
        elif scheme in ("order2", "order3"):
            op = taylor_full_face(p, k, int(scheme[-1]), role)
        else:
            raise ValueError(f"scheme {scheme!r} has no matrix form")
        _FULL_CACHE[key] = op
    return op


def build_operator(scheme, role, p, k, segment=None, half=None) -> Csr:
    """Row block of the cached full-face operator (taylor.py:252-308, csr.py:219-248)."""
    full = full_face_operator(scheme, role, p, k)
    if role == "interpolate" and segment is not None:
        rows = G.subregion_rows(G.ref_interp_target_full(p, k), G.ref_interp_target_segment(p, k, segment))
        return full.take_rows(rows)
    if role == "restrict" and half is not None:
        rows = G.subregion_rows(G.ref_restrict_target(p, k, None), G.ref_restrict_target(p, k, half))
        return full.take_rows(rows)
    return full
