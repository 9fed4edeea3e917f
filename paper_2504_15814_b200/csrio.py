"""CSR construction, row blocks and the text dump format (host side).

Reference counterparts:
  from_triplets                 csr.py:79-140   canonical CSR: sort (row, col, value),
                                                 sum duplicates in that order, drop |w| < 1e-14
  take_rows / extract_segment / csr.py:176-248   row blocks of a full-face operator
  extract_half
  dump_operator / dumps_operator / csr.py:255-287 text format: header
  load_operator                                  "n_rows n_cols nnz scheme_tag p k", then one
                                                 "row col value" line per entry (value %.17g)

These act on the host CSR view (`CsrOperator`) of the operators the C++ builder
makes (`DeviceOperator.csr()` / `operator_cache_get`); the device kernels never
see CSR.  A loaded or hand-built operator is applied on the GPU through
`apply()` (the C ABI's th_csr_apply).
"""

from __future__ import annotations

import io

import numpy as np

from . import geometry
from .errors import ConfigurationError, ContractViolationError
from .geometry import RegionShape
from .operators import CsrOperator, OperatorKey

DROP_TOLERANCE = 1e-14  # csr.py:20


def from_triplets(n_rows: int, n_cols: int, entries, scheme_tag: str = "matrix_linear",
                  built_for: OperatorKey | None = None, source_region: RegionShape | None = None,
                  target_region: RegionShape | None = None, max_condition: float = float("nan"),
                  condition_warnings: tuple = ()) -> CsrOperator:
    """Canonical CSR from (row, col, value) triplets (csr.py:79-140).

    Duplicate (row, col) entries are summed in ascending value order (so the
    result does not depend on the input order), columns are sorted within a
    row, and merged entries with |w| < 1e-14 are dropped."""
    arr = np.asarray(list(entries), dtype=object).reshape(-1, 3) if entries is not None else np.zeros((0, 3))
    rows = np.asarray(arr[:, 0], dtype=np.int64) if arr.size else np.zeros(0, np.int64)
    cols = np.asarray(arr[:, 1], dtype=np.int64) if arr.size else np.zeros(0, np.int64)
    vals = np.asarray(arr[:, 2], dtype=np.float64) if arr.size else np.zeros(0, np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= n_rows):
        raise ContractViolationError(f"row index outside [0, {n_rows})")
    if cols.size and (cols.min() < 0 or cols.max() >= n_cols):
        raise ContractViolationError(f"col index outside [0, {n_cols})")
    order = np.lexsort((vals, cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        head = np.ones(rows.size, dtype=bool)
        head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        gid = np.cumsum(head) - 1
        merged = np.zeros(int(gid[-1]) + 1)
        np.add.at(merged, gid, vals)  # sequential, in the sorted order
        rows, cols = rows[head], cols[head]
        keep = np.abs(merged) >= DROP_TOLERANCE
        rows, cols, vals = rows[keep], cols[keep], merged[keep]
    offsets = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=offsets[1:])
    return CsrOperator(int(n_rows), int(n_cols), offsets, cols, vals, scheme_tag, built_for, source_region,
                       target_region, max_condition, tuple(condition_warnings))


def take_rows(op: CsrOperator, row_ids, built_for: OperatorKey | None,
              target_region: RegionShape | None) -> CsrOperator:
    """Operator made of rows `row_ids` of `op`, in that order (csr.py:176-205)."""
    row_ids = np.asarray(row_ids, dtype=np.int64)
    starts, ends = op.row_offsets[row_ids], op.row_offsets[row_ids + 1]
    counts = ends - starts
    offsets = np.zeros(row_ids.size + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    # entry t of the new operator comes from starts[row] + (t - offsets[row])
    owner = np.repeat(np.arange(row_ids.size), counts)
    take = starts[owner] + (np.arange(offsets[-1]) - offsets[owner])
    return CsrOperator(int(row_ids.size), op.n_cols, offsets, op.col_indices[take], op.values[take], op.scheme_tag,
                       built_for, op.source_region, target_region, op.max_condition, op.condition_warnings)


def _subregion_rows(full: RegionShape, sub: RegionShape) -> np.ndarray:
    """Linear ids in `full` of the cells of `sub`, in `sub`'s x-fastest order (csr.py:208-220)."""
    shift = [int(round((sub.origin[d] - full.origin[d]) / full.spacing)) for d in range(3)]
    nx, ny, nz = sub.extents
    k2, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ids = np.stack([i.ravel() + shift[0], j.ravel() + shift[1], k2.ravel() + shift[2]])
    for d in range(3):
        if ids[d].size and (ids[d].min() < 0 or ids[d].max() >= full.extents[d]):
            raise ContractViolationError(f"sub-region outside region extents {full.extents}")
    sx, sy, sz = full.strides
    return (ids[0] * sx + ids[1] * sy + ids[2] * sz).astype(np.int64)


def extract_segment(op: CsrOperator, segment: int) -> CsrOperator:
    """Rows of fine segment `segment` (k x p x p) of a full-face interpolation operator."""
    if not 0 <= int(segment) <= 8:
        raise ConfigurationError(f"segment must be in [0, 8], got {segment}")
    key = op.built_for
    if key is None or key.role != "interpolate" or key.segment is not None:
        raise ContractViolationError("extract_segment needs a full-face interpolation operator")
    full = geometry.ref_interp_target_full(key.p, key.k)
    sub = geometry.ref_interp_target_segment(key.p, key.k, int(segment))
    return take_rows(op, _subregion_rows(full, sub),
                     OperatorKey(key.role, key.scheme, key.p, key.k, segment=int(segment)), sub)


def extract_half(op: CsrOperator, half: str) -> CsrOperator:
    """Rows of the inner / outer normal layers of a full restriction operator."""
    if half not in ("inner", "outer"):
        raise ConfigurationError(f"half must be 'inner' or 'outer', got {half!r}")
    key = op.built_for
    if key is None or key.role != "restrict" or key.half is not None:
        raise ContractViolationError("extract_half needs a full-target restriction operator")
    full = geometry.ref_restrict_target(key.p, key.k, None)
    sub = geometry.ref_restrict_target(key.p, key.k, half)
    return take_rows(op, _subregion_rows(full, sub), OperatorKey(key.role, key.scheme, key.p, key.k, half=half), sub)


def dump_operator(op: CsrOperator, stream) -> None:
    """Write the reference's text dump of `op` (csr.py:255-263)."""
    if op.built_for is None:
        raise ContractViolationError("operator has no fingerprint; cannot dump header")
    stream.write(f"{op.n_rows} {op.n_cols} {op.nnz} {op.scheme_tag} {op.built_for.p} {op.built_for.k}\n")
    rows = np.repeat(np.arange(op.n_rows), np.diff(op.row_offsets))
    stream.write("".join(f"{r} {c} {v:.17g}\n" for r, c, v in zip(rows.tolist(), op.col_indices.tolist(),
                                                                    op.values.tolist())))


def dumps_operator(op: CsrOperator) -> str:
    buf = io.StringIO()
    dump_operator(op, buf)
    return buf.getvalue()


def load_operator(stream):
    """Parse a dump; returns (operator, p, k).  The role is not recorded in the format."""
    header = stream.readline().split()
    if len(header) != 6:
        raise ContractViolationError("dump header must be 'n_rows n_cols nnz scheme_tag p k'")
    n_rows, n_cols, nnz = int(header[0]), int(header[1]), int(header[2])
    scheme_tag, p, k = header[3], int(header[4]), int(header[5])
    entries = []
    for line in stream:
        parts = line.split()
        if not parts:
            continue
        if len(parts) != 3:
            raise ContractViolationError(f"dump entry must be 'row col value', got {line.strip()!r}")
        entries.append((int(parts[0]), int(parts[1]), float(parts[2])))
    if len(entries) != nnz:
        raise ContractViolationError(f"dump announced {nnz} entries, found {len(entries)}")
    return from_triplets(n_rows, n_cols, entries, scheme_tag=scheme_tag), p, k
