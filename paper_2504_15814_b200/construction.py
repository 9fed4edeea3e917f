"""Host-side construction API of the reference, for drop-in callers.

The reference exports its operator-construction internals at top level
(/root/reference/pkg/src/trihalo/__init__.py:37-51): the d-linear axis
operators and their collapse (linear.py:22-112, 171-245) and the Taylor
least-squares pieces (taylor.py:33-232).  Here:

* the operators themselves come from the C++ builder (csrc/builder.cpp)
  through the operator cache — ``collapse_to_matrix``, ``build_interpolation``
  and ``build_restriction`` return the same CSR rows the reference builds
  (``matrix_linear`` bit for bit, Taylor rows within 1e-12 of the row maximum,
  tests/test_builder.py, tests/test_construction.py);
* ``apply_tensor_interpolate`` / ``apply_tensor_restrict`` run on the device
  (the tensor_linear kernels of th_apply_faces);
* the small pieces a caller can inspect (axis matrices, Taylor basis,
  nearest source cell, stencil selection, derivative fit) are restated here,
  the fit through the builder's own QR (``th_pseudoinverse_rows``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native, geometry
from .errors import ConfigurationError, ContractViolationError, StencilInfeasibleError
from .geometry import FaceConfig, HaloBuffer, RegionShape
from .operators import DEFAULT_CACHE, CsrOperator, OperatorKey

STENCIL_BLOCK = {2: 3, 3: 5}     # cube edge of a Taylor stencil per order (taylor.py:27)
STENCIL_MARGIN = 3               # cells beyond the basis size a stencil must hold (taylor.py:28)
CONDITION_WARN_THRESHOLD = 1e12  # taylor.py:29


# ---------------------------------------------------------------------------
# d-linear axis operators (linear.py:22-112)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class AxisOperator:
    kind: str  # 'tangential' | 'normal' | 'restrict_tangential' | 'restrict_normal'
    matrix: np.ndarray


def _linear_weights(levels: np.ndarray, x: float):
    """Two-point linear row at x over sorted levels: the bracketing pair inside, the outermost
    pair's line outside (constant slope), a single level -> weight 1."""
    if levels.size == 1:
        return np.array([0]), np.array([1.0])
    j = int(np.searchsorted(levels, x))
    a = min(max(j - 1, 0), levels.size - 2)
    t = (x - levels[a]) / (levels[a + 1] - levels[a])
    return np.array([a, a + 1]), np.array([1.0 - t, t])


def interp_row_1d(levels: np.ndarray, x: float):
    """(indices, weights) of the linear row at x over sorted levels (linear.py:28-47)."""
    return _linear_weights(np.asarray(levels, dtype=np.float64), x)


def _matrix(rows, n_cols: int) -> np.ndarray:
    m = np.zeros((len(rows), n_cols))
    for r, (idx, w) in enumerate(rows):
        m[r, idx] += w
    return m


def build_axis_tangential(p: int) -> AxisOperator:
    """3p x p: fine tangential centres (m + 1/2) from coarse centres 3 (j + 1/2)."""
    if p < 1:
        raise ConfigurationError(f"p must be >= 1, got {p}")
    lv = 3.0 * (np.arange(p) + 0.5)
    return AxisOperator("tangential", _matrix([_linear_weights(lv, m + 0.5) for m in range(3 * p)], p))


def build_axis_normal(k: int) -> AxisOperator:
    """k x 2k: fine halo layers (i + 1/2) from the 2k coarse layers 3 (j + 1/2 - k)."""
    if k < 1:
        raise ConfigurationError(f"k must be >= 1, got {k}")
    lv = 3.0 * (np.arange(2 * k) + 0.5 - k)
    return AxisOperator("normal", _matrix([_linear_weights(lv, i + 0.5) for i in range(k)], 2 * k))


def build_restrict_axis_tangential(p: int) -> AxisOperator:
    """p x 3p: mean of the three fine children of every coarse cell."""
    m = np.zeros((p, 3 * p))
    for j in range(p):
        m[j, 3 * j:3 * j + 3] = 1.0 / 3.0
    return AxisOperator("restrict_tangential", m)


def build_restrict_axis_normal(k: int) -> AxisOperator:
    """k x 2k: a coarse halo layer whose three fine children lie in the 2k source layers
    takes their mean; deeper layers continue the fine profile linearly."""
    lv = np.arange(2 * k) + 0.5 - k
    rows = []
    for j in range(k):
        first = k + 3 * j
        if first + 2 < 2 * k:
            rows.append((np.arange(first, first + 3), np.full(3, 1.0 / 3.0)))
        else:
            rows.append(_linear_weights(lv, 3.0 * (j + 0.5)))
    return AxisOperator("restrict_normal", _matrix(rows, 2 * k))


def apply_tensor_interpolate(cfg: FaceConfig, coarse: HaloBuffer, work: dict | None = None) -> HaloBuffer:
    """linear.py:171-183 on the device: the tensor_linear interpolation kernel.  ``work`` is
    accepted for signature compatibility (device buffers are cached per exchange)."""
    from .schemes import interpolate_halo

    return interpolate_halo(cfg, "tensor_linear", coarse)


def apply_tensor_restrict(cfg: FaceConfig, fine: HaloBuffer, half: str | None = None,
                          work: dict | None = None) -> HaloBuffer:
    """linear.py:186-199 on the device: the tensor_linear restriction kernel."""
    from .schemes import restrict_halo

    return restrict_halo(cfg, "tensor_linear", fine, half=half)


def _check_role(role: str) -> None:
    if role not in ("interpolate", "restrict"):
        raise ConfigurationError(f"role must be 'interpolate' or 'restrict', got {role!r}")


def collapse_to_matrix(cfg: FaceConfig, role: str) -> CsrOperator:
    """Full-face CSR of the d-linear product (linear.py:202-245), from the C++ builder."""
    _check_role(role)
    return DEFAULT_CACHE.get(OperatorKey(role, "matrix_linear", cfg.p, cfg.k))


# ---------------------------------------------------------------------------
# Taylor least-squares pieces (taylor.py:33-232)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class TaylorBasis:
    """Monomials x^a y^b z^c / (a! b! c!) of total degree <= order, graded lexicographic."""

    order: int
    exponents: tuple

    @property
    def n(self) -> int:
        return len(self.exponents)

    def design(self, points) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
        out = np.empty((pts.shape[0], self.n))
        for q, (a, b, c) in enumerate(self.exponents):
            scale = math.factorial(a) * math.factorial(b) * math.factorial(c)
            out[:, q] = pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c / scale
        return out

    def evaluate_point(self, delta) -> np.ndarray:
        return self.design(np.asarray(delta, dtype=np.float64)[None, :])[0]


def taylor_basis(order: int) -> TaylorBasis:
    if order not in (2, 3):
        raise ConfigurationError(f"order must be 2 or 3, got {order}")
    exps = tuple((a, b, d - a - b) for d in range(order + 1) for a in range(d, -1, -1)
                 for b in range(d - a, -1, -1))
    return TaylorBasis(order, exps)


@dataclass(frozen=True)
class StencilSpec:
    centre: tuple
    offsets: np.ndarray  # (s, 3) integer offsets from the centre, x fastest

    @property
    def s(self) -> int:
        return self.offsets.shape[0]


@dataclass(frozen=True)
class DerivativeFit:
    stencil: StencilSpec
    weights: np.ndarray  # (n, s): scaled derivatives as weights on the stencil values
    condition_estimate: float


def _requirement(order: int) -> str:
    return (f"order {order} needs at least {order + 1} source levels per axis "
            f"(interpolation: p >= {order + 1} tangentially; either role: k >= {math.ceil((order + 1) / 2)})")


def _regions(role: str, p: int, k: int):
    _check_role(role)
    if role == "interpolate":
        return geometry.ref_interp_target_full(p, k), geometry.ref_interp_source(p, k)
    return geometry.ref_restrict_target(p, k, None), geometry.ref_restrict_source(p, k)


def condition_warning(condition_estimate: float):
    """Warning text when a fit's triangular conditioning exceeds 1e12 (taylor.py:160-168)."""
    if condition_estimate > CONDITION_WARN_THRESHOLD:
        return (f"derivative fit condition_estimate {condition_estimate:.3e} exceeds "
                f"{CONDITION_WARN_THRESHOLD:g}; operator accuracy may floor well above machine precision")
    return None


def taylor_target_offset(target: tuple, role: str, p: int, k: int) -> np.ndarray:
    """Target centre minus its nearest source centre, in source spacings (taylor.py:235-249)."""
    tgt, src = _regions(role, p, k)
    c = nearest_source_cell(target, role, p, k)
    t_centre = np.asarray(tgt.origin) + (np.asarray(target) + 0.5) * tgt.spacing
    s_centre = np.asarray(src.origin) + (np.asarray(c) + 0.5) * src.spacing
    return (t_centre - s_centre) / src.spacing


def nearest_source_cell(target: tuple, role: str, p: int, k: int) -> tuple:
    """Source cell whose centre is closest to the target's, ties to the lower index per axis."""
    tgt, src = _regions(role, p, k)
    c = tgt.centre_of(target)
    return tuple(int(np.argmin(np.abs(src.origin[d] + (np.arange(src.extents[d]) + 0.5) * src.spacing - c[d])))
                 for d in range(3))


def select_stencil(centre: tuple, region: RegionShape, order: int) -> StencilSpec:
    """Cube of STENCIL_BLOCK[order] cells per axis around the centre, shifted inward to fit."""
    basis = taylor_basis(order)
    block = STENCIL_BLOCK[order]
    axes = []
    for d in range(3):
        ext = region.extents[d]
        if not 0 <= centre[d] < ext:
            raise ConfigurationError(f"stencil centre {centre} outside region extents {region.extents}")
        n = min(block, ext)
        if n < order + 1:
            raise StencilInfeasibleError(f"axis {d} of source region {region.extents} offers {ext} cells; "
                                         + _requirement(order))
        lo = max(0, min(centre[d] - block // 2, ext - n))
        axes.append(np.arange(lo, lo + n) - centre[d])
    s = axes[0].size * axes[1].size * axes[2].size
    if s < basis.n + STENCIL_MARGIN:
        raise StencilInfeasibleError(f"stencil of {s} cells cannot support {basis.n} derivatives "
                                     f"plus margin {STENCIL_MARGIN}; " + _requirement(order))
    offsets = np.array([(x, y, z) for z in axes[2] for y in axes[1] for x in axes[0]], dtype=np.int64)
    offsets.setflags(write=False)
    return StencilSpec(tuple(centre), offsets)


def build_derivative_fit(stencil: StencilSpec, basis: TaylorBasis, spacing_units: float = 1.0) -> DerivativeFit:
    """Least-squares weights of the scaled derivatives at the stencil centre (the builder's
    Householder QR, linalg.py:99-112)."""
    a = np.ascontiguousarray(basis.design(stencil.offsets * spacing_units))
    s, n = a.shape
    if s < n:
        raise ContractViolationError(f"system must have rows >= cols, got {a.shape}")
    w = np.empty((n, s))
    cond = ctypes.c_double()
    _native.check(_native.load().th_pseudoinverse_rows(a.ctypes.data, s, n, w.ctypes.data, ctypes.byref(cond)))
    return DerivativeFit(stencil, w, float(cond.value))


def _taylor(cfg: FaceConfig, order: int, role: str, half=None) -> CsrOperator:
    from .schemes import require_feasible

    taylor_basis(order)  # order validation, as the reference
    scheme = f"order{order}"
    require_feasible(scheme, role, cfg.p, cfg.k)
    return DEFAULT_CACHE.get(OperatorKey(role, scheme, cfg.p, cfg.k, half=half))


def build_interpolation(cfg: FaceConfig, order: int) -> CsrOperator:
    """Full-face order-2/3 interpolation operator (taylor.py:222-224), from the C++ builder."""
    return _taylor(cfg, order, "interpolate")


def build_restriction(cfg: FaceConfig, order: int, half: str | None = None) -> CsrOperator:
    """Order-2/3 restriction operator, optionally one half's rows (taylor.py:227-232)."""
    if half not in (None, "inner", "outer"):
        raise ConfigurationError(f"half must be 'inner', 'outer' or None, got {half!r}")
    return _taylor(cfg, order, "restrict", half)


# ---------------------------------------------------------------------------
# least squares (linalg.py:19-112) through the builder's Householder QR
# ---------------------------------------------------------------------------

class PseudoInverse(tuple):
    """(weights n x s, condition_estimate)."""

    def __new__(cls, weights, condition_estimate):
        return super().__new__(cls, (weights, condition_estimate))

    weights = property(lambda self: self[0])
    condition_estimate = property(lambda self: self[1])


class LeastSquaresSolution(tuple):
    """(coefficients, condition_estimate)."""

    def __new__(cls, coefficients, condition_estimate):
        return super().__new__(cls, (coefficients, condition_estimate))

    coefficients = property(lambda self: self[0])
    condition_estimate = property(lambda self: self[1])


def solve_pseudoinverse_rows(a) -> PseudoInverse:
    """Least-squares pseudo-inverse of a full-rank tall matrix: R^-1 Q^T, one QR (linalg.py:99-112)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ContractViolationError(f"matrix must be 2-D, got shape {a.shape}")
    a = np.ascontiguousarray(a)
    s, n = a.shape
    if s < n:
        raise ContractViolationError(f"system must have rows >= cols, got {a.shape}")
    w = np.empty((n, s))
    cond = ctypes.c_double()
    _native.check(_native.load().th_pseudoinverse_rows(a.ctypes.data, s, n, w.ctypes.data, ctypes.byref(cond)))
    return PseudoInverse(w, float(cond.value))


def qr_least_squares(a, b) -> LeastSquaresSolution:
    """argmin ||a x - b|| (linalg.py:86-96): x = A+ b with the same factorisation."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim == 2 and b.shape != (a.shape[0],):
        raise ContractViolationError(f"rhs must have length {a.shape[0]}, got {b.shape}")
    w, cond = solve_pseudoinverse_rows(a)
    return LeastSquaresSolution(w @ b, cond)


def _collapse(p: int, k: int, role: str) -> CsrOperator:
    """linear._collapse (linear.py:202-240), which the reference's own tests call directly."""
    _check_role(role)
    return DEFAULT_CACHE.get(OperatorKey(role, "matrix_linear", p, k))
