"""The reference's host construction API (trihalo/__init__.py:37-51) on the drop-in:
axis operators, Taylor basis, nearest source cell, stencil selection, derivative fit and
the full-face operators, checked against the oracle restatement (itself pinned to the
reference's goldens in test_oracle.py) and the reference's known answers.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2504_15814_b200 as th
from oracle import geometry as OG
from oracle import operators as OO


@pytest.mark.parametrize("p", (1, 2, 4, 9, 17))
def test_axis_operators_bit_exact(p):
    assert np.array_equal(th.build_axis_tangential(p).matrix, OO.axis_tangential(p))
    from paper_2504_15814_b200 import construction as C

    assert np.array_equal(C.build_restrict_axis_tangential(p).matrix, OO.restrict_axis_tangential(p))
    for k in range(1, min(p, 4) + 1):
        assert np.array_equal(th.build_axis_normal(k).matrix, OO.axis_normal(k))
        assert np.array_equal(C.build_restrict_axis_normal(k).matrix, OO.restrict_axis_normal(k))
    assert th.build_axis_tangential(p).kind == "tangential"


def test_axis_known_answers():
    # minimal segment weights 1/3, 2/3 (reference test_linear.py): fine centre 0.5 between
    # coarse centres 1.5 and 4.5 extrapolates with the first pair's slope
    m = th.build_axis_tangential(2).matrix
    assert np.allclose(m.sum(axis=1), 1.0)
    assert np.allclose(m[1], [1.0, 0.0]) and np.allclose(m[2], [2.0 / 3.0, 1.0 / 3.0])
    with pytest.raises(th.ConfigurationError):
        th.build_axis_tangential(0)
    with pytest.raises(th.ConfigurationError):
        th.build_axis_normal(0)


@pytest.mark.parametrize("order", (2, 3))
def test_taylor_basis(order):
    b = th.taylor_basis(order)
    assert list(b.exponents) == OO.basis_exponents(order)
    pts = np.random.default_rng(order).standard_normal((7, 3))
    assert np.array_equal(b.design(pts), OO.design(OO.basis_exponents(order), pts))
    assert b.n == {2: 10, 3: 20}[order]
    with pytest.raises(th.ConfigurationError):
        th.taylor_basis(4)


@pytest.mark.parametrize("role", ("interpolate", "restrict"))
def test_nearest_source_cell_and_stencil(role):
    p, k = 5, 3
    tgt = OG.ref_interp_target_full(p, k) if role == "interpolate" else OG.ref_restrict_target(p, k)
    src = OG.ref_interp_source(p, k) if role == "interpolate" else OG.ref_restrict_source(p, k)
    src_mirror = th.geometry.ref_interp_source(p, k) if role == "interpolate" else th.geometry.ref_restrict_source(p, k)
    for r in range(0, tgt.n, 7):
        t = tgt.unlin(r)
        c = th.nearest_source_cell(t, role, p, k)
        assert c == OO.nearest_cell(t, tgt, src)
        for order in (2, 3):
            st = th.select_stencil(c, src_mirror, order)
            assert st.centre == c
            assert np.array_equal(st.offsets, OO.stencil_offsets(c, src, order))


def test_stencil_infeasible_names_constraint():
    region = th.RegionShape((2, 9, 9), 3.0, (-6.0, 0.0, 0.0))
    with pytest.raises(th.StencilInfeasibleError) as err:
        th.select_stencil((0, 4, 4), region, 2)
    assert "k >= 2" in str(err.value)


def test_derivative_fit_matches_oracle_and_central_differences():
    basis = th.taylor_basis(2)
    st = th.select_stencil((2, 2, 2), th.RegionShape((5, 5, 5), 1.0, (0.0, 0.0, 0.0)), 2)
    fit = th.build_derivative_fit(st, basis)
    want, cond = OO.pseudo_inverse(OO.design(OO.basis_exponents(2), st.offsets))
    assert fit.weights.shape == (10, 27)
    assert np.abs(fit.weights - want).max() <= 1e-13 and abs(fit.condition_estimate - cond) <= 1e-12 * cond
    # reproduces a quadratic exactly: scaled derivatives of x^2/2 + 3 y z at the centre
    f = 0.5 * st.offsets[:, 0] ** 2 + 3.0 * st.offsets[:, 1] * st.offsets[:, 2] + 2.0
    d = fit.weights @ f
    ex = list(basis.exponents)
    assert abs(d[ex.index((0, 0, 0))] - 2.0) < 1e-12 and abs(d[ex.index((2, 0, 0))] - 1.0) < 1e-12
    assert abs(d[ex.index((0, 1, 1))] - 3.0) < 1e-12


def test_derivative_fit_singular_column():
    basis = th.taylor_basis(2)
    flat = th.StencilSpec((0, 0, 0), np.array([(x, y, 0) for y in range(-1, 2) for x in range(-1, 2)] * 2))
    with pytest.raises(th.SingularFitError) as err:
        th.build_derivative_fit(flat, basis)
    assert err.value.column >= 0


@pytest.mark.parametrize("p,k", ((4, 3), (5, 2), (9, 3)))
def test_full_face_operators(p, k):
    cfg = th.FaceConfig("x", "negative", 4, p, k, 3)
    for role in ("interpolate", "restrict"):
        got = th.collapse_to_matrix(cfg, role)
        want = OO.collapse_linear(p, k, role)
        assert np.array_equal(got.row_offsets, want.row_offsets) and np.array_equal(got.col_indices, want.col_indices)
        assert np.array_equal(got.values, want.values)
    for order in (2, 3):
        ok_i, _ = th.scheme_feasible(f"order{order}", "interpolate", p, k)
        if ok_i:
            got = th.build_interpolation(cfg, order)
            want = OO.taylor_full_face(p, k, order, "interpolate")
            assert np.array_equal(got.col_indices, want.col_indices)
            assert np.abs(got.values - want.values).max() <= 1e-12 * np.abs(want.values).max()
        for half in (None, "inner", "outer"):
            got = th.build_restriction(cfg, order, half=half)
            want = OO.build_operator(f"order{order}", "restrict", p, k, half=half)
            assert np.array_equal(got.col_indices, want.col_indices)
            assert np.abs(got.values - want.values).max() <= 1e-12 * np.abs(want.values).max()
    with pytest.raises(th.ConfigurationError):
        th.build_interpolation(cfg, 4)
    with pytest.raises(th.ConfigurationError):
        th.collapse_to_matrix(cfg, "prolong")
