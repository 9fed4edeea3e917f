"""Product host-side operator construction (C++ builder behind the C ABI)
against the oracle, and the feasibility / error contract.  CPU only: the
builder runs without a device (th_operator_create_host)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2504_15814_b200 as th
from oracle import operators as OO
from paper_2504_15814_b200.operators import HostOperator

CASES = [(1, 1), (2, 1), (2, 2), (3, 2), (3, 3), (4, 2), (4, 3), (5, 3), (6, 2), (6, 3), (9, 3), (17, 3)]


def _dense(c):
    d = np.zeros((c.n_rows, c.n_cols))
    rows = np.repeat(np.arange(c.n_rows), np.diff(c.row_offsets))
    d[rows, c.col_indices] = c.values
    return d


@pytest.mark.parametrize("scheme", th.SCHEMES)
@pytest.mark.parametrize("role", ("interpolate", "restrict"))
def test_exported_rows_match_oracle(scheme, role):
    """Same sparsity as the reference CSR (incl. the 1e-14 drop rule, csr.py:120) and
    weights within 1e-12 of the row's largest weight."""
    for p, k in CASES:
        ok, _ = th.scheme_feasible(scheme, role, p, k)
        if not ok:
            continue
        if p == 17 and scheme == "order3" and role == "interpolate":
            continue  # slow oracle build; p=17 covered by the GPU parity tests
        h = HostOperator(role, scheme, p, k)
        osch = "matrix_linear" if scheme == "tensor_linear" else scheme
        sels = [None] + list(range(9)) if role == "interpolate" else [None, "inner", "outer"]
        for sel in sels:
            mine = h.csr(segment=sel) if role == "interpolate" else h.csr(half=sel)
            ref = OO.build_operator(osch, role, p, k, segment=sel if role == "interpolate" else None,
                                    half=sel if role == "restrict" else None)
            assert np.array_equal(mine.row_offsets, ref.row_offsets), (p, k, sel)
            assert np.array_equal(mine.col_indices, ref.col_indices), (p, k, sel)
            if ref.values.size:
                scale = np.abs(ref.values).max()
                assert np.abs(mine.values - ref.values).max() <= 1e-12 * scale, (p, k, sel)
            if scheme == "matrix_linear":  # same arithmetic as linear.py:202-240: bit-exact
                assert np.array_equal(mine.values, ref.values)


def test_row_sums_are_one():
    for scheme in ("matrix_linear", "order2", "order3"):
        for role in ("interpolate", "restrict"):
            c = HostOperator(role, scheme, 9, 3).csr()
            rows = np.repeat(np.arange(c.n_rows), np.diff(c.row_offsets))
            sums = np.bincount(rows, weights=c.values, minlength=c.n_rows)
            assert np.abs(sums - 1.0).max() < 1e-12


def test_compressed_layout_is_small():
    """Interior blocks repeat: order2 interp keeps 9 distinct 27x27 blocks, order3 25."""
    assert HostOperator("interpolate", "order2", 9, 3).info.n_blocks == 9
    assert HostOperator("interpolate", "order3", 9, 3).info.n_blocks == 25
    assert HostOperator("interpolate", "order3", 17, 3).info.n_blocks == 25
    assert HostOperator("restrict", "order2", 9, 3).info.n_blocks == 1
    assert HostOperator("restrict", "order3", 9, 3).info.n_blocks == 9
    assert HostOperator("interpolate", "order2", 9, 3).info.max_items_per_face == 9


def test_condition_metadata():
    h = HostOperator("interpolate", "order2", 4, 3)
    assert np.isfinite(h.max_condition) and h.max_condition >= 1.0
    assert np.isnan(HostOperator("interpolate", "matrix_linear", 4, 3).max_condition)
    ref = OO.full_face_operator("order3", "restrict", 4, 3)
    assert abs(HostOperator("restrict", "order3", 4, 3).max_condition - ref.max_condition) < 1e-10 * ref.max_condition


@pytest.mark.parametrize(
    "scheme,role,p,k,expect",
    [  # the reference feasibility table, pkg/tests/test_schemes.py:11-32
        ("tensor_linear", "interpolate", 1, 1, True),
        ("matrix_linear", "restrict", 1, 1, True),
        ("order2", "interpolate", 3, 1, False),
        ("order2", "interpolate", 3, 2, True),
        ("order2", "interpolate", 2, 2, False),
        ("order2", "restrict", 1, 1, False),
        ("order2", "restrict", 3, 2, True),
        ("order3", "interpolate", 3, 3, False),
        ("order3", "interpolate", 4, 2, True),
        ("order3", "interpolate", 4, 1, False),
        ("order3", "restrict", 2, 2, True),
        ("order3", "restrict", 3, 3, True),
    ],
)
def test_feasibility_table(scheme, role, p, k, expect):
    ok, reason = th.scheme_feasible(scheme, role, p, k)
    assert ok == expect
    if not ok:
        assert "infeasible" in reason


def test_errors_mirror_reference():
    with pytest.raises(th.StencilInfeasibleError) as err:
        th.require_feasible("order2", "interpolate", 4, 1)
    assert "k >= 2" in str(err.value)
    with pytest.raises(th.StencilInfeasibleError) as err3:
        th.require_feasible("order3", "interpolate", 3, 3)
    assert "p >= 4" in str(err3.value)
    with pytest.raises(th.ConfigurationError):
        th.scheme_feasible("order4", "interpolate", 4, 3)
    with pytest.raises(th.ConfigurationError):
        th.scheme_feasible("order2", "sideways", 4, 3)
    with pytest.raises(th.ConfigurationError):
        th.scheme_feasible("order2", "interpolate", 4, 5)
    with pytest.raises(th.ConfigurationError):
        HostOperator("interpolate", "order2", 0, 0)
    with pytest.raises(th.StencilInfeasibleError):
        HostOperator("interpolate", "order3", 3, 3)
    with pytest.raises(th.ConfigurationError):
        th.FaceConfig("x", "negative", 9, 4, 3)
    with pytest.raises(th.ConfigurationError):
        th.build_reference_operator("tensor_linear", "interpolate", 4, 3)
