"""Accuracy gates through the B200 path.

The reference's acceptance criteria 1-4 (test_acceptance.py:30-140) and harness
tests (test_harness.py:55-160), with the same tolerances and ladders, run on the
device kernels via paper_2504_15814_b200.harness."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2504_15814_b200 as th
from paper_2504_15814_b200 import harness
from paper_2504_15814_b200.operators import CsrOperator

ORACLE_TOL = 1e-11
MATRIX_TOL = 1e-13
POLY_TOL = 1e-9
ROW_SUM_TOL = 1e-12
DENSE_TOL = 1e-13
CONVERGENCE_LADDERS = {
    "matrix_linear": np.geomspace(0.03, 0.001, 7),
    "order2": np.geomspace(0.05, 0.0025, 7),
    "order3": np.geomspace(0.12, 0.005, 8),
}
EXPECTED_ORDERS = {"matrix_linear": (2.0, 0.2), "order2": (3.0, 0.3), "order3": (4.0, 0.4)}
PLATEAU_WINDOW = (1e-10, 1e-6)


# ---- host-only checks (no GPU) -------------------------------------------------

def test_convergence_requires_three_distinct_h():
    cfg = th.FaceConfig()
    with pytest.raises(th.ConfigurationError):
        harness.run_convergence("matrix_linear", "interpolate", cfg, [0.1, 0.05])
    with pytest.raises(th.ConfigurationError):
        harness.run_convergence("matrix_linear", "interpolate", cfg, [0.1, 0.1, 0.05])


def test_fit_order_on_synthetic_power_law():
    hs = np.geomspace(0.5, 0.01, 6)
    order, ok = harness._fit_order(hs, 2.7 * hs ** 3, threshold=0.0)
    assert ok and order == pytest.approx(3.0, abs=1e-10)


def test_sample_field_channels():
    region = th.RegionShape((2, 1, 1), 1.0, (0.0, 0.0, 0.0))
    buf = harness.sample_field(region, harness.affine_field(0.0, 1.0, 0.0, 0.0), 3, h=1.0, channel_phase=0.5)
    grid = buf.values.reshape(2, 3)
    assert np.allclose(grid[:, 1] - grid[:, 0], 0.5) and np.allclose(grid[:, 2] - grid[:, 0], 1.0)


def test_convergence_infeasible_scheme_raises():
    with pytest.raises(th.StencilInfeasibleError):
        harness.run_convergence("order2", "interpolate", th.FaceConfig("x", "negative", 4, 4, 1, 1), [0.2, 0.1, 0.05])


# ---- device suites -----------------------------------------------------------------

@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _poly(rng, degree):
    exps = [(a, b, d - a - b) for d in range(degree + 1) for a in range(d, -1, -1) for b in range(d - a, -1, -1)]
    coef = rng.uniform(-1.0, 1.0, size=len(exps))

    def f(x, y, z):
        out = np.zeros_like(np.asarray(x, dtype=np.float64))
        for c, (a, b, e) in zip(coef, exps):
            out = out + c * x ** a * y ** b * z ** e
        return out

    return f


@pytest.mark.gpu
def test_criterion_1_linear_exactness_oracle(gpu):
    s = harness.run_unit_oracle(ps=(1, 3, 4, 6), ks=(1, 3), tol=ORACLE_TOL, matrix_tol=MATRIX_TOL, u=4, seed=0)
    assert s.all_pass, "\n" + s.format_table()
    assert all(c.detail for c in s.cases if c.status == "skipped")


@pytest.mark.gpu
def test_criterion_2_polynomial_reproduction(gpu):
    rng = np.random.default_rng(1)
    checked = 0
    for scheme, degree in (("order2", 2), ("order3", 3)):
        for role in ("interpolate", "restrict"):
            for p, k in [(p, k) for p in (3, 4, 6) for k in (1, 3) if k <= p]:
                if not th.scheme_feasible(scheme, role, p, k)[0]:
                    continue
                for normal, side in (("x", "negative"), ("y", "positive")):
                    cfg = th.FaceConfig(normal, side, 4, p, k, 2)
                    f = _poly(rng, degree)
                    for half in ((None,) if role == "interpolate" else ("inner", "outer")):
                        region = th.interp_source_shape(cfg) if role == "interpolate" else th.restrict_source_shape(cfg)
                        out = th.apply_scheme(cfg, scheme, role, harness.sample_field(region, f, 2, h=0.4), half=half)
                        want = harness.sample_field(out.region, f, 2, h=0.4)
                        err = float(np.abs(out.values - want.values).max())
                        assert err < POLY_TOL, (scheme, role, p, k, normal, half, err)
                        checked += 1
    assert checked > 20


@pytest.mark.gpu
def test_criterion_3_convergence_orders(gpu):
    cfg = th.FaceConfig("x", "negative", 4, 4, 3, 2)
    for scheme, (nominal, tol) in EXPECTED_ORDERS.items():
        for role in ("interpolate", "restrict"):
            rep = harness.run_convergence(scheme, role, cfg, CONVERGENCE_LADDERS[scheme].tolist())
            assert rep.fit_reliable, (scheme, role)
            for fitted in (rep.fitted_order_max, rep.fitted_order_l2):
                assert abs(fitted - nominal) <= tol, (scheme, role, fitted)
            if scheme == "order3":
                lo, hi = PLATEAU_WINDOW
                assert [pt for pt in rep.points if pt.plateau and lo <= pt.err_max <= hi], (role, rep.points)
                assert rep.condition_warnings and "condition_estimate" in rep.condition_warnings[0]


@pytest.mark.gpu
def test_criterion_4_consistency_invariants(gpu):
    cases = harness.run_consistency_suite(ps=(1, 3, 4, 6), ks=(1, 3), row_sum_tol=ROW_SUM_TOL, dense_tol=DENSE_TOL,
                                          u=4, seed=0)
    assert not [c for c in cases if c.status == "fail"]
    assert {c.check for c in cases} >= {"row_sum", "dense_oracle", "deterministic_rebuild"}


@pytest.mark.gpu
def test_convergence_affine_field_flags_unreliable_fit(gpu):
    rep = harness.run_convergence("matrix_linear", "interpolate", th.FaceConfig("x", "negative", 4, 4, 3, 1),
                                  [0.4, 0.2, 0.1], f=harness.affine_field(0.3, 1.0, -2.0, 0.5))
    assert all(pt.err_max < 1e-12 and pt.plateau for pt in rep.points)
    assert not rep.fit_reliable and math.isnan(rep.fitted_order_max)


@pytest.mark.gpu
def test_unit_oracle_small_grid_and_skips(gpu):
    s = harness.run_unit_oracle(ps=(3,), ks=(3,), u=2)
    assert s.all_pass
    skipped = [c for c in s.cases if c.scheme == "order3" and c.role == "interpolate"]
    assert skipped and all(c.status == "skipped" and "p >= 4" in c.detail for c in skipped)


@pytest.mark.gpu
def test_unit_oracle_detects_corrupted_operator(gpu):
    def corrupt(op):
        v = op.values.copy()
        if v.size:  # the outer half at k = 1 has no rows
            v[0] += 0.37
        return CsrOperator(op.n_rows, op.n_cols, op.row_offsets, op.col_indices, v, op.scheme_tag, op.built_for,
                           op.source_region, op.target_region, op.max_condition)

    s = harness.run_unit_oracle(which_schemes=("matrix_linear",), ps=(3,), ks=(1,), u=2, operator_transform=corrupt)
    assert s.failed > 0 and s.failures()[0].max_err > 1e-3


@pytest.mark.gpu
def test_unit_oracle_threads_match_serial(gpu):
    a = harness.run_unit_oracle(which_schemes=("matrix_linear",), ps=(3,), ks=(1,), u=2)
    b = harness.run_unit_oracle(which_schemes=("matrix_linear",), ps=(3,), ks=(1,), u=2, threads=4)
    assert [c.status for c in a.cases] == [c.status for c in b.cases]
    assert [c.max_err for c in a.cases] == [c.max_err for c in b.cases]


@pytest.mark.gpu
def test_bench_single_repetition_and_phases(gpu):
    rep = harness.run_bench("matrix_linear", "interpolate", th.FaceConfig("x", "negative", 4, 3, 1, 4), repetitions=1)
    assert rep.phase == "apply" and rep.repetitions == 1 and rep.total_ns > 0
    con = harness.run_bench("order2", "restrict", th.FaceConfig("x", "negative", 0, 3, 3, 4), repetitions=2,
                            include_construction=True)
    assert con.phase == "construct"
