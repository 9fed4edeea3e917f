"""Pin the CPU oracle to the reference: golden fixtures made by the real
reference package (tests/golden/make_golden.py) and the reference's own
known-answer tests.  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import exchange as OE
from oracle import geometry as OG
from oracle import operators as OO

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ops_npz():
    return np.load(os.path.join(GOLDEN, "operators.npz"))


@pytest.fixture(scope="module")
def maps_npz():
    return np.load(os.path.join(GOLDEN, "maps.npz"))


@pytest.fixture(scope="module")
def ex_npz():
    return np.load(os.path.join(GOLDEN, "exchange.npz"))


def _keys(npz):
    return sorted({k.rsplit("|", 1)[0] for k in npz.files})


def test_operators_bitwise_equal_reference(ops_npz):
    """Oracle CSR == reference OperatorCache.get CSR, bit for bit (taylor.py:252-308)."""
    n = 0
    for key in _keys(ops_npz):
        scheme, role, p, k = key.split("|")
        op = OO.full_face_operator(scheme, role, int(p), int(k))
        assert np.array_equal(op.row_offsets, ops_npz[key + "|ro"]), key
        assert np.array_equal(op.col_indices, ops_npz[key + "|ci"]), key
        assert np.array_equal(op.values, ops_npz[key + "|v"]), key
        if scheme != "matrix_linear":
            assert op.max_condition == ops_npz[key + "|cond"][0]
        n += 1
    assert n >= 66


def test_exchange_maps_bitwise_equal_reference(maps_npz):
    """Gather / scatter element maps == HaloExchange._gather/_scatter (schemes.py:147-151)."""
    n = 0
    for key in _keys(maps_npz):
        role, p, k, normal, side, sel = key.split("|")
        p, k = int(p), int(k)
        if role == "interp":
            ex = OE.OracleExchange(OG.FaceCfg(normal, side, int(sel), p, k, 1), "matrix_linear", "interpolate")
        else:
            half = None if sel == "None" else sel
            ex = OE.OracleExchange(OG.FaceCfg(normal, side, 0, p, k, 1), "matrix_linear", "restrict", half)
        assert np.array_equal(ex.gather, maps_npz[key + "|g"]), key
        assert np.array_equal(ex.scatter, maps_npz[key + "|s"]), key
        n += 1
    assert n == 4 * 6 * 12


def test_exchange_outputs_match_reference(ex_npz):
    """Oracle HaloExchange.run == reference run on seeded sources (<= 1e-14 relative)."""
    worst = 0.0
    for key in _keys(ex_npz):
        scheme, role, half, p, k, u, normal, side, seg = key.split("|")
        half = None if half == "None" else half
        cfg = OG.FaceCfg(normal, side, int(seg), int(p), int(k), int(u))
        ex = OE.exchange_for(cfg, scheme, role, half)
        src = np.random.default_rng(int(ex_npz[key + "|seed"][0])).standard_normal(ex.n_src)
        out = np.empty(ex.n_out)
        ex.run(src, out)
        want = ex_npz[key + "|out"]
        if want.size:
            err = np.abs(out - want).max() / max(np.abs(want).max(), 1e-300)
            worst = max(worst, err)
            assert err <= 1e-14, (key, err)


def test_dump_golden_p1k1():
    """The reference's own golden dump (pkg/tests/test_csr.py:185-194), rebuilt by the oracle."""
    with open(os.path.join(GOLDEN, "golden_p1k1.txt")) as fh:
        golden = fh.read()
    op = OO.collapse_linear(1, 1, "interpolate")
    lines = [f"{op.n_rows} {op.n_cols} {op.nnz} matrix_linear 1 1"]
    for r in range(op.n_rows):
        for t in range(op.row_offsets[r], op.row_offsets[r + 1]):
            lines.append(f"{r} {op.col_indices[t]} {op.values[t]:.17g}")
    assert "\n".join(lines) + "\n" == golden
    assert golden.splitlines()[1] == "0 0 0.33333333333333337"


def test_hand_derived_axis_rows():
    """Known answers of pkg/tests/test_linear.py:19-75."""
    t = OO.axis_tangential(4)
    assert np.array_equal(t[4], [0.0, 1.0, 0.0, 0.0])
    assert np.allclose(t[0], [4 / 3, -1 / 3, 0, 0], atol=1e-15)
    assert np.allclose(t[11], [0, 0, -1 / 3, 4 / 3], atol=1e-15)
    n = OO.axis_normal(3)
    assert np.allclose(n[0], [0, 0, 1 / 3, 2 / 3, 0, 0], atol=1e-15)
    assert np.array_equal(n[1], [0, 0, 0, 1.0, 0, 0])
    r = OO.restrict_axis_normal(3)
    assert np.allclose(r[0], [0, 0, 0, 1 / 3, 1 / 3, 1 / 3], atol=1e-15)
    assert np.allclose(r[1], [0, 0, 0, 0, -2.0, 3.0], atol=1e-13)
    assert np.allclose(r[2], [0, 0, 0, 0, -5.0, 6.0], atol=1e-13)
    assert np.allclose(OO.restrict_axis_normal(1), [[-1.0, 2.0]], atol=1e-14)
    r2 = OO.restrict_axis_normal(2)
    assert np.allclose(r2[0], [0, 0, 0, 1.0], atol=1e-15)
    assert np.allclose(r2[1], [0, 0, -3.0, 4.0], atol=1e-13)


def test_central_difference_fit_rows():
    """pkg/tests/test_linalg.py:54-61: rows (-1/2, 0, 1/2) and (1, -2, 1)."""
    d = np.array([-1.0, 0.0, 1.0])
    a = np.stack([np.ones(3), d, d ** 2 / 2.0], axis=1)
    w, _ = OO.pseudo_inverse(a)
    assert np.allclose(w[1], [-0.5, 0.0, 0.5], atol=1e-14)
    assert np.allclose(w[2], [1.0, -2.0, 1.0], atol=1e-13)
    bad = np.array([[1.0, 0.0, 1.0], [0.0, 1.0, 1.0], [1.0, 1.0, 2.0], [2.0, 1.0, 3.0]])
    with pytest.raises(OO.RankDeficient) as err:
        OO.pseudo_inverse(bad)
    assert err.value.column == 2


def test_nearest_cells_and_zero_offsets():
    """pkg/tests/test_taylor.py:45-82."""
    p, k = 4, 3
    tgt, src = OG.ref_interp_target_full(p, k), OG.ref_interp_source(p, k)
    for m in range(3 * p):
        assert OO.nearest_cell((0, m, 0), tgt, src)[1] == m // 3
    for i in range(k):
        assert OO.nearest_cell((i, 0, 0), tgt, src)[0] == k
    rt, rs = OG.ref_restrict_target(p, k), OG.ref_restrict_source(p, k)
    assert OO.nearest_cell((0, 0, 0), rt, rs)[0] == k + 1
    assert OO.nearest_cell((1, 0, 0), rt, rs)[0] == 2 * k - 1
    for j in range(p):
        assert OO.nearest_cell((0, j, 0), rt, rs)[1] == 3 * j + 1


def test_one_hot_orientation_map():
    """pkg/tests/test_geometry.py:148-165: normal=y, side=+ sends world (i,j,k2) to ref (2k-1-j, i, k2)."""
    p, k = 3, 2
    cfg = OG.FaceCfg("y", "positive", 0, p, k, 1)
    world = OG.interp_source_world(cfg)
    ref = OG.ref_interp_source(p, k)
    idx = OG.gather_cells(OG.frame_for(cfg), world)
    for (i, j, k2) in [(0, 0, 0), (2, 3, 1), (1, 2, 2), (0, 1, 2)]:
        assert idx[ref.lin(2 * k - 1 - j, i, k2)] == world.lin(i, j, k2)
