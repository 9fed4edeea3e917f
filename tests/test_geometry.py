"""Product geometry (host mirror of trihalo.geometry) and the kernels' index
arithmetic, bit-exact against the reference's HaloExchange maps captured in
tests/golden/maps.npz (p = 4, 5, 9, 17; all 6 orientations x 9 segments x
3 restriction halves).  CPU only."""

from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import paper_2504_15814_b200 as th
from paper_2504_15814_b200 import faces, geometry as G

FACES = list(itertools.product(("x", "y", "z"), ("negative", "positive")))


@pytest.fixture(scope="module")
def maps():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "maps.npz"))


def test_kernel_index_arithmetic_matches_reference_maps(maps):
    n = 0
    for p, k in ((4, 3), (5, 2), (9, 3), (17, 3)):
        for normal, side in FACES:
            for seg in range(9):
                cfg = G.FaceConfig(normal, side, seg, p, k, 1)
                key = f"interp|{p}|{k}|{normal}|{side}|{seg}"
                # reference: ref_src[r] = world[gather[r]]  -> the kernel's address of ref cell r
                assert np.array_equal(G.kernel_source_cells(cfg, "interpolate"), maps[key + "|g"]), key
                # reference: out[w] = ref_out[scatter[w]] -> kernel writes ref cell r to world cell t[r]
                t = G.kernel_target_cells(cfg, "interpolate")
                assert np.array_equal(t[maps[key + "|s"]], np.arange(t.size)), key
                n += 1
            for half in (None, "inner", "outer"):
                cfg = G.FaceConfig(normal, side, 0, p, k, 1)
                key = f"restrict|{p}|{k}|{normal}|{side}|{half}"
                assert np.array_equal(G.kernel_source_cells(cfg, "restrict"), maps[key + "|g"]), key
                t = G.kernel_target_cells(cfg, "restrict", half)
                assert np.array_equal(t[maps[key + "|s"]], np.arange(t.size)), key
                n += 1
    assert n == 4 * 6 * 12


def test_frame_maps_match_reference(maps):
    """gather_cell_indices (geometry.py:332-341) of the product mirror, bit-exact."""
    for p, k in ((4, 3), (9, 3)):
        for normal, side in FACES:
            cfg = G.FaceConfig(normal, side, 3, p, k, 1)
            fr = G.reference_frame(cfg)
            g = G.gather_cell_indices(fr, G.interp_source_shape(cfg))
            assert np.array_equal(g, maps[f"interp|{p}|{k}|{normal}|{side}|3|g"])
            s = G.gather_cell_indices(fr.inverse(), G.ref_restrict_target(p, k, "inner"))
            assert np.array_equal(s, maps[f"restrict|{p}|{k}|{normal}|{side}|inner|s"])


def test_region_shapes():
    """pkg/tests/test_geometry.py:37-120 shapes and origins."""
    cfg = G.FaceConfig("x", "negative", 0, 4, 3)
    r = G.interp_source_shape(cfg)
    assert (r.extents, r.spacing, r.origin) == ((6, 4, 4), 3.0, (-9.0, 0.0, 0.0))
    assert G.interp_target_shape(G.FaceConfig("x", "negative", 8, 4, 3)).origin == (0.0, 8.0, 8.0)
    assert G.interp_target_shape(G.FaceConfig("x", "negative", 0, 1, 1), full_face=True).extents == (1, 3, 3)
    s = G.restrict_source_shape(cfg)
    assert (s.extents, s.origin) == ((6, 12, 12), (-3.0, 0.0, 0.0))
    inner, outer = G.restrict_target_shape(cfg, "inner"), G.restrict_target_shape(cfg, "outer")
    assert inner.extents == (2, 4, 4) and outer.extents == (1, 4, 4) and outer.origin == (6.0, 0.0, 0.0)
    assert G.restrict_target_shape(G.FaceConfig("x", "negative", 0, 1, 1), "outer").extents == (0, 1, 1)
    tgt = G.interp_target_shape(G.FaceConfig("y", "positive", 0, 4, 3))
    ys = [tgt.centre_of(tgt.delinearize(n))[1] for n in range(tgt.cell_count)]
    assert max(ys) < 0.0 and min(ys) >= -3.0


def test_to_from_reference_round_trip():
    rng = np.random.default_rng(1)
    p, k, u = 3, 2, 2
    for normal, side in FACES:
        for seg in range(9):
            cfg = G.FaceConfig(normal, side, seg, p, k, u)
            for region in (G.interp_source_shape(cfg), G.interp_target_shape(cfg), G.restrict_source_shape(cfg),
                           G.restrict_target_shape(cfg), G.restrict_target_shape(cfg, "inner")):
                buf = G.HaloBuffer(region, u, rng.standard_normal(region.cell_count * u))
                back = G.from_reference(cfg, G.to_reference(cfg, buf))
                assert back.region == region and np.array_equal(back.values, buf.values)
    with pytest.raises(th.ContractViolationError):
        G.to_reference(G.FaceConfig(), G.HaloBuffer.zeros(G.RegionShape((5, 5, 5), 1.0, (0.0, 0.0, 0.0)), 1))
    with pytest.raises(th.ContractViolationError):
        G.HaloBuffer(G.RegionShape((2, 2, 2), 1.0, (0.0, 0.0, 0.0)), 2, np.zeros(7))


def test_slab_face_records_follow_world_boxes():
    """Face records of contiguous world boxes: strides are the world region strides."""
    p, k, u = 4, 3, 5
    for normal, side in FACES:
        cfg = G.FaceConfig(normal, side, 2, p, k, u)
        rec = faces.slab_faces("restrict", p, k, u, [cfg.normal], [cfg.side], half="inner")
        world = G.restrict_source_shape(cfg)
        assert tuple(rec["src_stride"][0]) == tuple(s * u for s in world.strides)
        tgt = G.restrict_target_shape(cfg, "inner")
        assert tuple(rec["dst_stride"][0]) == tuple(s * u for s in tgt.strides)
        t1, t2 = G.tangential_axes(cfg.normal)
        for b in range(9):
            corner = [0, 0, 0]
            corner[t1], corner[t2] = (b % 3) * p, (b // 3) * p
            assert rec["src"][0, b] == world.linearize(tuple(corner)) * u
