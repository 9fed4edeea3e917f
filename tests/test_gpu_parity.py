"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Tolerance: norm-wise relative error per face max|gpu - ref| / max|ref| <= 1e-12
(BASELINE.json north star, fp64).  Index maps are exercised bit-exactly by the
golden comparison (a wrong gather / scatter shows up as O(1) error).
"""

from __future__ import annotations

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12
FACES = list(itertools.product(("x", "y", "z"), ("negative", "positive")))


@pytest.fixture(scope="module")
def th():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    return th


def rel(a, b):
    scale = np.abs(b).max() if b.size else 1.0
    return float(np.abs(a - b).max() / max(scale, 1e-300)) if a.size else 0.0


def oracle_run(cfg, scheme, role, half, src):
    from oracle import exchange as OE
    from oracle import geometry as OG

    ocfg = OG.FaceCfg(cfg.normal_axis, cfg.coarse_side, cfg.segment, cfg.p, cfg.k, cfg.u)
    ex = OE.OracleExchange(ocfg, scheme, role, half)
    out = np.empty(ex.n_out)
    ex.run(src, out)
    return out


SMALL = [(4, 3, 3), (5, 2, 2), (6, 3, 5), (3, 3, 2), (1, 1, 2), (2, 2, 3), (4, 1, 1), (5, 3, 59), (5, 3, 70)]


@pytest.mark.parametrize("p,k,u", SMALL)
@pytest.mark.parametrize("scheme", ("tensor_linear", "matrix_linear", "order2", "order3"))
def test_exchange_all_faces_small(th, p, k, u, scheme):
    rng = np.random.default_rng(p * 100 + k * 10 + u)
    checked = 0
    for (normal, side), role_half in itertools.product(FACES, (("interpolate", None), ("restrict", None),
                                                              ("restrict", "inner"), ("restrict", "outer"))):
        role, half = role_half
        ok, _ = th.scheme_feasible(scheme, role, p, k)
        if not ok:
            continue
        segs = range(9) if role == "interpolate" else (0,)
        for seg in segs:
            cfg = th.FaceConfig(normal, side, seg, p, k, u)
            ex = th.HaloExchange(cfg, scheme, role, half=half)
            src, out = ex.make_buffers(rng)
            ex.run(src, out)
            want = oracle_run(cfg, scheme, role, half, src)
            assert rel(out, want) <= TOL, (scheme, role, half, normal, side, seg, rel(out, want))
            checked += 1
    if checked == 0:
        pytest.skip("scheme infeasible at this (p, k) for both roles")


def test_golden_exchange_outputs(th):
    """Reference HaloExchange.run outputs captured in tests/golden/exchange.npz."""
    import os

    data = np.load(os.path.join(os.path.dirname(__file__), "golden", "exchange.npz"))
    keys = sorted({k.rsplit("|", 1)[0] for k in data.files})
    worst = 0.0
    for key in keys:
        scheme, role, half, p, k, u, normal, side, seg = key.split("|")
        half = None if half == "None" else half
        p, k, u, seg = int(p), int(k), int(u), int(seg)
        cfg = th.FaceConfig(normal, side, seg, p, k, u)
        ex = th.HaloExchange(cfg, scheme, role, half=half)
        src = np.random.default_rng(int(data[key + "|seed"][0])).standard_normal(ex.n_src)
        out = np.zeros(ex.n_out)
        ex.run(src, out)
        err = rel(out, data[key + "|out"])
        worst = max(worst, err)
        assert err <= TOL, (key, err)
    assert len(keys) > 500


def test_functional_api_matches_exchange(th):
    rng = np.random.default_rng(3)
    for scheme in th.SCHEMES:
        cfg = th.FaceConfig("z", "positive", 7, 9, 3, 59)
        src_region = th.interp_source_shape(cfg)
        buf = th.HaloBuffer(src_region, 59, rng.standard_normal(src_region.cell_count * 59))
        got = th.interpolate_halo(cfg, scheme, buf)
        assert got.region == th.interp_target_shape(cfg)
        assert rel(got.values, oracle_run(cfg, scheme, "interpolate", None, buf.values)) <= TOL
        fr = th.restrict_source_shape(cfg)
        fb = th.HaloBuffer(fr, 59, rng.standard_normal(fr.cell_count * 59))
        for half in (None, "inner", "outer"):
            got = th.apply_scheme(cfg, scheme, "restrict", fb, half=half)
            assert got.region == th.restrict_target_shape(cfg, half)
            assert rel(got.values, oracle_run(cfg, scheme, "restrict", half, fb.values)) <= TOL


def test_nonfinite_source_raises(th):
    cfg = th.FaceConfig("x", "negative", 0, 4, 3, 2)
    ex = th.HaloExchange(cfg, "order2", "interpolate")
    src, out = ex.make_buffers(np.random.default_rng(0))
    src[5] = np.nan
    with pytest.raises(th.ContractViolationError):
        ex.run(src, out)
    src[5] = 0.0
    src[-1] = np.inf  # outside the operator support still counts (schemes.py:186)
    with pytest.raises(th.ContractViolationError):
        ex.run(src, out)
    src[-1] = 0.0
    ex.run(src, out)  # flag was cleared


def test_wrong_region_raises(th):
    cfg = th.FaceConfig("x", "negative", 0, 4, 3, 2)
    wrong = th.HaloBuffer.zeros(th.restrict_source_shape(cfg), 2)
    with pytest.raises(th.ContractViolationError):
        th.interpolate_halo(cfg, "matrix_linear", wrong)
    with pytest.raises(th.StencilInfeasibleError):
        th.HaloExchange(th.FaceConfig("x", "negative", 0, 4, 1, 1), "order2", "interpolate")


def test_csr_apply_matches_dense(th):
    """csr.apply on the device vs a dense product (reference test_csr.py:79-89 analogue)."""
    rng = np.random.default_rng(1)
    op = th.build_reference_operator("order3", "interpolate", 5, 3, segment=4)
    src = th.HaloBuffer(op.source_region, 58, rng.standard_normal(op.n_cols * 58))
    got = th.apply(op, src).values.reshape(op.n_rows, 58)
    want = op.to_dense() @ src.values.reshape(op.n_cols, 58)
    assert np.abs(got - want).max() < 1e-13 * max(1.0, np.abs(want).max())


# ---------------------------------------------------------------------------
# batched faces: slab and pool layouts
# ---------------------------------------------------------------------------

def _world_box(pool, E, u, pid, lo, ext):
    """Extract a world box (x-fastest AoS) from pool patch `pid`: lo/ext per world axis."""
    g = pool[pid].reshape(E, E, E, u)  # (z, y, x, u)
    return np.ascontiguousarray(g[lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]]).reshape(-1)


def _interp_box(p, k, normal, side):
    """Independent derivation of the coarse-patch box feeding interpolation."""
    lo, ext = [k, k, k], [p, p, p]
    lo[normal] = p if side == 0 else 0
    ext[normal] = 2 * k
    return lo, ext


@pytest.mark.parametrize("scheme", ("tensor_linear", "matrix_linear", "order2", "order3"))
@pytest.mark.parametrize("p", (9, 17))
def test_pool_interp_batch(th, scheme, p):
    import torch

    k, u = 3, 59
    rng = np.random.default_rng(p)
    E = p + 2 * k
    n_patch, n_face = 6, 40
    pool = rng.standard_normal((n_patch, E ** 3 * u))
    cid = rng.integers(0, n_patch, n_face)
    nrm = rng.integers(0, 3, n_face)
    sid = rng.integers(0, 2, n_face)
    seg = rng.integers(0, 9, n_face)
    rec = th.pool_interp_faces(p, k, u, cid, nrm, sid, seg)
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    batch = th.FaceBatch(op, rec, u)
    dev = torch.device("cuda")
    src = torch.from_numpy(pool.reshape(-1)).to(dev)
    dst = torch.full((n_face * k * p * p * u,), np.nan, dtype=torch.float64, device=dev)
    batch.launch(src, dst)
    out = dst.cpu().numpy().reshape(n_face, -1)
    assert not batch.nonfinite()
    for f in range(n_face):
        lo, ext = _interp_box(p, k, int(nrm[f]), int(sid[f]))
        box = _world_box(pool, E, u, int(cid[f]), lo, ext)
        cfg = th.FaceConfig("xyz"[nrm[f]], ("negative", "positive")[sid[f]], int(seg[f]), p, k, u)
        want = oracle_run(cfg, scheme, "interpolate", None, box)
        assert rel(out[f], want) <= TOL, (f, rel(out[f], want))


@pytest.mark.parametrize("scheme,p,n_face", (("order3", 17, 900), ("order2", 17, 900), ("order3", 9, 1500),
                                             ("order2", 9, 1500), ("order2", 4, 4000), ("order3", 5, 3000),
                                             ("tensor_linear", 17, 900), ("matrix_linear", 17, 900),
                                             ("tensor_linear", 9, 1500), ("matrix_linear", 5, 3000)))
def test_pool_interp_long_batch(th, scheme, p, n_face):
    """Batches long enough that every persistent CTA walks many tiles (148 CTAs, 2-4 tiles per
    face): the slice ring's slots, their sequence numbers and reader counts are reused tens of
    times, and the staged tiles run their double buffers in steady state (p = 4 / 5: tiles of 3-5
    slices, the widest skew between the ring's producers and consumers in tiles).  Every 7th face plus
    the last 40 are checked against the oracle; every output value must be written."""
    import torch

    k, u = 3, 59
    rng = np.random.default_rng(p * 3 + len(scheme))
    E = p + 2 * k
    n_patch = 8
    pool = rng.standard_normal((n_patch, E ** 3 * u))
    cid = rng.integers(0, n_patch, n_face)
    nrm = rng.integers(0, 3, n_face)
    sid = rng.integers(0, 2, n_face)
    seg = rng.integers(0, 9, n_face)
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    batch = th.FaceBatch(op, th.pool_interp_faces(p, k, u, cid, nrm, sid, seg), u)
    dev = torch.device("cuda")
    dst = torch.full((n_face * k * p * p * u,), np.nan, dtype=torch.float64, device=dev)
    batch.launch(torch.from_numpy(pool.reshape(-1)).to(dev), dst)
    assert not batch.nonfinite()
    assert bool(torch.isfinite(dst).all())
    out = dst.cpu().numpy().reshape(n_face, -1)
    for f in sorted(set(range(0, n_face, 7)) | set(range(n_face - 40, n_face))):
        lo, ext = _interp_box(p, k, int(nrm[f]), int(sid[f]))
        box = _world_box(pool, E, u, int(cid[f]), lo, ext)
        cfg = th.FaceConfig("xyz"[nrm[f]], ("negative", "positive")[sid[f]], int(seg[f]), p, k, u)
        want = oracle_run(cfg, scheme, "interpolate", None, box)
        assert rel(out[f], want) <= TOL, (f, rel(out[f], want))


@pytest.mark.parametrize("u", (1, 33, 65, 130, 200))
@pytest.mark.parametrize("scheme,p", (("tensor_linear", 9), ("order2", 9), ("order3", 9), ("order2", 17)))
def test_pool_interp_unknown_counts(th, scheme, p, u):
    """Interpolation across unknown counts: the staged tile kernel's flattened (block, unknown)
    items and its [unknown][cell] box at u = 1 (one item per block), 33 / 65 (items straddling
    warps), 130 (a 156 KB box pair: one CTA per SM), 200 (boxes beyond shared memory: the
    per-warp slide takes over); the slide's ragged 32-unknown chunks; for order3 the two-phase
    tiles' chunks of <= 31 unknowns, on 4-unknown sector boundaries (33, 65, 130) or not (200:
    aligned boundaries would leave a 32-unknown chunk)."""
    import torch

    k = 3
    rng = np.random.default_rng(u * 7 + p)
    E = p + 2 * k
    n_patch, n_face = 5, 12
    pool = rng.standard_normal((n_patch, E ** 3 * u))
    cid = rng.integers(0, n_patch, n_face)
    nrm, sid, seg = np.arange(n_face) % 3, (np.arange(n_face) // 3) % 2, rng.integers(0, 9, n_face)
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    batch = th.FaceBatch(op, th.pool_interp_faces(p, k, u, cid, nrm, sid, seg), u)
    dev = torch.device("cuda")
    dst = torch.full((n_face * k * p * p * u,), np.nan, dtype=torch.float64, device=dev)
    batch.launch(torch.from_numpy(pool.reshape(-1)).to(dev), dst)
    out = dst.cpu().numpy().reshape(n_face, -1)
    assert not batch.nonfinite()
    for f in range(n_face):
        lo, ext = _interp_box(p, k, int(nrm[f]), int(sid[f]))
        box = _world_box(pool, E, u, int(cid[f]), lo, ext)
        cfg = th.FaceConfig("xyz"[nrm[f]], ("negative", "positive")[sid[f]], int(seg[f]), p, k, u)
        want = oracle_run(cfg, scheme, "interpolate", None, box)
        assert rel(out[f], want) <= TOL, (scheme, p, u, f, rel(out[f], want))


@pytest.mark.parametrize("scheme", ("tensor_linear", "matrix_linear", "order2", "order3"))
@pytest.mark.parametrize("p,half", ((9, None), (17, None), (9, "inner"), (9, "outer")))
def test_pool_restrict_batch(th, scheme, p, half):
    import torch

    k, u = 3, 59
    rng = np.random.default_rng(p + 7)
    E = p + 2 * k
    n_patch, n_face = 12, 16
    pool = rng.standard_normal((n_patch, E ** 3 * u))
    nrm = rng.integers(0, 3, n_face)
    sid = rng.integers(0, 2, n_face)
    fine = rng.integers(0, n_patch, (n_face, 9))
    rec = th.pool_restrict_faces(p, k, u, fine, nrm, sid, half=half)
    op = th.operators.DEFAULT_CACHE.device_operator("restrict", scheme, p, k)
    batch = th.FaceBatch(op, rec, u)
    dev = torch.device("cuda")
    src = torch.from_numpy(pool.reshape(-1)).to(dev)
    lo_h, hi_h = th.geometry.half_layers(k, half)
    ncell = (hi_h - lo_h) * p * p
    dst = torch.full((n_face * ncell * u,), np.nan, dtype=torch.float64, device=dev)
    batch.launch(src, dst)
    out = dst.cpu().numpy().reshape(n_face, -1)
    for f in range(n_face):
        n = int(nrm[f])
        t1, t2 = [d for d in range(3) if d != n]
        # assemble the world restriction source (2k x 3p x 3p) from the nine fine patches
        ext = [3 * p, 3 * p, 3 * p]
        ext[n] = 2 * k
        world = np.zeros((ext[2], ext[1], ext[0], u))
        for b in range(9):
            b1, b2 = b % 3, b // 3
            lo = [k, k, k]
            lo[n] = 0 if sid[f] == 0 else p
            e = [p, p, p]
            e[n] = 2 * k
            blk = _world_box(pool, E, u, int(fine[f, b]), lo, e).reshape(e[2], e[1], e[0], u)
            off = [0, 0, 0]
            off[t1], off[t2] = b1 * p, b2 * p
            world[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = blk
        cfg = th.FaceConfig("xyz"[n], ("negative", "positive")[sid[f]], 0, p, k, u)
        want = oracle_run(cfg, scheme, "restrict", half, world.reshape(-1))
        assert rel(out[f], want) <= TOL, (f, rel(out[f], want))


def test_restrict_into_coarse_halo(th):
    """Restriction written straight into the coarse patches' halo layers of the pool."""
    import torch

    p, k, u = 9, 3, 5
    rng = np.random.default_rng(11)
    E = p + 2 * k
    fine_pool = rng.standard_normal((9, E ** 3 * u))
    coarse_pool = np.zeros((2, E ** 3 * u))
    dev = torch.device("cuda")
    for half in (None, "inner", "outer"):
        rec = th.pool_restrict_faces(p, k, u, np.arange(9)[None, :].repeat(2, 0), [1, 2], [0, 1], half=half,
                                     coarse_ids=[0, 1])
        rec_slab = th.pool_restrict_faces(p, k, u, np.arange(9)[None, :].repeat(2, 0), [1, 2], [0, 1], half=half)
        op = th.operators.DEFAULT_CACHE.device_operator("restrict", "order2", p, k)
        src = torch.from_numpy(fine_pool.reshape(-1)).to(dev)
        cdst = torch.from_numpy(coarse_pool.reshape(-1)).to(dev)
        th.FaceBatch(op, rec, u).launch(src, cdst)
        lo_h, hi_h = th.geometry.half_layers(k, half)
        sdst = torch.zeros(2 * (hi_h - lo_h) * p * p * u, dtype=torch.float64, device=dev)
        th.FaceBatch(op, rec_slab, u).launch(src, sdst)
        slab = sdst.cpu().numpy().reshape(2, -1)
        cp = cdst.cpu().numpy().reshape(2, E, E, E, u)
        for f, (n, side) in enumerate(((1, 0), (2, 1))):
            lo, ext = [k, k, k], [p, p, p]
            lo[n] = p + k + lo_h if side == 0 else k - hi_h
            ext[n] = hi_h - lo_h
            box = cp[f, lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]].reshape(-1)
            assert np.array_equal(box, slab[f])


def _transpose_records(rec, E, u, patch, fields=("src",)):
    """Re-address pool records for a z-fastest pool ([patch][x][y][z][u]); strides permuted."""
    out = rec.copy()
    for name in fields:
        off = out[name].astype(np.int64)
        pid, rem = np.divmod(off, patch)
        cell, q = np.divmod(rem, u)
        assert not q.any()
        z, yx = np.divmod(cell, E * E)
        y, x = np.divmod(yx, E)
        out[name] = pid * patch + ((x * E + y) * E + z) * u
    out["src_stride"] = [E * E * u, E * u, u]
    return out


@pytest.mark.parametrize("scheme", ("tensor_linear", "matrix_linear", "order2", "order3"))
@pytest.mark.parametrize("p", (9, 17))
def test_pool_transposed_layout(th, scheme, p):
    """A z-fastest pool: x- and y-normal faces have no contiguous normal / t1 axis, so the
    staged order3 restriction takes its one-copy-per-cell path (mode 2), z-normal faces
    its normal-run path.  Results must equal the x-fastest run bit for bit."""
    import torch

    k, u = 3, 59
    rng = np.random.default_rng(p + 31)
    E = p + 2 * k
    patch = E ** 3 * u
    n_patch, n_face = 12, 24
    pool = rng.standard_normal((n_patch, E, E, E, u))  # (z, y, x, u) per patch
    pool_t = np.ascontiguousarray(pool.transpose(0, 3, 2, 1, 4))  # (x, y, z, u)
    dev = torch.device("cuda")
    src = torch.from_numpy(pool.reshape(-1)).to(dev)
    src_t = torch.from_numpy(pool_t.reshape(-1)).to(dev)
    nrm = np.arange(n_face) % 3
    sid = (np.arange(n_face) // 3) % 2
    cases = [("restrict", th.pool_restrict_faces(p, k, u, rng.integers(0, n_patch, (n_face, 9)), nrm, sid), k * p * p)]
    if p == 9:
        cases.append(("interpolate", th.pool_interp_faces(p, k, u, rng.integers(0, n_patch, n_face), nrm, sid,
                                                          rng.integers(0, 9, n_face)), k * p * p))
    for role, rec, ncell in cases:
        op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
        rec_t = _transpose_records(rec, E, u, patch)
        outs = []
        for s, r in ((src, rec), (src_t, rec_t)):
            dst = torch.full((n_face * ncell * u,), np.nan, dtype=torch.float64, device=dev)
            th.FaceBatch(op, r, u).launch(s, dst)
            outs.append(dst.cpu().numpy())
        assert np.isfinite(outs[0]).all()
        assert np.array_equal(outs[0], outs[1]), (role, scheme, np.abs(outs[0] - outs[1]).max())


@pytest.mark.parametrize("env", ({"TH_GRAM": "3"}, {"TH_TILE": "0"}, {"TH_TILE3": "0"},
                                 {"TH_TILE": "0", "TH_GRAM": "0"}, {"TH_RING": "15"},
                                 {"TH_RING": "15", "TH_RING_NA": "3", "TH_RING_R": "6"}, {"TH_RING": "0"},
                                 {"TH_ROWN": "0"}))
def test_alternative_kernel_paths(th, env):
    """Kernel choices are read once per process from the environment; re-run the
    parity tests in a child process with the alternative paths (the per-warp order3
    restriction slide; the per-warp interpolation slide instead of the staged tile kernel;
    the per-warp slide for order3 interpolation instead of the two-phase order3 tiles; the
    fixed-window kernels with neither tiles nor Gram slides; the slice ring (ring_interp.cuh)
    for every interpolation (Gram and d-linear), also with 3 A warps and the smallest ring; the
    per-warp slide instead of the slice ring at p = 17; the staged order3 restriction with one
    consumer warp per t1 group instead of the line owners)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(here, "test_gpu_parity.py"),
         "-k", "exchange_all_faces_small or pool_interp_batch or pool_interp_long_batch or pool_restrict_batch or transposed "
         "or unknown_counts"],
        env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


@pytest.mark.parametrize("u", (1, 33, 65, 130))
@pytest.mark.parametrize("p", (9, 17))
def test_pool_restrict_order3_unknown_counts(th, u, p):
    """Staged order3 restriction across unknown counts: 1 (mostly idle lanes), 33 / 65 (ragged
    chunks), 130 (3 chunks of 64 -> tiles of 3 t1 groups, several tiles per face)."""
    import torch

    k = 3
    rng = np.random.default_rng(u * 10 + p)
    E = p + 2 * k
    n_patch, n_face = 10, 6
    pool = rng.standard_normal((n_patch, E ** 3 * u))
    nrm = np.arange(n_face) % 3
    sid = (np.arange(n_face) // 3) % 2
    fine = rng.integers(0, n_patch, (n_face, 9))
    rec = th.pool_restrict_faces(p, k, u, fine, nrm, sid)
    op = th.operators.DEFAULT_CACHE.device_operator("restrict", "order3", p, k)
    dev = torch.device("cuda")
    dst = torch.full((n_face * k * p * p * u,), np.nan, dtype=torch.float64, device=dev)
    th.FaceBatch(op, rec, u).launch(torch.from_numpy(pool.reshape(-1)).to(dev), dst)
    out = dst.cpu().numpy().reshape(n_face, -1)
    for f in range(n_face):
        n = int(nrm[f])
        t1, t2 = [d for d in range(3) if d != n]
        ext = [3 * p, 3 * p, 3 * p]
        ext[n] = 2 * k
        world = np.zeros((ext[2], ext[1], ext[0], u))
        for b in range(9):
            b1, b2 = b % 3, b // 3
            lo = [k, k, k]
            lo[n] = 0 if sid[f] == 0 else p
            e = [p, p, p]
            e[n] = 2 * k
            blk = _world_box(pool, E, u, int(fine[f, b]), lo, e).reshape(e[2], e[1], e[0], u)
            off = [0, 0, 0]
            off[t1], off[t2] = b1 * p, b2 * p
            world[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = blk
        cfg = th.FaceConfig("xyz"[n], ("negative", "positive")[sid[f]], 0, p, k, u)
        want = oracle_run(cfg, "order3", "restrict", None, world.reshape(-1))
        assert rel(out[f], want) <= TOL, (u, p, f, rel(out[f], want))


@pytest.mark.parametrize("p", (5, 6, 7, 8, 10, 11, 12, 13, 16))
def test_pool_restrict_order3_patch_sizes(th, p):
    """Staged order3 restriction across patch sizes: the line-owner consumers' line ranges, the
    helper warp and the partial hand-over for every tile shape (one tile of p groups at p <= 9,
    two tiles of p / 2 groups above; clipped first / last windows; p = 17 keeps one warp per
    group and is covered above)."""
    test_pool_restrict_order3_unknown_counts(th, 59, p)


@pytest.mark.parametrize("scheme", ("tensor_linear", "order2", "order3"))
def test_interp_into_fine_patches(th, scheme):
    """Interpolation written into the fine patches' reference target cells equals the slab run."""
    import torch

    p, k, u = 9, 3, 7
    rng = np.random.default_rng(5)
    E = p + 2 * k
    n_face = 12
    coarse = rng.standard_normal((4, E ** 3 * u))
    fine = np.zeros((n_face, E ** 3 * u))
    cid = rng.integers(0, 4, n_face)
    nrm, sid, seg = np.arange(n_face) % 3, (np.arange(n_face) // 3) % 2, rng.integers(0, 9, n_face)
    dev = torch.device("cuda")
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    src = torch.from_numpy(coarse.reshape(-1)).to(dev)
    slab = torch.zeros(n_face * k * p * p * u, dtype=torch.float64, device=dev)
    th.FaceBatch(op, th.pool_interp_faces(p, k, u, cid, nrm, sid, seg), u).launch(src, slab)
    fdst = torch.from_numpy(fine.reshape(-1)).to(dev)
    rec = th.pool_interp_faces(p, k, u, cid, nrm, sid, seg, fine_ids=np.arange(n_face))
    th.FaceBatch(op, rec, u).launch(src, fdst)
    slab = slab.cpu().numpy().reshape(n_face, -1)
    fp = fdst.cpu().numpy().reshape(n_face, E, E, E, u)
    for f in range(n_face):
        lo, ext = [k, k, k], [p, p, p]
        lo[nrm[f]] = k if sid[f] == 0 else p
        ext[nrm[f]] = k
        box = fp[f, lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]].reshape(-1)
        assert np.array_equal(box, slab[f])
        fp[f, lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]] = 0.0
    assert not fp.any()  # nothing written outside the target boxes


@pytest.mark.parametrize("scheme", ("tensor_linear", "order2", "order3"))
def test_interp_wide_target_strides(th, scheme):
    """Target strides beyond 2^21 elements take the kernels' 64-bit offset path; the values
    must equal those written through compact slabs bit for bit."""
    import torch

    p, k, u = 9, 3, 59
    rng = np.random.default_rng(77)
    E = p + 2 * k
    n_patch, n_face = 4, 3
    pool = torch.from_numpy(rng.standard_normal(n_patch * E ** 3 * u)).to("cuda")
    nrm, sid, seg = np.array([0, 1, 2]), np.array([0, 1, 0]), np.array([4, 0, 8])
    rec = th.pool_interp_faces(p, k, u, rng.integers(0, n_patch, n_face), nrm, sid, seg)
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    ncell = k * p * p
    dst = torch.full((n_face * ncell * u,), np.nan, dtype=torch.float64, device="cuda")
    th.FaceBatch(op, rec, u).launch(pool, dst)
    want = dst.cpu().numpy().reshape(n_face, ncell * u)
    wide = rec.copy()
    # t1 / z strides spread out, z beyond 2^21 elements for every face
    scale = np.ones((n_face, 3), dtype=np.int64)
    scale[:, 1] = 7
    scale[:, 2] = 2 ** 21 // rec["dst_stride"][:, 2] + 1
    wide["dst_stride"] = rec["dst_stride"] * scale
    span = int((wide["dst_stride"] * (np.where(np.arange(3)[None, :] == nrm[:, None], k, p) - 1)).sum(1).max()) + u
    wide["dst"] = np.arange(n_face, dtype=np.int64) * span
    assert (wide["dst_stride"].max(1) >= 2 ** 21).all()
    big = torch.full((n_face * span,), np.nan, dtype=torch.float64, device="cuda")
    th.FaceBatch(op, wide, u).launch(pool, big)
    big = big.cpu().numpy()
    for f in range(n_face):
        ext = np.where(np.arange(3) == nrm[f], k, p)
        c = np.arange(ncell)
        x, y, z = c % ext[0], (c // ext[0]) % ext[1], c // (ext[0] * ext[1])
        base = wide["dst"][f] + x * wide["dst_stride"][f, 0] + y * wide["dst_stride"][f, 1] + z * wide["dst_stride"][f, 2]
        got = big[(base[:, None] + np.arange(u)[None, :]).reshape(-1)]
        assert np.array_equal(got, want[f]), (scheme, f)


@pytest.mark.parametrize("scheme", ("tensor_linear", "order2", "order3"))
def test_interp_batch_nonfinite_flag(th, scheme):
    """A NaN / Inf inside a face's support raises the batch's non-finite flag (every
    interpolation kernel: staged tiles, per-warp slide); a finite pool does not."""
    import torch

    p, k, u = 9, 3, 59
    E = p + 2 * k
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    rec = th.pool_interp_faces(p, k, u, [1, 0], [2, 0], [0, 1], [4, 0])
    batch = th.FaceBatch(op, rec, u)
    src = torch.zeros(2 * E ** 3 * u, dtype=torch.float64, device="cuda")
    out = torch.empty(2 * k * p * p * u, dtype=torch.float64, device="cuda")
    batch.launch(src, out)
    assert not batch.nonfinite()
    for bad in (float("nan"), float("inf")):
        src.zero_()
        # coarse patch 1, normal z, side 0: support layers [p, p + 2k) around segment 4's cells
        src.view(2, E, E, E, u)[1, p + 2, k + 4, k + 4, 58] = bad
        batch.launch(src, out)
        assert batch.nonfinite(), (scheme, bad)
