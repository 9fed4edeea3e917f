"""Same-level halo fill of the patch pool: the record builder
(`faces.pool_same_level_faces`, host logic, CPU) and the sm_100a copy through the C ABI
(`th_copy_faces`, GPU) against the oracle restatement `oracle.geometry.same_level_fill`.
A copy is bit-exact: every comparison here is `array_equal`."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import geometry as OG


def _pairs(rng, n_patches, n_faces):
    src = rng.integers(0, n_patches, n_faces)
    dst = (src + rng.integers(1, n_patches, n_faces)) % n_patches  # never the same patch
    return src, dst, rng.integers(0, 3, n_faces), rng.integers(0, 2, n_faces)


def _apply_records_numpy(pool_flat, rec, n_ext, t_ext, u):
    """Host emulation of th_copy_faces over the records (world strides, x fastest)."""
    out = pool_flat.copy()
    for r in rec:
        ext = [t_ext] * 3
        ext[int(r["normal"])] = n_ext
        for z in range(ext[2]):
            for y in range(ext[1]):
                for x in range(ext[0]):
                    s = r["src"][0] + x * r["src_stride"][0] + y * r["src_stride"][1] + z * r["src_stride"][2]
                    d = r["dst"] + x * r["dst_stride"][0] + y * r["dst_stride"][1] + z * r["dst_stride"][2]
                    out[d:d + u] = pool_flat[s:s + u]
    return out


@pytest.mark.parametrize("p,k,u", [(4, 1, 2), (5, 2, 3), (9, 3, 5)])
def test_records_match_oracle(p, k, u):
    from paper_2504_15814_b200.faces import pool_same_level_faces

    rng = np.random.default_rng(p * 10 + k)
    E = p + 2 * k
    n = 5
    pool = rng.standard_normal((n, E, E, E, u))
    src, dst, nrm, sid = _pairs(rng, n, 12)
    # one face per (normal, side) at least
    nrm[:6], sid[:6] = np.repeat(np.arange(3), 2), np.tile(np.arange(2), 3)
    rec = pool_same_level_faces(p, k, u, src, dst, nrm, sid)
    got = _apply_records_numpy(pool.ravel(), rec, k, p, u).reshape(pool.shape)
    want = OG.same_level_fill(pool, p, k, src, dst, nrm, sid)
    assert np.array_equal(got, want)
    # only halo cells of the destination patches changed
    changed = np.argwhere((got != pool).any(axis=-1))
    assert changed.size
    inside = ((changed[:, 1:] >= k) & (changed[:, 1:] < p + k)).all(axis=1)
    assert not inside.any()


@pytest.mark.gpu
@pytest.mark.parametrize("p,k,u,n_patches,n_faces", [(5, 2, 3, 6, 24), (9, 3, 59, 64, 384), (17, 3, 59, 8, 48)])
def test_copy_faces_bit_exact(p, k, u, n_patches, n_faces):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    rng = np.random.default_rng(n_faces)
    E = p + 2 * k
    pool = rng.standard_normal((n_patches, E, E, E, u))
    src, dst, nrm, sid = _pairs(rng, n_patches, n_faces)
    nrm[:6], sid[:6] = np.repeat(np.arange(3), 2), np.tile(np.arange(2), 3)
    # distinct (dst, normal, side) so no two faces write the same halo cells
    key = dst * 6 + nrm * 2 + sid
    _, keep = np.unique(key, return_index=True)
    src, dst, nrm, sid = src[keep], dst[keep], nrm[keep], sid[keep]
    rec = th.pool_same_level_faces(p, k, u, src, dst, nrm, sid)
    d = torch.from_numpy(pool.ravel().copy()).cuda()
    th.copy_faces(d, d, rec, k, p, u)
    torch.cuda.synchronize()
    want = OG.same_level_fill(pool, p, k, src, dst, nrm, sid)
    assert np.array_equal(d.cpu().numpy().reshape(pool.shape), want)


@pytest.mark.gpu
def test_copy_faces_empty_and_errors():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    d = torch.zeros(10, dtype=torch.float64, device="cuda")
    th.copy_faces(d, d, th.pool_same_level_faces(5, 2, 1, [], [], [], []), 2, 5, 1)  # empty batch: no-op
    with pytest.raises(th.ConfigurationError):
        th.copy_faces(d, d, th.pool_same_level_faces(5, 2, 1, [0], [1], [0], [0]), 0, 5, 1)
    with pytest.raises(th.ContractViolationError):
        th.copy_faces(d.float(), d, th.pool_same_level_faces(5, 2, 1, [0], [1], [0], [0]), 2, 5, 1)


@pytest.mark.gpu
def test_copy_faces_general_strides():
    """Target cells spaced two cells apart along x (not a contiguous run): the general path."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    p, k, u = 5, 2, 3
    E = p + 2 * k
    rng = np.random.default_rng(7)
    pool = rng.standard_normal((2, E, E, E, u))
    for normal in range(3):
        rec = th.pool_same_level_faces(p, k, u, [0], [1], [normal], [1])
        ext = [p, p, p]
        ext[normal] = k
        rec["dst"] = 0
        rec["dst_stride"] = [2 * u, 2 * u * ext[0], 2 * u * ext[0] * ext[1]]
        out = torch.zeros(2 * u * ext[0] * ext[1] * ext[2], dtype=torch.float64, device="cuda")
        th.copy_faces(torch.from_numpy(pool.ravel().copy()).cuda(), out, rec, k, p, u)
        got = out.cpu().numpy().reshape(ext[2], ext[1], ext[0], 2, u)[:, :, :, 0]
        idx = [slice(k, k + p)] * 3
        idx[2 - normal] = slice(k, 2 * k)
        assert np.array_equal(got, pool[(0, *idx)])
        assert not out.cpu().numpy().reshape(ext[2], ext[1], ext[0], 2, u)[:, :, :, 1].any()
