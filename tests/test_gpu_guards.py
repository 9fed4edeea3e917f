"""Guard-band tests of the batch kernels (compute-sanitizer is not available on the GPU pool, so
out-of-bounds behaviour is checked by construction): the patch pool sits between NaN guards and the
target between sentinel guards inside larger allocations, at both 8-byte alignments of the first
cell.  A kernel that writes outside its targets breaks a sentinel; one that USES a value from
outside the pool (the staged restriction's widened bulk copies and its lanes past u read a few
doubles beyond their cells by design, and must discard them) turns a result into NaN or raises the
batch's non-finite flag; and the results must equal the unguarded run's bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ("tensor_linear", "matrix_linear", "order2", "order3")
GUARD = 4096
SENTINEL = -12345.678


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    return th, torch


def _records(th, role, p, k, u, n_patch, n_face, rng):
    nrm = rng.integers(0, 3, n_face)
    sid = rng.integers(0, 2, n_face)
    if role == "interpolate":
        cid = rng.integers(0, n_patch, n_face)
        # the first and the last patch of the pool are always used: their cells border the guards
        cid[0], cid[-1] = 0, n_patch - 1
        return th.pool_interp_faces(p, k, u, cid, nrm, sid, rng.integers(0, 9, n_face)), k * p * p * u
    fine = rng.integers(0, n_patch, (n_face, 9))
    fine[0, :], fine[-1, :] = 0, n_patch - 1
    return th.pool_restrict_faces(p, k, u, fine, nrm, sid), k * p * p * u


@pytest.mark.parametrize("shift", (0, 1))
@pytest.mark.parametrize("role", ("interpolate", "restrict"))
@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("p,u,n_face", ((9, 59, 400), (17, 59, 150), (5, 7, 500), (9, 64, 200)))
def test_guards_untouched_and_unused(env, scheme, role, p, u, n_face, shift):
    th, torch = env
    k = 3
    if scheme == "order3" and p < 5:
        pytest.skip("infeasible")
    rng = np.random.default_rng(1000 * p + u + (role == "restrict"))
    E = p + 2 * k
    n_patch = 10
    rec, per = _records(th, role, p, k, u, n_patch, n_face, rng)
    op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
    batch = th.FaceBatch(op, rec, u)
    dev = torch.device("cuda")
    pool = torch.from_numpy(rng.standard_normal(n_patch * E ** 3 * u)).to(dev)
    n_src, n_dst = pool.numel(), n_face * per

    ref = torch.full((n_dst,), float("nan"), dtype=torch.float64, device=dev)
    batch.launch(pool, ref)
    assert not batch.nonfinite()
    assert bool(torch.isfinite(ref).all())

    g = GUARD + shift  # shift = 1: the first cell sits on the other 8-byte alignment
    big_src = torch.full((g + n_src + GUARD,), float("nan"), dtype=torch.float64, device=dev)
    big_src[g:g + n_src] = pool
    big_dst = torch.full((g + n_dst + GUARD,), SENTINEL, dtype=torch.float64, device=dev)
    batch.launch(big_src[g:g + n_src], big_dst[g:g + n_dst])
    torch.cuda.synchronize()
    assert not batch.nonfinite(), "a value from outside the pool reached a result"
    assert bool((big_dst[:g] == SENTINEL).all()) and bool((big_dst[g + n_dst:] == SENTINEL).all()), \
        "write outside the target"
    assert torch.equal(big_dst[g:g + n_dst], ref), "results depend on the buffers' placement"
    assert bool(torch.isnan(big_src[:g]).all()) and bool(torch.isnan(big_src[g + n_src:]).all())


@pytest.mark.parametrize("scheme", ("order2", "order3"))
def test_interp_into_patches_leaves_other_cells(env, scheme):
    """Interpolation written into fine patches: every cell that is not a face's target keeps its
    sentinel (the kernels store only the children inside the face's ghost layers)."""
    th, torch = env
    p, k, u = 9, 3, 59
    rng = np.random.default_rng(5)
    E = p + 2 * k
    n_patch, n_face = 6, 60
    dev = torch.device("cuda")
    cid = rng.integers(0, n_patch, n_face)
    nrm, sid, seg = rng.integers(0, 3, n_face), rng.integers(0, 2, n_face), rng.integers(0, 9, n_face)
    # one fine patch per face, so no two faces write the same patch
    rec_p = th.pool_interp_faces(p, k, u, cid, nrm, sid, seg, fine_ids=np.arange(n_face))
    rec_s = th.pool_interp_faces(p, k, u, cid, nrm, sid, seg)
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", scheme, p, k)
    src = torch.from_numpy(rng.standard_normal(n_patch * E ** 3 * u)).to(dev)
    slab = torch.empty(n_face * k * p * p * u, dtype=torch.float64, device=dev)
    th.FaceBatch(op, rec_s, u).launch(src, slab)
    fine = torch.full((n_face * E ** 3 * u,), SENTINEL, dtype=torch.float64, device=dev)
    th.FaceBatch(op, rec_p, u).launch(src, fine)
    written = fine != SENTINEL
    assert int(written.sum()) == n_face * k * p * p * u
    assert torch.equal(torch.sort(fine[written]).values, torch.sort(slab).values)


@pytest.mark.parametrize("role,scheme,p,n_face", (("interpolate", "order3", 9, 3000), ("interpolate", "order3", 17, 1200),
                                                  ("interpolate", "order2", 17, 1200), ("interpolate", "tensor_linear", 17, 1200),
                                                  ("interpolate", "order2", 9, 3000), ("restrict", "order3", 9, 600),
                                                  ("restrict", "order3", 17, 300), ("restrict", "order2", 9, 600)))
def test_repeated_launches_bitwise_identical(env, role, scheme, p, n_face):
    """Hand-off stress for the persistent kernels (slice ring, warp-specialised tiles, staged
    restriction): every CTA walks tens of tiles through its rings; 25 launches of the same batch,
    alternating with a launch that overwrites the target, must give the same bits every time (a
    slot read before it is published, or recycled before its last reader, would not)."""
    th, torch = env
    k, u = 3, 59
    rng = np.random.default_rng(p + n_face)
    E = p + 2 * k
    n_patch = 16
    rec, per = _records(th, role, p, k, u, n_patch, n_face, rng)
    op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
    batch = th.FaceBatch(op, rec, u)
    dev = torch.device("cuda")
    pool = torch.from_numpy(rng.standard_normal(n_patch * E ** 3 * u)).to(dev)
    first = torch.empty(n_face * per, dtype=torch.float64, device=dev)
    batch.launch(pool, first)
    out = torch.empty_like(first)
    for it in range(25):
        out.fill_(float(it))
        batch.launch(pool, out)
        assert torch.equal(out, first), f"launch {it} differs"
    assert not batch.nonfinite()
