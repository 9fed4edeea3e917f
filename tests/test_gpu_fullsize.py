"""GPU tests at BASELINE.json's full sizes, through size-independent properties
(constant preservation, linearity) plus an oracle sample, and batch edge cases
(empty batch, non-finite detection)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ("tensor_linear", "matrix_linear", "order2", "order3")


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    return th, torch


def _batches(th, torch, p, k, u, n_face, n_patch, seed):
    rng = np.random.default_rng(seed)
    cid = rng.integers(0, n_patch, n_face)
    nrm = rng.integers(0, 3, n_face)
    sid = rng.integers(0, 2, n_face)
    seg = rng.integers(0, 9, n_face)
    fine = rng.integers(0, n_patch, (n_face, 9))
    rec_i = th.pool_interp_faces(p, k, u, cid, nrm, sid, seg)
    rec_r = th.pool_restrict_faces(p, k, u, fine, nrm, sid)
    return rec_i, rec_r, (cid, nrm, sid, seg, fine)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_config2_size_constant_and_linearity(env, scheme):
    """4,096 faces, p = 9, u = 59 (config 2 shape) for both roles."""
    th, torch = env
    p, k, u, n_face, n_patch = 9, 3, 59, 4096, 512
    E = p + 2 * k
    dev = torch.device("cuda")
    rec_i, rec_r, _ = _batches(th, torch, p, k, u, n_face, n_patch, 3)
    per = k * p * p * u
    gen = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(n_patch * E ** 3 * u, dtype=torch.float64, device=dev, generator=gen)
    b = torch.randn(n_patch * E ** 3 * u, dtype=torch.float64, device=dev, generator=gen)
    const = torch.full_like(a, 2.5)
    for role, rec in (("interpolate", rec_i), ("restrict", rec_r)):
        op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
        batch = th.FaceBatch(op, rec, u)
        outs = []
        for src in (const, a, b, 1.7 * a - 0.3 * b):
            out = torch.empty(n_face * per, dtype=torch.float64, device=dev)
            batch.launch(src, out)
            outs.append(out)
        assert not batch.nonfinite()
        assert float((outs[0] - 2.5).abs().max()) < 2e-11  # row sums are 1; extrapolating rows have L1 norm ~170
        lin = 1.7 * outs[1] - 0.3 * outs[2]
        assert float((outs[3] - lin).abs().max() / lin.abs().max()) < 1e-12


@pytest.mark.parametrize("scheme", ("order2", "order3"))
def test_config4_size_p17_oracle_sample(env, scheme):
    """p = 17 (config 4 shape), 6,144 faces per role; 12 sampled faces vs the oracle."""
    th, torch = env
    from oracle import exchange as OE
    from oracle import geometry as OG

    p, k, u, n_face, n_patch = 17, 3, 59, 6144, 96
    E = p + 2 * k
    dev = torch.device("cuda")
    rec_i, rec_r, (cid, nrm, sid, seg, fine) = _batches(th, torch, p, k, u, n_face, n_patch, 5)
    per = k * p * p * u
    pool = torch.randn(n_patch * E ** 3 * u, dtype=torch.float64, device=dev,
                       generator=torch.Generator(device="cuda").manual_seed(2))
    host = pool.cpu().numpy().reshape(n_patch, E, E, E, u)
    rng = np.random.default_rng(0)
    for role, rec in (("interpolate", rec_i), ("restrict", rec_r)):
        op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
        out = torch.empty(n_face * per, dtype=torch.float64, device=dev)
        th.FaceBatch(op, rec, u).launch(pool, out)
        got_all = out.cpu().numpy().reshape(n_face, per)
        for f in rng.choice(n_face, 12, replace=False):
            n, sd = int(nrm[f]), int(sid[f])
            t1, t2 = [d for d in range(3) if d != n]
            if role == "interpolate":
                lo, ext = [k, k, k], [p, p, p]
                lo[n], ext[n] = (p if sd == 0 else 0), 2 * k
                src = host[cid[f], lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]].reshape(-1)
                s = int(seg[f])
            else:
                ext = [3 * p, 3 * p, 3 * p]
                ext[n] = 2 * k
                box = np.zeros((ext[2], ext[1], ext[0], u))
                for bb in range(9):
                    lo, e = [k, k, k], [p, p, p]
                    lo[n], e[n] = (0 if sd == 0 else p), 2 * k
                    off = [0, 0, 0]
                    off[t1], off[t2] = (bb % 3) * p, (bb // 3) * p
                    box[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = \
                        host[fine[f, bb], lo[2]:lo[2] + e[2], lo[1]:lo[1] + e[1], lo[0]:lo[0] + e[0]]
                src = box.reshape(-1)
                s = 0
            ex = OE.exchange_for(OG.FaceCfg("xyz"[n], ("negative", "positive")[sd], s, p, k, u), scheme, role)
            want = np.empty(ex.n_out)
            ex.run(src, want)
            assert np.abs(got_all[f] - want).max() / np.abs(want).max() <= 1e-12


def test_empty_batch_and_nonfinite_flag(env):
    th, torch = env
    p, k, u = 9, 3, 59
    E = p + 2 * k
    dev = torch.device("cuda")
    op = th.operators.DEFAULT_CACHE.device_operator("interpolate", "order2", p, k)
    empty = th.FaceBatch(op, th.pool_interp_faces(p, k, u, [], [], [], []), u)
    src = torch.zeros(4 * E ** 3 * u, dtype=torch.float64, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    empty.launch(src, out)  # no-op
    assert not empty.nonfinite()
    rec = th.pool_interp_faces(p, k, u, [1], [2], [0], [4])
    batch = th.FaceBatch(op, rec, u)
    out = torch.empty(k * p * p * u, dtype=torch.float64, device=dev)
    # a NaN inside the face's support (coarse patch 1, normal z, side 0: layers [p, p+2k))
    src.view(4, E, E, E, u)[1, p + 2, k + 4, k + 4, 7] = float("nan")
    batch.launch(src, out)
    assert batch.nonfinite()
    assert not batch.nonfinite()  # read-and-clear


def test_pool_offsets_beyond_2_31_elements(env):
    """Config-5-sized element offsets: a pool of 11,000 patches (2.19e9 elements, 17.5 GB)
    whose faces read patches past element 2^31 -- every scheme, both roles, against the oracle,
    and the same-level copy bit for bit (64-bit offsets in every kernel)."""
    th, torch = env
    from oracle import exchange as OE
    from oracle import geometry as OG

    p, k, u = 9, 3, 59
    E = p + 2 * k
    patch = E ** 3 * u
    n_patch = 11000
    assert n_patch * patch > 2 ** 31
    dev = torch.device("cuda")
    free, _ = torch.cuda.mem_get_info()
    if free < 24 * 2 ** 30:
        pytest.skip("needs ~24 GB of free device memory")
    pool = torch.empty(n_patch * patch, dtype=torch.float64, device=dev)
    gen = torch.Generator(device="cuda").manual_seed(11)
    for a in range(0, n_patch, 1000):  # fill in slices (randn of 2e9 values at once needs 2x)
        b = min(n_patch, a + 1000)
        pool[a * patch:b * patch] = torch.randn((b - a) * patch, dtype=torch.float64, device=dev, generator=gen)
    rng = np.random.default_rng(4)
    hi = 2 ** 31 // patch + 1  # first patch entirely past element 2^31
    n_face = 24
    cid = rng.integers(hi, n_patch, n_face)
    nrm, sid, seg = rng.integers(0, 3, n_face), rng.integers(0, 2, n_face), rng.integers(0, 9, n_face)
    fine = rng.integers(hi, n_patch, (n_face, 9))
    need = np.unique(np.concatenate([cid, fine.ravel()]))
    host = {int(g): pool[g * patch:(g + 1) * patch].cpu().numpy().reshape(E, E, E, u) for g in need}
    per = k * p * p * u
    for scheme in ("tensor_linear", "matrix_linear", "order2", "order3"):
        for role in ("interpolate", "restrict"):
            rec = (th.pool_interp_faces(p, k, u, cid, nrm, sid, seg) if role == "interpolate"
                   else th.pool_restrict_faces(p, k, u, fine, nrm, sid))
            op = th.operators.DEFAULT_CACHE.device_operator(role, scheme, p, k)
            out = torch.empty(n_face * per, dtype=torch.float64, device=dev)
            th.FaceBatch(op, rec, u).launch(pool, out)
            got = out.cpu().numpy().reshape(n_face, per)
            for f in range(0, n_face, 3):
                n, sd = int(nrm[f]), int(sid[f])
                t1, t2 = [d for d in range(3) if d != n]
                if role == "interpolate":
                    lo, ext = [k, k, k], [p, p, p]
                    lo[n], ext[n] = (p if sd == 0 else 0), 2 * k
                    src = host[int(cid[f])][lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]]
                    src, s = src.reshape(-1), int(seg[f])
                else:
                    ext = [3 * p, 3 * p, 3 * p]
                    ext[n] = 2 * k
                    box = np.zeros((ext[2], ext[1], ext[0], u))
                    for bb in range(9):
                        lo, e = [k, k, k], [p, p, p]
                        lo[n], e[n] = (0 if sd == 0 else p), 2 * k
                        off = [0, 0, 0]
                        off[t1], off[t2] = (bb % 3) * p, (bb // 3) * p
                        box[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = \
                            host[int(fine[f, bb])][lo[2]:lo[2] + e[2], lo[1]:lo[1] + e[1], lo[0]:lo[0] + e[0]]
                    src, s = box.reshape(-1), 0
                ex = OE.exchange_for(OG.FaceCfg("xyz"[n], ("negative", "positive")[sd], s, p, k, u), scheme, role)
                want = np.empty(ex.n_out)
                ex.run(src, want)
                assert np.abs(got[f] - want).max() / np.abs(want).max() <= 1e-12, (scheme, role, f)
    # same-level halo copy between patches past 2^31
    src_ids, dst_ids = fine[:4, 0], fine[:4, 1]
    rec = th.pool_same_level_faces(p, k, u, src_ids, dst_ids, nrm[:4], sid[:4])
    if len(set(dst_ids.tolist())) == 4 and not set(src_ids.tolist()) & set(dst_ids.tolist()):
        th.copy_faces(pool, pool, rec, k, p, u)
        v = pool.view(n_patch, E, E, E, u)
        for i in range(4):
            ax = 2 - int(nrm[i])
            a = [slice(k, k + p)] * 3
            b = list(a)
            a[ax] = slice(p, p + k) if sid[i] == 0 else slice(k, 2 * k)
            b[ax] = slice(0, k) if sid[i] == 0 else slice(p + k, p + 2 * k)
            assert torch.equal(v[(int(src_ids[i]), *a)], v[(int(dst_ids[i]), *b)])
    del pool
    torch.cuda.empty_cache()
