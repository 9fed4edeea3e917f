"""Multi-GPU layer host logic on CPU: partition, ownership plan, source-box shipping,
staging of straddling restriction blocks and the grouped P2P exchange.

The kernels are replaced by a stub that reads every face's source cells through the
same face records the GPU batches use (the kernels' address arithmetic, restated in
numpy) and writes a checksum of them, so a misplaced pack / unpack / receive offset or
record shows up as a wrong checksum.  World sizes 1-4 in one process (loopback
transport) and 2 and 4 over gloo (the NCCL code path with the gloo backend)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_15814_b200 import _native
from paper_2504_15814_b200.multigpu import (
    LoopbackTransport,
    NcclTransport,
    Partition,
    Support,
    Sweep,
    attach_source,
    batch_ids,
    face_records,
    pack_records,
    plan_sweep,
    unpack_records,
)

P, K, U = 4, 2, 3
E = P + 2 * K
PATCH = E ** 3 * U
# order3-like supports (reference coordinates): the segment boxes are smaller than the output
SUPPORT = Support(P, K, tuple((1, 3, (s % 3 > 0) * 1, 3, (s // 3 > 0) * 1, 3) for s in range(9)), (1, 3))


def make_faces(n_patches, n_faces, world, seed=0, cross=0.3, straddle=0.15):
    rng = np.random.default_rng(seed)
    part = Partition(n_patches, world)
    coarse = rng.integers(0, n_patches, n_faces)
    c_own = part.owner(coarse)
    f_own = c_own.copy()
    flip = rng.random(n_faces) < cross
    if world > 1:
        f_own[flip] = (c_own[flip] + rng.integers(1, world, flip.sum())) % world
    fine = np.stack([rng.integers(part.bounds[r], part.bounds[r + 1], 9) for r in f_own])
    if world > 1:  # some faces whose nine fine patches straddle ranks
        st = rng.random(n_faces) < straddle
        fine[st, rng.integers(0, 9, st.sum())] = rng.integers(0, n_patches, st.sum())
    seg = rng.integers(0, 9, n_faces)
    normal = rng.integers(0, 3, n_faces)
    side = rng.integers(0, 2, n_faces)
    return part, coarse, fine, seg, normal, side


def global_pool(n_patches):
    return np.random.default_rng(99).standard_normal(n_patches * PATCH)


def read_face(src, rec, role, support=SUPPORT, p=P, k=K, u=U):
    """Source values a kernel reads for one face record (reference order), from the flat
    source array: the decode_face / src_addr arithmetic of csrc/trihalo.cu in numpy."""
    n, sd = int(rec["normal"]), int(rec["side"])
    t1 = 1 if n == 0 else 0
    t2 = 1 if n == 2 else 2
    st = rec["src_stride"]
    ssn = int(st[n])
    sn = -ssn if sd else ssn
    sadj = (2 * k - 1) * ssn if sd else 0
    q = np.arange(u)
    vals = []
    if role == "interpolate":
        l0, c0, l1, c1, l2, c2 = support.interp[int(rec["segment"])]
        for a2 in range(l2, l2 + c2):
            for a1 in range(l1, l1 + c1):
                for a0 in range(l0, l0 + c0):
                    a = int(rec["src"][0]) + sadj + a0 * sn + a1 * int(st[t1]) + a2 * int(st[t2])
                    vals.append(src[a + q])
    else:
        l0, c0 = support.restrict
        for b in range(9):
            for a2 in range(p):
                for a1 in range(p):
                    for a0 in range(l0, l0 + c0):
                        a = int(rec["src"][b]) + sadj + a0 * sn + a1 * int(st[t1]) + a2 * int(st[t2])
                        vals.append(src[a + q])
    return np.concatenate(vals)


def expected_face(pool, f, role, coarse, fine, seg, normal, side, support=SUPPORT, p=P, k=K, u=U):
    """The same values straight from the global pool (world coordinates inside patches)."""
    g = pool.reshape(-1, E, E, E, u)
    n, sd = int(normal[f]), int(side[f])
    t1 = 1 if n == 0 else 0
    t2 = 1 if n == 2 else 2
    vals = []

    def cell(pid, wn, w1, w2):
        idx = [0, 0, 0]
        idx[n], idx[t1], idx[t2] = wn, w1, w2
        return g[pid, idx[2], idx[1], idx[0]]

    if role == "interpolate":
        l0, c0, l1, c1, l2, c2 = support.interp[int(seg[f])]
        ns = p if sd == 0 else 0
        for a2 in range(l2, l2 + c2):
            for a1 in range(l1, l1 + c1):
                for a0 in range(l0, l0 + c0):
                    vals.append(cell(int(coarse[f]), ns + (2 * k - 1 - a0 if sd else a0), k + a1, k + a2))
    else:
        l0, c0 = support.restrict
        nf = 0 if sd == 0 else p
        for b in range(9):
            for a2 in range(p):
                for a1 in range(p):
                    for a0 in range(l0, l0 + c0):
                        vals.append(cell(int(fine[f, b]), nf + (2 * k - 1 - a0 if sd else a0), k + a1, k + a2))
    return np.concatenate(vals)


def weights(n):
    return np.random.default_rng(n).standard_normal(n)


def checksum(vals):
    return float(vals @ weights(vals.size))


def copy_boxes_np(src, dst, rec, u=U):
    """numpy restatement of th_copy_boxes."""
    import torch

    r = np.frombuffer(rec.numpy().tobytes(), dtype=_native.BOX_DTYPE) if isinstance(rec, torch.Tensor) else rec
    s_np, d_np = src.numpy(), dst.numpy()
    for b in r:
        ex, ey, ez = (int(v) for v in b["ext"])
        for z in range(ez):
            for y in range(ey):
                for x in range(ex):
                    so = int(b["src"]) + x * int(b["src_stride"][0]) + y * int(b["src_stride"][1]) + z * int(b["src_stride"][2])
                    do = int(b["dst"]) + x * int(b["dst_stride"][0]) + y * int(b["dst_stride"][1]) + z * int(b["dst_stride"][2])
                    d_np[do:do + u] = s_np[so:so + u]


def _rank_setup(part, coarse, fine, seg, normal, side, rank, pool, transport):
    import torch

    plan = plan_sweep(part, coarse, fine, seg, rank, normal, side, support=SUPPORT)
    lo, hi = int(part.bounds[rank]), int(part.bounds[rank + 1])
    src = torch.zeros(plan.src_elems(P, K, U), dtype=torch.float64)
    src[: (hi - lo) * PATCH] = torch.from_numpy(pool[lo * PATCH:hi * PATCH])
    boxes = [b for b in plan.src_send if b.size]
    pack = pack_records(np.concatenate(boxes), SUPPORT, P, K, U, lo) if boxes else None
    unpack = unpack_records(plan, SUPPORT, P, K, U)
    sweep = Sweep(plan, K * P * P * U, torch.device("cpu"), torch.float64, transport, src=src, u=U,
                  copy_boxes=copy_boxes_np, pack=pack, unpack=unpack if unpack.size else None)
    attach_source(sweep, plan, src, P, K, U)
    recs = {}
    for role in plan.roles:
        for kind in ("send", "local", "staged"):
            ids = batch_ids(plan, role, kind)
            if ids.size:
                recs[(role, kind)] = face_records(plan, role, kind, ids, SUPPORT, P, K, U, coarse, fine, normal,
                                                  side, seg, lo)
    calls = []

    def compute(role, kind, ids, out):
        calls.append((role, kind, ids.size))
        rec = recs[(role, kind)]
        assert rec.size == ids.size
        pf = K * P * P * U
        o = out.numpy().reshape(ids.size, pf)
        for i, f in enumerate(ids):
            o[i, 0] = checksum(read_face(src.numpy(), rec[i], role))
            o[i, 1:] = f
    return plan, sweep, compute, calls


def _check_outputs(plan, sweep, pool, coarse, fine, seg, normal, side):
    pf = K * P * P * U
    for role, rp in plan.items():
        got = sweep.out[role][: rp.n_out * pf].numpy().reshape(-1, pf)
        order = rp.out_order()
        assert np.array_equal(got[:, 1:], np.repeat(order[:, None], pf - 1, axis=1).astype(float)), role
        for j, f in enumerate(order):
            want = checksum(expected_face(pool, f, role, coarse, fine, seg, normal, side))
            assert abs(got[j, 0] - want) <= 1e-9 * (1 + abs(want)), (role, f, got[j, 0], want)


def test_partition_and_plan_cover_every_face_once():
    for world in (1, 2, 3, 4):
        part, coarse, fine, seg, normal, side = make_faces(50, 400, world, seed=world)
        assert part.owner(part.bounds[:-1]).tolist() == list(range(world))
        plans = [plan_sweep(part, coarse, fine, seg, r, normal, side, support=SUPPORT) for r in range(world)]
        for role in ("interpolate", "restrict"):
            seen_out, seen_comp = [], []
            for r in range(world):
                rp = plans[r][role]
                seen_out.extend(rp.out_order().tolist())
                seen_comp.extend(rp.local.tolist() + rp.staged.tolist() + rp.send_order().tolist())
                for peer in range(world):  # what r sends to peer is what peer receives from r
                    assert np.array_equal(rp.send[peer], plans[peer][role].recv[r])
            assert sorted(seen_out) == list(range(400)) and sorted(seen_comp) == list(range(400))
        for r in range(world):
            for q in range(world):  # source boxes: sender and receiver agree on the list
                assert np.array_equal(plans[r].src_send[q], plans[q].src_recv[r])
            rp = plans[r]["interpolate"]
            # local / sent faces read local coarse patches; staged ones received their box
            assert (part.owner(coarse[np.concatenate([rp.local, rp.send_order()])]) == r).all()
            assert (part.owner(fine[rp.staged, seg[rp.staged]]) == r).all()
            rr = plans[r]["restrict"]
            comp = np.concatenate([rr.local, rr.send_order()])
            assert (part.owner(fine[comp]) == r).all()
            assert (part.owner(coarse[rr.staged]) == r).all()
        if world > 1:  # the generator produces every kind of cross face
            assert any(plans[r]["restrict"].staged.size for r in range(world))
            assert any(plans[r]["interpolate"].staged.size for r in range(world))
            assert any(plans[r]["restrict"].n_send for r in range(world))


def test_straddling_restriction_needs_support():
    part, coarse, fine, seg, normal, side = make_faces(40, 200, 2, seed=3)
    with pytest.raises(ValueError):
        plan_sweep(part, coarse, fine, seg, 0, normal, side)


@pytest.mark.parametrize("world", (1, 2, 3, 4))
def test_loopback_sweep_reads_the_right_sources(world):
    """All ranks in one process; every face's source cells, read through its record after
    packing, exchange, unpacking and staging, equal the global pool's cells."""
    part, coarse, fine, seg, normal, side = make_faces(24, 120, world, seed=10 + world)
    pool = global_pool(24)
    hub = LoopbackTransport(world)
    ranks = [_rank_setup(part, coarse, fine, seg, normal, side, r, pool, hub.endpoint(r)) for r in range(world)]
    for _, sweep, compute, _ in ranks:
        sweep.pre(compute)
    for _, sweep, compute, _ in ranks:
        sweep.local(compute)
    hub.deliver()
    for _, sweep, compute, _ in ranks:
        sweep.post(compute)
    for plan, sweep, _, _ in ranks:
        _check_outputs(plan, sweep, pool, coarse, fine, seg, normal, side)


def _worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    part, coarse, fine, seg, normal, side = make_faces(24, 150, world, seed=11)
    pool = global_pool(24)
    plan, sweep, compute, calls = _rank_setup(part, coarse, fine, seg, normal, side, rank, pool,
                                              NcclTransport(torch.device("cpu")))
    dist.barrier()
    sweep.run(compute)
    try:
        _check_outputs(plan, sweep, pool, coarse, fine, seg, normal, side)
        ok = True
    except AssertionError as exc:
        ok = repr(exc)
    dist.barrier()
    dist.destroy_process_group()
    result_q.put((rank, ok, calls))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", (2, 4))
def test_sweep_exchange_gloo(world):
    """The grouped P2P exchange of source boxes and results over gloo at world size 2 and 4
    (every rank sends to and receives from several peers in one batch)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok is True for _, ok, _ in res), res
    kinds = {kind for _, _, calls in res for _, kind, n in calls}
    assert {"send", "local", "staged"} <= kinds
