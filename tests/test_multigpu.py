"""Multi-GPU layer host logic on CPU: partition, ownership plan and the grouped
P2P exchange, world sizes 2 and 4 over gloo (the kernels are replaced by a stamp so
the bookkeeping is checked exactly)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_15814_b200.multigpu import Partition, Sweep, plan_sweep


def make_faces(n_patches, n_faces, world, seed=0, cross=0.3):
    rng = np.random.default_rng(seed)
    part = Partition(n_patches, world)
    coarse = rng.integers(0, n_patches, n_faces)
    c_own = part.owner(coarse)
    f_own = c_own.copy()
    flip = rng.random(n_faces) < cross
    if world > 1:
        f_own[flip] = (c_own[flip] + rng.integers(1, world, flip.sum())) % world
    fine = np.stack([rng.integers(part.bounds[r], part.bounds[r + 1], 9) for r in f_own])
    seg = rng.integers(0, 9, n_faces)
    return part, coarse, fine, seg


def test_partition_and_plan_cover_every_face_once():
    for world in (1, 2, 3, 4):
        part, coarse, fine, seg = make_faces(50, 400, world, seed=world)
        assert part.owner(part.bounds[:-1]).tolist() == list(range(world))
        for role in ("interpolate", "restrict"):
            seen_out, seen_comp = [], []
            for r in range(world):
                plan = plan_sweep(part, coarse, fine, seg, r)[role]
                seen_out.extend(plan.out_order().tolist())
                seen_comp.extend(plan.local.tolist() + plan.send_order().tolist())
                for peer in range(world):  # what r sends to peer is what peer receives from r
                    other = plan_sweep(part, coarse, fine, seg, peer)[role]
                    assert np.array_equal(plan.send[peer], other.recv[r])
            assert sorted(seen_out) == list(range(400)) and sorted(seen_comp) == list(range(400))
        # computing rank owns the sources
        for r in range(world):
            plans = plan_sweep(part, coarse, fine, seg, r)
            comp_i = np.concatenate([plans["interpolate"].local, plans["interpolate"].send_order()])
            assert (part.owner(coarse[comp_i]) == r).all()
            comp_r = np.concatenate([plans["restrict"].local, plans["restrict"].send_order()])
            assert (part.owner(fine[comp_r, 0]) == r).all()


def stamp(role, face_ids, per_face):
    code = 0.5 if role == "interpolate" else 0.25
    return (face_ids[:, None] * 1000.0 + code + np.arange(per_face)[None, :]).reshape(-1)


def _worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    part, coarse, fine, seg = make_faces(40, 300, world, seed=11)
    plans = plan_sweep(part, coarse, fine, seg, rank)
    pf = 7
    sweep = Sweep(plans, pf, torch.device("cpu"), torch.float64)
    calls = []

    def compute(role, kind, ids, out):
        calls.append((role, kind, ids.size))
        out.copy_(torch.from_numpy(stamp(role, ids, pf)))

    sweep.run(compute)
    ok = True
    for role, plan in plans.items():
        got = sweep.out[role][: plan.n_out * pf].numpy()
        ok &= np.array_equal(got, stamp(role, plan.out_order(), pf))
    dist.barrier()
    dist.destroy_process_group()
    result_q.put((rank, bool(ok), calls))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", (2, 4))
def test_sweep_exchange_gloo(world):
    """The grouped P2P exchange of cross faces over gloo at world size 2 and 4 (every rank
    sends to and receives from several peers in one batch)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    # cross faces exist in both directions for both roles
    assert all(any(kind == "send" for _, kind, n in calls) for _, _, calls in res)
