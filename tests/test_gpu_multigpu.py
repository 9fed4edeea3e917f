"""The cross-GPU path on ONE GPU: config-5-shaped sweeps of 2-4 simulated ranks in one
process (one source tensor per rank, the real sm_100a kernels and th_copy_boxes
packing / unpacking; the NCCL send/recv replaced by LoopbackTransport's device copies,
which match messages exactly as NCCL P2P does).  Every output face of every rank —
local, computed from received source boxes (staged), or received as a result — is
checked against the oracle, and against the single-rank sweep bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALE = 0.003  # 98 patches, 589 faces of config 5's shape (p = 9, k = 3, u = 59, order3)


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_15814_b200 as th

    return th, torch


def _simulate(th, torch, world, straddle, faces_world=None, p=None, scheme="order3", scale=SCALE):
    """Sweep of config-5-shaped faces (generated for `faces_world` ranks) over `world`
    simulated ranks."""
    import dataclasses

    import workloads as W
    from paper_2504_15814_b200.multigpu import LoopbackTransport, Partition, Support, make_rank_sweep, plan_sweep

    wl0 = W.describe_multi(faces_world or world, scale=scale, straddle=straddle, p=p)
    wl0 = dataclasses.replace(wl0, part=Partition(wl0.spec.n_patches, world))
    s = wl0.spec
    p, k, u = s.p, s.k, s.u
    ops = {r: th.operators.DEFAULT_CACHE.device_operator(r, scheme, p, k) for r in ("interpolate", "restrict")}
    support = Support.from_operators(ops["interpolate"], ops["restrict"], p, k)
    hub = LoopbackTransport(world)
    ranks = []
    for r in range(world):
        plan = plan_sweep(wl0.part, wl0.coarse, wl0.fine, wl0.segment, r, wl0.normal, wl0.side, support=support)
        src = torch.zeros(plan.src_elems(p, k, u), dtype=torch.float64, device="cuda")
        W.fill_pool(wl0, r, src)
        sweep, comp = make_rank_sweep(plan, ops, support, p, k, u, src, hub.endpoint(r), wl0.coarse, wl0.fine,
                                      wl0.normal, wl0.side, wl0.segment, int(wl0.part.bounds[r]))
        ranks.append((plan, sweep, comp, src))
    for _ in range(2):  # twice: buffers are reused across sweeps
        for plan, sweep, comp, _ in ranks:
            sweep.pre(comp)
        for plan, sweep, comp, _ in ranks:
            sweep.local(comp)
        hub.deliver()
        for plan, sweep, comp, _ in ranks:
            sweep.post(comp)
    torch.cuda.synchronize()
    for _, _, comp, _ in ranks:
        assert not comp.nonfinite()
    per = k * p * p * u
    results = {}
    kinds = {}
    for plan, sweep, comp, _ in ranks:
        for role, rp in plan.items():
            out = sweep.out[role][: rp.n_out * per].view(rp.n_out, per).cpu()
            nl, ns = rp.local.size, rp.staged.size
            for j, f in enumerate(rp.out_order()):
                assert (role, int(f)) not in results
                results[(role, int(f))] = out[j]
                kinds[(role, int(f))] = "local" if j < nl else "staged" if j < nl + ns else "received"
    assert len(results) == 2 * s.n_faces
    return wl0, results, kinds


def _oracle_check(wl, results, kinds, scheme="order3"):
    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    s = wl.spec
    vals = W.patch_values(wl, np.arange(s.n_patches))
    patches = {g: vals[g] for g in range(s.n_patches)}
    jobs = []
    for (role, f), got in results.items():
        seg = int(wl.segment[f]) if role == "interpolate" else 0
        cfg = OG.FaceCfg("xyz"[int(wl.normal[f])], ("negative", "positive")[int(wl.side[f])], seg, s.p, s.k, s.u)
        ex = OE.exchange_for(cfg, scheme, role)
        jobs.append((ex, W.face_source(wl, f, role, patches), np.empty(ex.n_out), got.numpy(), kinds[(role, f)]))
    st = OE.run_many([j[0] for j in jobs], [j[1] for j in jobs], [j[2] for j in jobs], 8)
    assert (st == 0).all()
    worst = {}
    for ex, src, want, got, kind in jobs:
        err = float(np.abs(got - want).max() / np.abs(want).max())
        worst[kind] = max(worst.get(kind, 0.0), err)
    return worst


@pytest.mark.parametrize("world,straddle", [(2, 0.0), (3, 0.15), (4, 0.15)])
def test_simulated_ranks_match_oracle_and_single_rank(env, world, straddle):
    th, torch = env
    wl, res_n, kinds = _simulate(th, torch, world, straddle)
    counts = {k: sum(1 for v in kinds.values() if v == k) for k in ("local", "staged", "received")}
    assert counts["staged"] > 0 and counts["received"] > 0, counts
    worst = _oracle_check(wl, res_n, kinds)
    assert set(worst) == {"local", "staged", "received"}
    assert max(worst.values()) <= 1e-12, worst
    # where a face is computed does not change its arithmetic: bitwise equal to one rank
    _, res_1, kinds_1 = _simulate(th, torch, 1, straddle, faces_world=world)
    assert set(kinds_1.values()) == {"local"}
    for key, v in res_n.items():
        assert torch.equal(v, res_1[key]), key


@pytest.mark.parametrize("p,scheme", [(17, "order3"), (17, "order2"), (9, "tensor_linear"), (9, "matrix_linear")])
def test_simulated_ranks_other_schemes(env, p, scheme):
    """The same cross-GPU path for the other schemes and for p = 17 (segments that cut coarse
    blocks; source boxes of up to 11 x 11 cells): 3 simulated ranks with straddling faces."""
    th, torch = env
    scale = 0.0015 if p == 17 else SCALE
    wl, res_n, kinds = _simulate(th, torch, 3, 0.15, p=p, scheme=scheme, scale=scale)
    counts = {k: sum(1 for v in kinds.values() if v == k) for k in ("local", "staged", "received")}
    assert counts["staged"] > 0 and counts["received"] > 0, counts
    worst = _oracle_check(wl, res_n, kinds, scheme)
    assert max(worst.values()) <= 1e-12, worst
    _, res_1, _ = _simulate(th, torch, 1, 0.15, faces_world=3, p=p, scheme=scheme, scale=scale)
    for key, v in res_n.items():
        assert torch.equal(v, res_1[key]), key
