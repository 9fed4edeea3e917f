"""Multi-GPU sweep: one process per GPU, patches block-partitioned, one P2P step.

SURVEY §8e: faces are independent; the only exchange is for faces whose coarse
and fine patches live on different GPUs.  Ownership rule (the GPU holding the
larger input computes):
  * interpolation of a face runs on the owner of its coarse patch and its
    result (k p^2 u values) belongs to the owner of the fine patch it fills;
  * restriction runs on the owner of its nine fine patches and its result
    (k p^2 u coarse halo values) belongs to the coarse owner.
Cross faces are therefore computed where their sources are and only their
~115 KB results travel, with one grouped send/recv per peer
(torch.distributed.batch_isend_irecv -> ncclGroupStart / ncclSend / ncclRecv
/ ncclGroupEnd on NCCL) issued on a side stream while the local faces run.

Output layout on every rank, per role: [local faces][faces received from
rank 0][from rank 1]...; results of faces sent away are computed into a send
buffer grouped by destination in the same order, so received blocks land
directly in place (no scatter).

``plan_sweep`` is pure host logic (numpy), identical on every rank; ``Sweep``
executes a plan with any face "compute" callable so that the exchange
bookkeeping can be tested on CPU with gloo (tests/test_multigpu.py); the
product compute is ``GpuCompute`` (the sm_100a kernels through the C ABI).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class Partition:
    """Block partition of patch ids 0..n-1 over `world` ranks (contiguous ranges)."""

    def __init__(self, n_patches: int, world: int):
        self.n, self.world = int(n_patches), int(world)
        self.bounds = np.array([(self.n * r) // self.world for r in range(self.world + 1)], dtype=np.int64)

    def owner(self, ids) -> np.ndarray:
        return np.searchsorted(self.bounds, np.asarray(ids, dtype=np.int64), side="right") - 1

    def local(self, ids, rank: int) -> np.ndarray:
        return np.asarray(ids, dtype=np.int64) - self.bounds[rank]

    def size(self, rank: int) -> int:
        return int(self.bounds[rank + 1] - self.bounds[rank])


@dataclass
class RolePlan:
    """Faces of one role as seen from one rank."""

    role: str
    local: np.ndarray                 # face ids computed here, result kept here
    send: list = field(default_factory=list)   # send[peer] = face ids computed here, result sent to peer
    recv: list = field(default_factory=list)   # recv[peer] = face ids computed by peer, result received here

    @property
    def n_out(self) -> int:
        return int(self.local.size + sum(r.size for r in self.recv))

    @property
    def n_send(self) -> int:
        return int(sum(s.size for s in self.send))

    def out_order(self) -> np.ndarray:
        """Face ids in this rank's output buffer order."""
        return np.concatenate([self.local] + list(self.recv)) if self.recv else self.local

    def send_order(self) -> np.ndarray:
        return np.concatenate(self.send) if self.send else np.zeros(0, dtype=np.int64)


def plan_sweep(part: Partition, coarse_ids, fine_ids, segments, rank: int, roles=("interpolate", "restrict")):
    """Per-role plans for `rank`.  fine_ids is (n_faces, 9); the interpolation target
    of face f is fine_ids[f, segment[f]]; restriction reads all nine (one owner)."""
    coarse_ids = np.asarray(coarse_ids, dtype=np.int64)
    fine_ids = np.asarray(fine_ids, dtype=np.int64).reshape(-1, 9)
    segments = np.asarray(segments, dtype=np.int64)
    c_own = part.owner(coarse_ids)
    f_own_all = part.owner(fine_ids)
    if not (f_own_all == f_own_all[:, :1]).all():
        raise ValueError("the nine fine patches of a face must live on one rank")
    f_own = f_own_all[:, 0]
    t_own = part.owner(fine_ids[np.arange(fine_ids.shape[0]), segments])  # interp target owner
    plans = {}
    for role in roles:
        comp, dest = (c_own, t_own) if role == "interpolate" else (f_own, c_own)
        mine = comp == rank
        plan = RolePlan(role, np.flatnonzero(mine & (dest == rank)))
        plan.send = [np.flatnonzero(mine & (dest == peer)) if peer != rank else np.zeros(0, dtype=np.int64)
                     for peer in range(part.world)]
        plan.recv = [np.flatnonzero((comp == peer) & (dest == rank)) if peer != rank else np.zeros(0, dtype=np.int64)
                     for peer in range(part.world)]
        plans[role] = plan
    return plans


class Sweep:
    """Executes one rank's plan: cross faces first (into the send buffer), P2P on a
    side stream overlapped with the local faces, received blocks land in place.

    compute(role, kind, face_ids, out_tensor), kind in {"send", "local"}, must
    write len(face_ids) results of `per_face` values each into out_tensor (a
    contiguous slice), in face_ids order."""

    def __init__(self, plans: dict, per_face: int, device, dtype, group=None, use_streams: bool = True):
        import torch

        self.plans, self.per_face, self.device, self.group = plans, int(per_face), device, group
        self.out = {r: torch.empty(max(1, p.n_out * self.per_face), dtype=dtype, device=device) for r, p in plans.items()}
        self.sendbuf = {r: torch.empty(max(1, p.n_send * self.per_face), dtype=dtype, device=device)
                        for r, p in plans.items()}
        self.use_streams = use_streams and device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(device=device) if self.use_streams else None

    def _p2p_ops(self, role: str):
        import torch.distributed as dist

        plan, pf = self.plans[role], self.per_face
        ops = []
        off = 0
        for peer, ids in enumerate(plan.send):
            if ids.size:
                ops.append(dist.P2POp(dist.isend, self.sendbuf[role][off * pf:(off + ids.size) * pf], peer, self.group))
            off += ids.size
        off = plan.local.size
        for peer, ids in enumerate(plan.recv):
            if ids.size:
                ops.append(dist.P2POp(dist.irecv, self.out[role][off * pf:(off + ids.size) * pf], peer, self.group))
            off += ids.size
        return ops

    def run(self, compute) -> None:
        import torch
        import torch.distributed as dist

        pf = self.per_face
        # 1. results that must leave this rank first
        for role, plan in self.plans.items():
            if plan.n_send:
                compute(role, "send", plan.send_order(), self.sendbuf[role][: plan.n_send * pf])
        ops = [op for role in self.plans for op in self._p2p_ops(role)]
        works = []
        if ops:
            if self.use_streams:
                ready = torch.cuda.Event()
                ready.record(torch.cuda.current_stream(self.device))
                self.comm_stream.wait_event(ready)
                with torch.cuda.stream(self.comm_stream):
                    works = dist.batch_isend_irecv(ops)
            else:
                works = dist.batch_isend_irecv(ops)
        # 2. local faces overlap the exchange
        for role, plan in self.plans.items():
            if plan.local.size:
                compute(role, "local", plan.local, self.out[role][: plan.local.size * pf])
        # 3. received blocks are in place once the P2P work completes
        for w in works:
            w.wait()
        if self.use_streams and ops:
            torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)


class GpuCompute:
    """Product compute for Sweep: prebuilt FaceBatches per (role, kind), records
    pointing at this rank's patch pool and at consecutive output slots."""

    def __init__(self, plans: dict, make_records, operators: dict, sources: dict, u: int):
        from .faces import FaceBatch

        self.sources = sources
        self.batches = {}
        for role, plan in plans.items():
            for kind, ids in (("send", plan.send_order()), ("local", plan.local)):
                if ids.size:
                    self.batches[(role, kind)] = FaceBatch(operators[role], make_records(role, ids), u)

    def __call__(self, role, kind, face_ids, out) -> None:
        self.batches[(role, kind)].launch(self.sources[role], out, check_flag=False)

    @property
    def launches(self) -> int:
        return len(self.batches)
