"""Multi-GPU sweep: one process per GPU, patches block-partitioned, one P2P step.

SURVEY §8e: faces are independent; the only exchange is for faces whose coarse
and fine patches live on different GPUs.  Per face the sweep moves whichever is
smaller, the source cells the kernels read or the result:

  * interpolation of a cross face (coarse patch on GPU c, the fine patch of its
    segment on GPU t != c): the coarse owner ships the face's source box — the
    union of the kernel windows of that segment (``th_operator_source_box``:
    5 x 5..7 x 5..7 coarse cells for order3 at p = 9, 75.8 KB on average) — and
    t computes, when that box is smaller than the k p^2 output (114.7 KB);
    otherwise c computes and ships the result;
  * restriction of a face whose nine fine patches all live on GPU a runs on a
    and, when a != coarse owner c, ships its k p^2-cell result to c (115 KB
    instead of 1-1.7 MB of fine support);
  * restriction of a face whose nine fine patches straddle GPUs runs on c: every
    remote fine block ships the normal layers its kernels read
    (``th_operator_support_layers`` x p x p cells), and c unpacks them into
    patch-shaped staging slots after its own pool, so the face's record addresses
    local and staged blocks alike.

One grouped send/recv per peer (torch.distributed.batch_isend_irecv ->
ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd on NCCL) carries both the
packed source boxes and the results, on a side stream while the local faces
run.  Faces computed from received sources ("staged") run after it.

Output layout on every rank, per role: [local][staged][received from rank 0]
[from rank 1]...; results of faces sent away are computed into a send buffer
grouped by destination in the same order, so received blocks land in place.

Source buffer of every rank (``SweepPlan.src_elems``): one tensor holding
[its pool of n_local patches][staging slots, patch-shaped][received source
boxes, compact x-fastest][guard]; all face records of the rank are element
offsets into it.

``plan_sweep`` is pure host logic (numpy), identical on every rank.  ``Sweep``
executes a plan through a transport (``NcclTransport``, or ``LoopbackTransport``
which runs several ranks' sweeps in one process — the one-GPU parity test of
the cross-GPU path) and a compute callable: ``GpuCompute`` (the sm_100a kernels
through the C ABI) or, in the CPU tests, a stub.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .faces import _records, _tangential, pool_geometry, world_box_strides

ROLES = ("interpolate", "restrict")


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
class Support:
    """Source cells the kernels read, in reference source coordinates.

    interp[s] = (lo0, n0, lo1, n1, lo2, n2) of segment s's 2k x p x p source region;
    restrict = (lo, n) normal layers of each fine block (all p x p tangential cells)."""

    p: int
    k: int
    interp: tuple
    restrict: tuple

    @classmethod
    def from_operators(cls, interp_op, restrict_op, p: int, k: int) -> "Support":
        return cls(p, k, tuple(interp_op.source_box(s) for s in range(9)), tuple(restrict_op.support_layers()))

    @classmethod
    def full(cls, p: int, k: int) -> "Support":
        return cls(p, k, tuple((0, 2 * k, 0, p, 0, p) for _ in range(9)), (0, 2 * k))

    def interp_cells(self) -> np.ndarray:
        return np.array([b[1] * b[3] * b[5] for b in self.interp], dtype=np.int64)

    @property
    def out_cells(self) -> int:
        return self.k * self.p * self.p

    @property
    def block_cells(self) -> int:
        return self.restrict[1] * self.p * self.p


@dataclass
class RolePlan:
    """Faces of one role as seen from one rank."""

    role: str
    local: np.ndarray                 # computed here from local sources, result kept here
    staged: np.ndarray = None         # computed here from (partly) received sources, kept here
    send: list = field(default_factory=list)   # send[peer] = computed here, result sent to peer
    recv: list = field(default_factory=list)   # recv[peer] = computed by peer, result received here

    def __post_init__(self):
        if self.staged is None:
            self.staged = np.zeros(0, dtype=np.int64)

    @property
    def n_out(self) -> int:
        return int(self.local.size + self.staged.size + sum(r.size for r in self.recv))

    @property
    def n_send(self) -> int:
        return int(sum(s.size for s in self.send))

    def out_order(self) -> np.ndarray:
        """Face ids in this rank's output buffer order."""
        return np.concatenate([self.local, self.staged] + list(self.recv))

    def send_order(self) -> np.ndarray:
        return np.concatenate(self.send) if self.send else np.zeros(0, dtype=np.int64)


BOXLIST_DTYPE = np.dtype([("kind", "<i8"), ("face", "<i8"), ("patch", "<i8"), ("normal", "<i8"), ("side", "<i8"),
                          ("segment", "<i8"), ("cells", "<i8")])


@dataclass
class SweepPlan:
    """Everything rank `rank` does in one sweep."""

    rank: int
    world: int
    n_local: int                       # patches of this rank's pool
    roles: dict                        # role -> RolePlan
    src_send: list                     # src_send[peer]: BOXLIST_DTYPE boxes packed here for peer
    src_recv: list                     # src_recv[peer]: boxes peer packs for this rank (same order)
    slots: np.ndarray                  # global fine patch ids staged here (slot i = patch n_local + i)
    restrict_src: dict = field(default_factory=dict)  # staged restriction face -> (9,) virtual patch ids

    def __getitem__(self, role):
        return self.roles[role]

    def items(self):
        return self.roles.items()

    @property
    def n_src_send_cells(self) -> int:
        return int(sum(b["cells"].sum() for b in self.src_send))

    @property
    def n_src_recv_cells(self) -> int:
        return int(sum(b["cells"].sum() for b in self.src_recv))

    def recv_cell_offsets(self) -> list:
        """Cell offset of every received box inside the received-box region, per peer."""
        out, off = [], 0
        for b in self.src_recv:
            c = np.cumsum(b["cells"]) - b["cells"] + off
            out.append(c)
            off += int(b["cells"].sum())
        return out

    def src_elems(self, p: int, k: int, u: int, guard_cells: int = 64) -> int:
        """Elements of this rank's source tensor: pool + staging slots + received boxes + guard."""
        patch = (p + 2 * k) ** 3 * u
        return (self.n_local + self.slots.size) * patch + (self.n_src_recv_cells + guard_cells) * u

    def recv_base(self, p: int, k: int, u: int) -> int:
        return (self.n_local + self.slots.size) * (p + 2 * k) ** 3 * u


def plan_sweep(part: Partition, coarse_ids, fine_ids, segments, rank: int, normals=None, sides=None,
               support: Support | None = None, roles=ROLES) -> SweepPlan:
    """Plan of `rank` (see the module docstring).  fine_ids is (n_faces, 9) global patch ids
    (block b1 + 3 b2); the interpolation target of face f is fine_ids[f, segments[f]]."""
    coarse_ids = np.asarray(coarse_ids, dtype=np.int64)
    fine_ids = np.asarray(fine_ids, dtype=np.int64).reshape(-1, 9)
    segments = np.asarray(segments, dtype=np.int64)
    nf = coarse_ids.size
    normals = np.zeros(nf, dtype=np.int64) if normals is None else np.asarray(normals, dtype=np.int64)
    sides = np.zeros(nf, dtype=np.int64) if sides is None else np.asarray(sides, dtype=np.int64)
    W = part.world
    c_own = part.owner(coarse_ids)
    f_own = part.owner(fine_ids)
    t_own = f_own[np.arange(nf), segments]
    none = np.zeros(0, dtype=np.int64)
    plans = {}
    boxes = {}  # (sender, receiver) -> list of box arrays
    restrict_src = {}
    slot_ids = []
    for role in roles:
        if role == "interpolate":
            cross = c_own != t_own
            if support is not None:
                ship_src = cross & (support.interp_cells()[segments] < support.out_cells)
            else:
                ship_src = np.zeros(nf, dtype=bool)
            comp = np.where(ship_src, t_own, c_own)
            dest = t_own
            needs_recv = ship_src
        else:
            same = (f_own == f_own[:, :1]).all(axis=1)
            comp = np.where(same, f_own[:, 0], c_own)
            dest = c_own
            needs_recv = ~same
        mine = comp == rank
        plan = RolePlan(role, np.flatnonzero(mine & (dest == rank) & ~needs_recv),
                        np.flatnonzero(mine & (dest == rank) & needs_recv))
        plan.send = [np.flatnonzero(mine & (dest == peer)) if peer != rank else none for peer in range(W)]
        plan.recv = [np.flatnonzero((comp == peer) & (dest == rank)) if peer != rank else none for peer in range(W)]
        if role == "interpolate":  # coarse-patch order: contiguous pool ranges (e2e pipelining, L2 reuse)
            plan.local = plan.local[np.argsort(coarse_ids[plan.local], kind="stable")]
        plans[role] = plan
        # source boxes shipped between every (sender, receiver) pair that involves this rank
        if role == "interpolate" and support is not None:
            cells = support.interp_cells()
            f = np.flatnonzero(ship_src & ((c_own == rank) | (t_own == rank)))
            for s_, r_ in set(zip(c_own[f].tolist(), t_own[f].tolist())):
                g = f[(c_own[f] == s_) & (t_own[f] == r_)]
                b = np.zeros(g.size, dtype=BOXLIST_DTYPE)
                b["kind"], b["face"], b["patch"] = 0, g, coarse_ids[g]
                b["normal"], b["side"], b["segment"], b["cells"] = normals[g], sides[g], segments[g], cells[segments[g]]
                boxes.setdefault((s_, r_), []).append(b)
        elif role == "restrict":
            st = np.flatnonzero(~same)
            if st.size and support is None:
                raise ValueError("faces whose nine fine patches straddle ranks need `support`")
            bc = support.block_cells if support is not None else 0
            for s_ in range(W):
                for r_ in range(W):
                    if s_ == r_ or (rank not in (s_, r_)):
                        continue
                    g = st[c_own[st] == r_]
                    if g.size == 0:
                        continue
                    fb, bb = np.nonzero(f_own[g] == s_)
                    if fb.size == 0:
                        continue
                    key = np.stack([fine_ids[g[fb], bb], normals[g[fb]], sides[g[fb]]], axis=1)
                    key = np.unique(key, axis=0)  # one box per (fine patch, orientation)
                    b = np.zeros(key.shape[0], dtype=BOXLIST_DTYPE)
                    b["kind"], b["face"], b["patch"] = 1, -1, key[:, 0]
                    b["normal"], b["side"], b["segment"], b["cells"] = key[:, 1], key[:, 2], -1, bc
                    boxes.setdefault((s_, r_), []).append(b)
            mine_st = plan.staged
            if mine_st.size:
                remote = np.unique(fine_ids[mine_st][f_own[mine_st] != rank])
                slot_ids = remote
                slot_of = {int(pid): i for i, pid in enumerate(remote)}
                lo = part.bounds[rank]
                nl = part.size(rank)
                for f in mine_st:
                    v = np.empty(9, dtype=np.int64)
                    for b in range(9):
                        pid = int(fine_ids[f, b])
                        v[b] = pid - lo if f_own[f, b] == rank else nl + slot_of[pid]
                    restrict_src[int(f)] = v

    def cat(s_, r_):
        lst = boxes.get((s_, r_), [])
        return np.concatenate(lst) if lst else np.zeros(0, dtype=BOXLIST_DTYPE)

    src_send = [cat(rank, q) if q != rank else np.zeros(0, dtype=BOXLIST_DTYPE) for q in range(W)]
    src_recv = [cat(q, rank) if q != rank else np.zeros(0, dtype=BOXLIST_DTYPE) for q in range(W)]
    return SweepPlan(rank, W, part.size(rank), plans, src_send, src_recv,
                     np.asarray(slot_ids, dtype=np.int64), restrict_src)


# ---------------------------------------------------------------------------
# box geometry (world boxes inside patches and their compact packed copies)
# ---------------------------------------------------------------------------

def _box_world(box, support: Support, p: int, k: int):
    """(world low corner (x, y, z) inside the patch, world extents) of a shipped box."""
    n, sd = int(box["normal"]), int(box["side"])
    t1, t2 = (int(a[0]) for a in _tangential(np.array([n])))
    lo, ext = [0, 0, 0], [0, 0, 0]
    if box["kind"] == 0:  # interpolation support inside the coarse patch's source region
        l0, c0, l1, c1, l2, c2 = support.interp[int(box["segment"])]
        ns = p if sd == 0 else 0
        lo[n] = ns + l0 if sd == 0 else ns + 2 * k - l0 - c0
        ext[n] = c0
        lo[t1], ext[t1], lo[t2], ext[t2] = k + l1, c1, k + l2, c2
    else:  # restriction fine block: support normal layers x p x p
        l0, c0 = support.restrict
        nf = 0 if sd == 0 else p
        lo[n] = nf + l0 if sd == 0 else nf + 2 * k - l0 - c0
        ext[n] = c0
        lo[t1], ext[t1], lo[t2], ext[t2] = k, p, k, p
    return lo, ext


def _compact_strides(ext, u):
    return np.array([u, ext[0] * u, ext[0] * ext[1] * u], dtype=np.int64)


def pack_records(boxes: np.ndarray, support: Support, p: int, k: int, u: int, lo_patch: int) -> np.ndarray:
    """th_box records copying each box from this rank's pool into a compact send buffer."""
    _, patch, strides = pool_geometry(p, k, u)
    rec = np.zeros(boxes.size, dtype=_native.BOX_DTYPE)
    off = 0
    for i, b in enumerate(boxes):
        lo, ext = _box_world(b, support, p, k)
        rec[i]["src"] = (int(b["patch"]) - lo_patch) * patch + int(np.dot(lo, strides))
        rec[i]["src_stride"] = strides
        rec[i]["dst"] = off
        rec[i]["dst_stride"] = _compact_strides(ext, u)
        rec[i]["ext"] = ext
        off += int(b["cells"]) * u
    return rec


def unpack_records(plan: SweepPlan, support: Support, p: int, k: int, u: int) -> np.ndarray:
    """th_box records moving received restriction blocks into their staging slots."""
    _, patch, strides = pool_geometry(p, k, u)
    base = plan.recv_base(p, k, u)
    slot = {int(pid): i for i, pid in enumerate(plan.slots)}
    out = []
    for boxes, offs in zip(plan.src_recv, plan.recv_cell_offsets()):
        for b, o in zip(boxes, offs):
            if b["kind"] != 1:
                continue
            lo, ext = _box_world(b, support, p, k)
            r = np.zeros(1, dtype=_native.BOX_DTYPE)
            r["src"] = base + int(o) * u
            r["src_stride"] = _compact_strides(ext, u)
            r["dst"] = (plan.n_local + slot[int(b["patch"])]) * patch + int(np.dot(lo, strides))
            r["dst_stride"] = strides
            r["ext"] = ext
            out.append(r)
    return np.concatenate(out) if out else np.zeros(0, dtype=_native.BOX_DTYPE)


def staged_interp_records(plan: SweepPlan, support: Support, p: int, k: int, u: int) -> np.ndarray:
    """Face records of the staged interpolation faces, reading their received source boxes.

    src[0] is the element offset of the (virtual) low corner of the face's 2k x p x p world
    source region in the box's compact strides; the kernels only read inside the box."""
    base = plan.recv_base(p, k, u)
    where = {}
    for boxes, offs in zip(plan.src_recv, plan.recv_cell_offsets()):
        for b, o in zip(boxes, offs):
            if b["kind"] == 0:
                where[int(b["face"])] = (b, int(o))
    faces = plan["interpolate"].staged
    rec = _records(faces.size)
    for i, f in enumerate(faces):
        b, o = where[int(f)]
        lo, ext = _box_world(b, support, p, k)
        st = _compact_strides(ext, u)
        n, sd = int(b["normal"]), int(b["side"])
        corner = [k, k, k]
        corner[n] = p if sd == 0 else 0
        rel = sum((corner[d] - lo[d]) * int(st[d]) for d in range(3))  # region corner minus box corner
        rec[i]["src"][0] = base + o * u + rel
        rec[i]["src_stride"] = st
        rec[i]["normal"], rec[i]["side"], rec[i]["segment"] = n, sd, int(b["segment"])
    rec["dst_stride"] = world_box_strides(rec["normal"].astype(np.int64), k, p, u)
    rec["dst"] = np.arange(faces.size, dtype=np.int64) * k * p * p * u
    return rec


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class NcclTransport:
    """torch.distributed point-to-point (NCCL on GPUs, gloo on CPU) on a side stream."""

    def __init__(self, device, group=None, use_streams: bool = True):
        import torch

        self.group = group
        self.device = device
        self.use_streams = use_streams and device.type == "cuda"
        self.stream = torch.cuda.Stream(device=device) if self.use_streams else None
        self._works = []

    def start(self, sends: list, recvs: list) -> None:
        """sends / recvs: [(peer, tensor)] in matching per-peer order on both sides."""
        import torch
        import torch.distributed as dist

        ops = [dist.P2POp(dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for peer, t in recvs]
        self._ops = bool(ops)
        if not ops:
            return
        if self.use_streams:
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(self.device))
            self.stream.wait_event(ready)
            with torch.cuda.stream(self.stream):
                self._works = dist.batch_isend_irecv(ops)
        else:
            self._works = dist.batch_isend_irecv(ops)

    def finish(self) -> None:
        import torch

        for w in self._works:
            w.wait()
        self._works = []
        if self.use_streams and getattr(self, "_ops", False):
            torch.cuda.current_stream(self.device).wait_stream(self.stream)


class LoopbackTransport:
    """Several ranks' sweeps in ONE process (one device): every rank posts its sends and
    receives, and ``deliver()`` matches them per (sender, receiver) pair in posting order
    and copies — the same message matching NCCL P2P does.  For the one-GPU test of the
    cross-GPU path; nothing waits on another rank's kernels."""

    def __init__(self, world: int):
        self.world = world
        self.posted = {}

    def endpoint(self, rank: int) -> "LoopbackTransport._End":
        return LoopbackTransport._End(self, rank)

    class _End:
        def __init__(self, hub, rank):
            self.hub, self.rank = hub, rank

        def start(self, sends, recvs):
            self.hub.posted[self.rank] = (list(sends), list(recvs))

        def finish(self):
            pass

    def deliver(self) -> int:
        """Copy every posted send into its matching receive; returns messages moved."""
        moved = 0
        for r in range(self.world):
            _, recvs = self.posted.get(r, ([], []))
            per_peer = {}
            for peer, t in recvs:
                per_peer.setdefault(peer, []).append(t)
            for peer, ts in per_peer.items():
                sends = [t for q, t in self.posted.get(peer, ([], []))[0] if q == r]
                if len(sends) != len(ts):
                    raise RuntimeError(f"rank {peer} posts {len(sends)} sends to {r}, which expects {len(ts)}")
                for s, d in zip(sends, ts):
                    if s.numel() != d.numel():
                        raise RuntimeError(f"message size mismatch {peer}->{r}: {s.numel()} vs {d.numel()}")
                    d.copy_(s)
                    moved += 1
        self.posted = {}
        return moved


# ---------------------------------------------------------------------------
# the sweep
# ---------------------------------------------------------------------------

class Sweep:
    """Executes one rank's plan in four phases (``run`` = all four with the real transport):

    1. ``pre``: pack the source boxes peers need, compute the faces whose result leaves;
    2. the exchange starts (sources and results, one grouped P2P per peer);
    3. ``local``: faces with local sources and local results overlap the exchange;
    4. ``post``: wait, unpack received restriction blocks, compute the staged faces.

    compute(role, kind, face_ids, out_tensor), kind in {"send", "local", "staged"}, writes
    len(face_ids) results of `per_face` values each into out_tensor (a contiguous slice) in
    face_ids order.  ``copy_boxes(src, dst, records)`` packs / unpacks source boxes."""

    def __init__(self, plan: SweepPlan, per_face: int, device, dtype, transport, src=None, u: int = 0,
                 copy_boxes=None, pack=None, unpack=None):
        import torch

        self.plan, self.per_face, self.device = plan, int(per_face), device
        self.transport = transport
        self.out = {r: torch.empty(max(1, p.n_out * self.per_face), dtype=dtype, device=device)
                    for r, p in plan.items()}
        self.sendbuf = {r: torch.empty(max(1, p.n_send * self.per_face), dtype=dtype, device=device)
                        for r, p in plan.items()}
        self.u = int(u)
        self.src = src
        self.copy_boxes = copy_boxes
        self.pack, self.unpack = pack, unpack  # device record tensors (or None)
        self.src_sendbuf = torch.empty(max(1, plan.n_src_send_cells * self.u), dtype=dtype, device=device)
        self.recv_base = None

    def _messages(self):
        plan, pf, u = self.plan, self.per_face, self.u
        sends, recvs = [], []
        # per peer, in this order on both sides: source boxes, then results role by role
        s_off = [0]
        for b in plan.src_send:
            s_off.append(s_off[-1] + int(b["cells"].sum()) * u)
        r_off = [0]
        for b in plan.src_recv:
            r_off.append(r_off[-1] + int(b["cells"].sum()) * u)
        res_send, res_recv = {}, {}
        for role, rp in plan.items():
            off = 0
            for peer, ids in enumerate(rp.send):
                res_send[(role, peer)] = (off, ids.size)
                off += ids.size
            off = rp.local.size + rp.staged.size
            for peer, ids in enumerate(rp.recv):
                res_recv[(role, peer)] = (off, ids.size)
                off += ids.size
        for peer in range(plan.world):
            if s_off[peer + 1] > s_off[peer]:
                sends.append((peer, self.src_sendbuf[s_off[peer]:s_off[peer + 1]]))
            if r_off[peer + 1] > r_off[peer]:
                base = self.recv_base
                recvs.append((peer, self.src[base + r_off[peer]:base + r_off[peer + 1]]))
            for role in plan.roles:
                a, n = res_send[(role, peer)]
                if n:
                    sends.append((peer, self.sendbuf[role][a * pf:(a + n) * pf]))
                a, n = res_recv[(role, peer)]
                if n:
                    recvs.append((peer, self.out[role][a * pf:(a + n) * pf]))
        return sends, recvs

    def pre(self, compute) -> None:
        pf = self.per_face
        if self.pack is not None and self.plan.n_src_send_cells:
            self.copy_boxes(self.src, self.src_sendbuf, self.pack)
        for role, rp in self.plan.items():
            if rp.n_send:
                compute(role, "send", rp.send_order(), self.sendbuf[role][: rp.n_send * pf])
        sends, recvs = self._messages()
        self.transport.start(sends, recvs)

    def local(self, compute, roles=None) -> None:
        pf = self.per_face
        for role, rp in self.plan.items():
            if rp.local.size and (roles is None or role in roles):
                compute(role, "local", rp.local, self.out[role][: rp.local.size * pf])

    def post(self, compute) -> None:
        pf = self.per_face
        self.transport.finish()
        if self.unpack is not None and len(self.unpack):
            self.copy_boxes(self.src, self.src, self.unpack)
        for role, rp in self.plan.items():
            if rp.staged.size:
                a = rp.local.size
                compute(role, "staged", rp.staged, self.out[role][a * pf:(a + rp.staged.size) * pf])

    def run(self, compute) -> None:
        self.pre(compute)
        self.local(compute)
        self.post(compute)


def attach_source(sweep: Sweep, plan: SweepPlan, src, p: int, k: int, u: int) -> None:
    """Point a sweep at its rank's source tensor (plan.src_elems elements)."""
    sweep.src = src
    sweep.recv_base = plan.recv_base(p, k, u)


def face_records(plan: SweepPlan, role: str, kind: str, ids, support: Support, p: int, k: int, u: int,
                 coarse_ids, fine_ids, normals, sides, segments, lo_patch: int) -> np.ndarray:
    """th_face records of one (role, kind) batch of `plan`, as element offsets into the rank's
    source tensor; targets are consecutive k p^2-cell slabs in `ids` order."""
    from .faces import pool_interp_faces, pool_restrict_faces

    if role == "interpolate":
        if kind == "staged":
            return staged_interp_records(plan, support, p, k, u)
        return pool_interp_faces(p, k, u, coarse_ids[ids] - lo_patch, normals[ids], sides[ids], segments[ids])
    if kind == "staged":
        fid = np.stack([plan.restrict_src[int(f)] for f in ids])
    else:
        fid = fine_ids[ids] - lo_patch
    return pool_restrict_faces(p, k, u, fid, normals[ids], sides[ids])


def batch_ids(plan: SweepPlan, role: str, kind: str) -> np.ndarray:
    rp = plan[role]
    return {"send": rp.send_order(), "local": rp.local, "staged": rp.staged}[kind]


class GpuCompute:
    """Product compute for Sweep: prebuilt FaceBatches per (role, kind), records pointing
    into the rank's source tensor (pool + staging + received boxes) and at consecutive
    output slots.  ``events[(role, kind)] = (start, end)`` CUDA events, when set, bracket
    each launch (per-kernel timing inside the bench's timed region)."""

    def __init__(self, plan: SweepPlan, operators: dict, support: Support, p: int, k: int, u: int, src,
                 coarse_ids, fine_ids, normals, sides, segments, lo_patch: int):
        from .faces import FaceBatch

        self.src = src
        self.batches = {}
        self.events = None
        for role in plan.roles:
            for kind in ("send", "local", "staged"):
                ids = batch_ids(plan, role, kind)
                if ids.size:
                    rec = face_records(plan, role, kind, ids, support, p, k, u, coarse_ids, fine_ids, normals,
                                       sides, segments, lo_patch)
                    self.batches[(role, kind)] = FaceBatch(operators[role], rec, u)

    def __call__(self, role, kind, face_ids, out) -> None:
        b = self.batches[(role, kind)]
        ev = self.events.get((role, kind)) if self.events is not None else None
        if ev is not None:
            ev[0].record()
        b.launch(self.src, out, check_flag=True)
        if ev is not None:
            ev[1].record()

    @property
    def launches(self) -> int:
        return len(self.batches)

    def nonfinite(self) -> bool:
        return any(b.nonfinite() for b in self.batches.values())


def box_copier(device, u: int):
    """copy_boxes(src, dst, records) through th_copy_boxes on the current stream."""
    import torch

    lib = _native.load()

    def copy(src, dst, rec):
        n = rec.numel() // _native.BOX_DTYPE.itemsize
        s = torch.cuda.current_stream(device).cuda_stream
        _native.check(lib.th_copy_boxes(src.data_ptr(), dst.data_ptr(), rec.data_ptr(), n, u, s))

    return copy


def device_records(rec: np.ndarray, device):
    import torch

    return torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8).ravel().copy()).to(device)


def make_rank_sweep(plan: SweepPlan, operators: dict, support: Support, p: int, k: int, u: int, src, transport,
                    coarse_ids, fine_ids, normals, sides, segments, lo_patch: int):
    """(Sweep, GpuCompute) of one rank on the current CUDA device.  `src` is the rank's source
    tensor of plan.src_elems(p, k, u) float64 elements whose first n_local patches are its pool."""
    import torch

    if src.numel() < plan.src_elems(p, k, u):
        raise ValueError(f"source tensor holds {src.numel()} elements, the plan needs {plan.src_elems(p, k, u)}")
    dev = src.device
    boxes = [b for b in plan.src_send if b.size]
    pack = pack_records(np.concatenate(boxes), support, p, k, u, lo_patch) if boxes else None
    unpack = unpack_records(plan, support, p, k, u)
    sweep = Sweep(plan, k * p * p * u, dev, torch.float64, transport, src=src, u=u, copy_boxes=box_copier(dev, u),
                  pack=device_records(pack, dev) if pack is not None else None,
                  unpack=device_records(unpack, dev) if unpack.size else None)
    attach_source(sweep, plan, src, p, k, u)
    comp = GpuCompute(plan, operators, support, p, k, u, src, coarse_ids, fine_ids, normals, sides, segments,
                      lo_patch)
    return sweep, comp
