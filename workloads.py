"""Synthetic workloads of BASELINE.json's five configs (bench + tests).

The reference measures only on analytic fields (harness.py:37-68); there is no
dataset.  These generators restate BASELINE.json's config text with seeded
synthetic data, generated directly in HBM (torch fp64 on the device) because
the larger configs hold tens of GB:

* coarse patches sit on an m^3 lattice filling the unit cube (m = ceil(n^(1/3))),
  coarse width H = 1/(m p), fine width h = H/3; each patch is stored with its
  halo, (p+2k)^3 cells, AoS (u unknowns innermost), x fastest;
* field per unknown c: a cubic polynomial with 20 N(0,1) coefficients
  (configs 1, 2, 3, 5) or, for config 4, a sum of 8 Gaussian bumps
  exp(-|x - c_b|^2 / (2 w_b^2)) with centres U[0,1]^3 and widths U(0.05, 0.2)
  shared by all unknowns and amplitudes N(0,1) per (unknown, bump);
  plus 1e-6 N(0,1) noise on every stored value (torch Philox, seeded);
* faces: coarse patch, orientation (normal, coarse side) and fine segment drawn
  uniformly (numpy PCG64, seeded); config 3 takes all 6 faces of every patch;
* restriction sources are per-face fine slabs: the reference's restrict source
  buffer (2k x 3p x 3p fine cells, world layout) sampled from the same field
  at fine cell centres on the fine side of the face.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import os

import numpy as np

import paper_2504_15814_b200 as th
from paper_2504_15814_b200 import faces as F

K_HALO = 3
U = int(os.environ.get("TH_BENCH_U", "59"))  # 59 (BASELINE); the override is for layout A/B runs only


@dataclass
class Spec:
    config: int
    name: str
    p: int
    n_patches: int
    n_faces: int
    seed: int
    passes: list            # [(role, scheme)], launched in this order every step
    field: str = "cubic"
    all_six: bool = False   # config 3: every patch's 6 faces
    mixed: bool = False     # config 4: half the faces interpolate, half restrict
    k: int = K_HALO
    u: int = U


SPECS = {
    1: Spec(1, "p9_o2_interp_1024", 9, 256, 1024, 0, [("interpolate", "order2")]),
    2: Spec(2, "p9_tensor+o2_interp+restrict_4096", 9, 1024, 4096, 1,
            [("interpolate", "tensor_linear"), ("interpolate", "order2"),
             ("restrict", "tensor_linear"), ("restrict", "order2")]),
    3: Spec(3, "p9_o3_interp+restrict_24576", 9, 4096, 24576, 2,
            [("interpolate", "order3"), ("restrict", "order3")], all_six=True),
    4: Spec(4, "p17_o2+o3_interp+restrict_12288_bumps", 17, 2048, 12288, 3,
            [("interpolate", "order2"), ("restrict", "order2"), ("interpolate", "order3"), ("restrict", "order3")],
            field="bumps", mixed=True),
    5: Spec(5, "p9_o3_multi_gpu_196608", 9, 32768, 196608, 4, [("interpolate", "order3")]),
}


def cubic_exponents():
    return [(a, b, d - a - b) for d in range(4) for a in range(d, -1, -1) for b in range(d - a, -1, -1)]


@dataclass
class Field:
    kind: str
    coef: np.ndarray = None      # (u, 20) cubic
    centres: np.ndarray = None   # (8, 3) bumps
    widths: np.ndarray = None    # (8,)
    amps: np.ndarray = None      # (u, 8)

    @classmethod
    def make(cls, kind: str, u: int, rng: np.random.Generator) -> "Field":
        if kind == "cubic":
            return cls(kind, coef=rng.standard_normal((u, 20)))
        return cls(kind, centres=rng.uniform(0.0, 1.0, (8, 3)), widths=rng.uniform(0.05, 0.2, 8),
                   amps=rng.standard_normal((u, 8)))

    def eval_torch(self, xyz):
        """(N, 3) float64 CUDA coordinates -> (N, u) values."""
        import torch

        if self.kind == "cubic":
            x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
            mono = torch.stack([x ** a * y ** b * z ** c for a, b, c in cubic_exponents()], dim=1)
            return mono @ torch.from_numpy(self.coef.T.copy()).to(xyz.device)
        c = torch.from_numpy(self.centres).to(xyz.device)
        w = torch.from_numpy(self.widths).to(xyz.device)
        r2 = ((xyz[:, None, :] - c[None, :, :]) ** 2).sum(-1)
        g = torch.exp(-r2 / (2.0 * w[None, :] ** 2))
        return g @ torch.from_numpy(self.amps.T.copy()).to(xyz.device)

    def eval_numpy(self, xyz: np.ndarray) -> np.ndarray:
        if self.kind == "cubic":
            x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
            mono = np.stack([x ** a * y ** b * z ** c for a, b, c in cubic_exponents()], axis=1)
            return mono @ self.coef.T
        r2 = ((xyz[:, None, :] - self.centres[None]) ** 2).sum(-1)
        return np.exp(-r2 / (2.0 * self.widths[None] ** 2)) @ self.amps.T


@dataclass
class Faces:
    coarse: np.ndarray
    normal: np.ndarray
    side: np.ndarray
    segment: np.ndarray
    role: np.ndarray   # 0 interpolate, 1 restrict (config 4 mixes; otherwise every face does all passes)


@dataclass
class Workload:
    spec: Spec
    fld: Field
    faces: Faces
    m: int
    H: float
    pool: object = None              # CUDA tensor (n_patches * E^3 * u)
    fine: object = None              # CUDA tensor (n_restrict_faces * 2k*9p^2 * u)
    restrict_ids: np.ndarray = None  # face ids with a fine slab
    interp_ids: np.ndarray = None
    extra: dict = field(default_factory=dict)

    @property
    def E(self) -> int:
        return self.spec.p + 2 * self.spec.k


def lattice(n_patches: int):
    m = int(math.ceil(round(n_patches ** (1.0 / 3.0), 9)))
    while m ** 3 < n_patches:
        m += 1
    return m


def make_faces(spec: Spec, rng: np.random.Generator) -> Faces:
    n = spec.n_faces
    if spec.all_six:
        coarse = np.repeat(np.arange(spec.n_patches), 6)[:n]
        orient = np.tile(np.arange(6), spec.n_patches)[:n]
    else:
        coarse = rng.integers(0, spec.n_patches, n)
        orient = rng.integers(0, 6, n)
    segment = rng.integers(0, 9, n)
    role = (np.arange(n) % 2) if spec.mixed else np.zeros(n, dtype=np.int64)
    return Faces(coarse.astype(np.int64), (orient // 2).astype(np.int64), (orient % 2).astype(np.int64),
                 segment.astype(np.int64), role.astype(np.int64))


def patch_cell_centres(spec: Spec, m: int, H: float, ids: np.ndarray):
    """(len(ids) * E^3, 3) centres of the stored cells (halo included), storage order."""
    import torch

    p, k = spec.p, spec.k
    E = p + 2 * k
    ids = torch.as_tensor(ids, dtype=torch.int64, device="cuda")
    pos = torch.stack([ids % m, (ids // m) % m, ids // (m * m)], dim=1).to(torch.float64)  # (n, 3)
    r = torch.arange(E, device="cuda", dtype=torch.float64) - k + 0.5
    zz, yy, xx = torch.meshgrid(r, r, r, indexing="ij")
    local = torch.stack([xx.reshape(-1), yy.reshape(-1), zz.reshape(-1)], dim=1)  # (E^3, 3) storage order
    return ((pos[:, None, :] * p + local[None]) * H).reshape(-1, 3)


def fine_slab_centres(spec: Spec, m: int, H: float, fc: Faces, ids: np.ndarray):
    """(len(ids) * 2k*9p^2, 3) centres of each face's world restriction source box."""
    import torch

    p, k = spec.p, spec.k
    h = H / 3.0
    dev = "cuda"
    ids_t = torch.as_tensor(ids, dtype=torch.int64, device=dev)
    cid = torch.as_tensor(fc.coarse, device=dev)[ids_t]
    nrm = torch.as_tensor(fc.normal, device=dev)[ids_t]
    sd = torch.as_tensor(fc.side, device=dev)[ids_t]
    pos = torch.stack([cid % m, (cid // m) % m, cid // (m * m)], dim=1).to(torch.float64)
    lo_corner = pos * p * H                                   # patch interior low corner
    n_f = ids_t.numel()
    # world box extents: 2k along the normal, 3p along the others (x fastest)
    out = torch.empty((n_f, 2 * k * 9 * p * p, 3), dtype=torch.float64, device=dev)
    for nn in range(3):
        sel = (nrm == nn).nonzero().flatten()
        if sel.numel() == 0:
            continue
        ext = [3 * p, 3 * p, 3 * p]
        ext[nn] = 2 * k
        ax = [torch.arange(e, device=dev, dtype=torch.float64) + 0.5 for e in ext]
        zz, yy, xx = torch.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        loc = torch.stack([xx.reshape(-1), yy.reshape(-1), zz.reshape(-1)], dim=1) * h  # (cells, 3)
        base = lo_corner[sel].clone()
        # face plane: coarse on the negative side -> the patch's +n face
        plane = base[:, nn] + torch.where(sd[sel] == 0, p * H, 0.0)
        base[:, nn] = plane - k * h
        out[sel] = base[:, None, :] + loc[None]
    return out.reshape(-1, 3)


def _fill(dst, centres_fn, n_items, per_item, fld: Field, u: int, gen, chunk_cells=1 << 21):
    import torch

    step = max(1, chunk_cells // per_item)
    view = dst.view(n_items, per_item, u)
    for a in range(0, n_items, step):
        b = min(n_items, a + step)
        xyz = centres_fn(a, b)
        vals = fld.eval_torch(xyz).reshape(b - a, per_item, u)
        vals += 1e-6 * torch.randn(vals.shape, dtype=torch.float64, device=dst.device, generator=gen)
        view[a:b] = vals


def describe(config: int, rank: int = 0, scale: float = 1.0) -> Workload:
    """Host part of a workload: spec, field, faces and lattice (no device data)."""
    spec = SPECS[config]
    if scale != 1.0:
        spec = Spec(**{**spec.__dict__, "n_patches": max(8, int(spec.n_patches * scale)),
                       "n_faces": max(12, int(spec.n_faces * scale))})
        if spec.all_six:
            spec.n_faces = spec.n_patches * 6
    seed = spec.seed + 1000 * rank
    rng = np.random.default_rng(seed)
    fld = Field.make(spec.field, spec.u, rng)
    fc = make_faces(spec, rng)
    m = lattice(spec.n_patches)
    wl = Workload(spec, fld, fc, m, 1.0 / (m * spec.p))
    wl.extra["seed"] = seed
    roles = {r for r, _ in spec.passes}
    if spec.mixed:
        wl.interp_ids = np.flatnonzero(fc.role == 0)
        wl.restrict_ids = np.flatnonzero(fc.role == 1)
    else:
        wl.interp_ids = np.arange(spec.n_faces) if "interpolate" in roles else np.zeros(0, dtype=np.int64)
        wl.restrict_ids = np.arange(spec.n_faces) if "restrict" in roles else np.zeros(0, dtype=np.int64)
    return wl


def host_sources(wl: Workload, f: int, role: str, rng: np.random.Generator) -> np.ndarray:
    """Host (numpy) world source buffer of face f for one role, same field (fresh noise).
    Used by the CPU reference arm, which must not need a GPU."""
    s, fc = wl.spec, wl.faces
    p, k, H = s.p, s.k, wl.H
    c = int(fc.coarse[f])
    pos = np.array([c % wl.m, (c // wl.m) % wl.m, c // (wl.m * wl.m)], dtype=np.float64)
    n, sd = int(fc.normal[f]), int(fc.side[f])
    if role == "interpolate":
        ext = [p, p, p]
        ext[n] = 2 * k
        lo = np.full(3, float(k))
        lo[n] = p if sd == 0 else 0
        ax = [np.arange(e) + lo[d] - k + 0.5 for d, e in enumerate(ext)]
        scale, base = H, pos * p * H
    else:
        ext = [3 * p, 3 * p, 3 * p]
        ext[n] = 2 * k
        h = H / 3.0
        base = pos * p * H
        base[n] = base[n] + (p * H if sd == 0 else 0.0) - k * h
        ax = [np.arange(e) + 0.5 for e in ext]
        scale = h
    zz, yy, xx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    xyz = base + scale * np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)
    vals = wl.fld.eval_numpy(xyz) + 1e-6 * rng.standard_normal((xyz.shape[0], s.u))
    return np.ascontiguousarray(vals.reshape(-1))


def build(config: int, rank: int = 0, scale: float = 1.0, with_fine: bool = True) -> Workload:
    """Generate the workload of one config on the current CUDA device.

    ``rank`` offsets the seed (weak scaling: every rank owns an independent
    shard of the same shape); ``scale`` shrinks patch / face counts (tests)."""
    import torch

    wl = describe(config, rank, scale)
    spec, fld, fc, m, H = wl.spec, wl.fld, wl.faces, wl.m, wl.H
    seed = wl.extra["seed"]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    E, u = wl.E, spec.u
    wl.pool = torch.empty(spec.n_patches * E ** 3 * u, dtype=torch.float64, device="cuda")
    _fill(wl.pool, lambda a, b: patch_cell_centres(spec, m, H, np.arange(a, b)), spec.n_patches, E ** 3, fld, u,
          gen)
    if with_fine and wl.restrict_ids.size:
        per = 2 * spec.k * 9 * spec.p ** 2
        wl.fine = torch.empty(wl.restrict_ids.size * per * u, dtype=torch.float64, device="cuda")
        ids = wl.restrict_ids
        _fill(wl.fine, lambda a, b: fine_slab_centres(spec, m, H, fc, ids[a:b]), ids.size, per, fld, u, gen)
    return wl


def interp_records(wl: Workload) -> np.ndarray:
    s, fc, ids = wl.spec, wl.faces, wl.interp_ids
    return F.pool_interp_faces(s.p, s.k, s.u, fc.coarse[ids], fc.normal[ids], fc.side[ids], fc.segment[ids])


def restrict_records(wl: Workload, half=None) -> np.ndarray:
    s, fc, ids = wl.spec, wl.faces, wl.restrict_ids
    return F.slab_faces("restrict", s.p, s.k, s.u, fc.normal[ids], fc.side[ids], half=half)


def interp_source_boxes(wl: Workload, ids: np.ndarray):
    """(len(ids), 2k p^2 u) world interpolation source buffers cut out of the pool (device)."""
    import torch

    s = wl.spec
    p, k, u, E = s.p, s.k, s.u, wl.E
    pool = wl.pool.view(s.n_patches, E, E, E, u)
    out = torch.empty((ids.size, 2 * k * p * p * u), dtype=torch.float64, device=wl.pool.device)
    for i, f in enumerate(ids):
        n, sd, c = int(wl.faces.normal[f]), int(wl.faces.side[f]), int(wl.faces.coarse[f])
        lo, ext = [k, k, k], [p, p, p]
        lo[n] = p if sd == 0 else 0
        ext[n] = 2 * k
        out[i] = pool[c, lo[2]:lo[2] + ext[2], lo[1]:lo[1] + ext[1], lo[0]:lo[0] + ext[0]].reshape(-1)
    return out


def face_cfg(wl: Workload, f: int) -> th.FaceConfig:
    s = wl.spec
    return th.FaceConfig("xyz"[wl.faces.normal[f]], ("negative", "positive")[wl.faces.side[f]],
                         int(wl.faces.segment[f]), s.p, s.k, s.u)


# ---------------------------------------------------------------------------
# config 5: patches block-partitioned over ranks, fine patches drawn from the
# pool via index lists, 10% of faces with their fine patches on another rank
# ---------------------------------------------------------------------------

@dataclass
class MultiWorkload:
    spec: Spec
    fld: Field
    part: object
    coarse: np.ndarray
    normal: np.ndarray
    side: np.ndarray
    segment: np.ndarray
    fine: np.ndarray          # (n_faces, 9) global patch ids, one owner per face
    m: int
    H: float
    pool: object = None       # this rank's patches [lo, hi)
    src: object = None        # source tensor: pool + staging slots + received boxes


def describe_multi(world: int, scale: float = 1.0, cross: float = 0.10, straddle: float = 0.0,
                   fine_layout: str = "random", p: int | None = None) -> MultiWorkload:
    """Global face list of config 5 (identical on every rank).

    BASELINE: 10% of faces have coarse and fine patches on different GPUs, the partner GPU
    uniform at random; all nine fine patches of such a face live on the partner.  With
    ``straddle`` > 0 that fraction of faces additionally gets one fine patch drawn from the
    whole pool (its nine fine patches then straddle GPUs; tests and A/B runs only)."""
    from paper_2504_15814_b200.multigpu import Partition

    spec = SPECS[5]
    if scale != 1.0:
        spec = Spec(**{**spec.__dict__, "n_patches": max(8 * world, int(spec.n_patches * scale)),
                       "n_faces": max(12, int(spec.n_faces * scale))})
    if p is not None and p != spec.p:  # tests: config-5-shaped faces at another patch size
        spec = Spec(**{**spec.__dict__, "p": int(p)})
    rng = np.random.default_rng(spec.seed)
    fld = Field.make(spec.field, spec.u, rng)
    n, nf = spec.n_patches, spec.n_faces
    part = Partition(n, world)
    coarse = rng.integers(0, n, nf)
    orient = rng.integers(0, 6, nf)
    segment = rng.integers(0, 9, nf)
    c_own = part.owner(coarse)
    f_own = c_own.copy()
    if world > 1:
        flip = rng.random(nf) < cross
        f_own[flip] = (c_own[flip] + rng.integers(1, world, int(flip.sum()))) % world
    lo = part.bounds[f_own]
    size = part.bounds[f_own + 1] - lo
    fine = lo[:, None] + (rng.random((nf, 9)) * size[:, None]).astype(np.int64)
    if fine_layout == "siblings":  # diagnosis only: the nine fine patches are consecutive ids
        base = lo + (rng.random(nf) * np.maximum(size - 9, 1)).astype(np.int64)
        fine = base[:, None] + np.arange(9)[None, :]
    if straddle > 0:
        srng = np.random.default_rng(spec.seed + 17)
        st = srng.random(nf) < straddle
        fine[st, srng.integers(0, 9, int(st.sum()))] = srng.integers(0, n, int(st.sum()))
    m = lattice(n)
    return MultiWorkload(spec, fld, part, coarse.astype(np.int64), (orient // 2).astype(np.int64),
                         (orient % 2).astype(np.int64), segment.astype(np.int64), fine, m, 1.0 / (m * spec.p))


NOISE_GROUP = 64  # patches per noise generator


def _patch_group(wl: MultiWorkload, g: int, device):
    """Values of patches [g*64, g*64 + 64) clipped to the pool: field + 1e-6 N(0,1) noise from a
    generator seeded with (seed, g), so a patch's values do not depend on the partition."""
    import torch

    s = wl.spec
    per = (s.p + 2 * s.k) ** 3
    a, b = g * NOISE_GROUP, min((g + 1) * NOISE_GROUP, s.n_patches)
    gen = torch.Generator(device=device)
    gen.manual_seed(s.seed * 1000003 + g)
    noise = 1e-6 * torch.randn((NOISE_GROUP, per, s.u), dtype=torch.float64, device=device, generator=gen)
    vals = wl.fld.eval_torch(patch_cell_centres(s, wl.m, wl.H, np.arange(a, b))).reshape(b - a, per, s.u)
    return vals + noise[: b - a]


def fill_pool(wl: MultiWorkload, rank: int, pool) -> None:
    """Fill `pool` with this rank's patches [lo, hi) of the global pool (E^3 u values each)."""
    s = wl.spec
    per = (s.p + 2 * s.k) ** 3
    lo, hi = int(wl.part.bounds[rank]), int(wl.part.bounds[rank + 1])
    view = pool[: (hi - lo) * per * s.u].view(hi - lo, per, s.u)
    for g in range(lo // NOISE_GROUP, (hi + NOISE_GROUP - 1) // NOISE_GROUP):
        vals = _patch_group(wl, g, pool.device)
        a = g * NOISE_GROUP
        a0, b0 = max(a, lo), min(a + vals.shape[0], hi)
        view[a0 - lo:b0 - lo] = vals[a0 - a:b0 - a]


def patch_values(wl: MultiWorkload, ids, device="cuda"):
    """(len(ids), E, E, E, u) values of global patches `ids` (any rank's), regenerated."""
    import torch

    s = wl.spec
    E = s.p + 2 * s.k
    ids = np.asarray(ids, dtype=np.int64)
    out = torch.empty((ids.size, E, E, E, s.u), dtype=torch.float64, device=device)
    for g in np.unique(ids // NOISE_GROUP):
        vals = _patch_group(wl, int(g), device).view(-1, E, E, E, s.u)
        sel = np.flatnonzero(ids // NOISE_GROUP == g)
        out[torch.as_tensor(sel, device=device)] = vals[torch.as_tensor(ids[sel] - g * NOISE_GROUP, device=device)]
    return out


def build_multi(world: int, rank: int, scale: float = 1.0, src_elems: int | None = None,
                straddle: float = 0.0, fine_layout: str = "random") -> MultiWorkload:
    """Config 5 on this rank: its pool (patches [lo, hi)) at the front of a source tensor of
    `src_elems` elements (multigpu.SweepPlan.src_elems: pool + staging + received boxes)."""
    import torch

    wl = describe_multi(world, scale, straddle=straddle, fine_layout=fine_layout)
    s = wl.spec
    E = s.p + 2 * s.k
    lo, hi = int(wl.part.bounds[rank]), int(wl.part.bounds[rank + 1])
    n_pool = (hi - lo) * E ** 3 * s.u
    wl.src = torch.empty(max(1, n_pool, src_elems or 0), dtype=torch.float64, device="cuda")
    wl.src[n_pool:].zero_()
    wl.pool = wl.src[:n_pool]
    fill_pool(wl, rank, wl.pool)
    return wl


def face_source(wl: MultiWorkload, f: int, role: str, patches) -> np.ndarray:
    """World-layout reference source buffer (numpy) of config-5 face f, cut from patch arrays
    {global id: (E, E, E, u)} (torch or numpy): the buffer the reference HaloExchange.run takes
    (interpolation: the coarse patch's 2k x p x p box; restriction: the nine fine patches'
    2k x p x p blocks side by side, geometry.py:244-261)."""
    s = wl.spec
    p, k, u = s.p, s.k, s.u
    n, sd = int(wl.normal[f]), int(wl.side[f])
    t1, t2 = [d for d in range(3) if d != n]

    def host(x):
        return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)

    if role == "interpolate":
        lo3, ext = [k, k, k], [p, p, p]
        lo3[n], ext[n] = (p if sd == 0 else 0), 2 * k
        v = patches[int(wl.coarse[f])]
        return np.ascontiguousarray(host(v[lo3[2]:lo3[2] + ext[2], lo3[1]:lo3[1] + ext[1],
                                           lo3[0]:lo3[0] + ext[0]]).reshape(-1))
    ext = [3 * p, 3 * p, 3 * p]
    ext[n] = 2 * k
    box = np.zeros((ext[2], ext[1], ext[0], u))
    for b in range(9):
        lo3, e = [k, k, k], [p, p, p]
        lo3[n], e[n] = (0 if sd == 0 else p), 2 * k
        blk = patches[int(wl.fine[f, b])][lo3[2]:lo3[2] + e[2], lo3[1]:lo3[1] + e[1], lo3[0]:lo3[0] + e[0]]
        off = [0, 0, 0]
        off[t1], off[t2] = (b % 3) * p, (b // 3) * p
        box[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = host(blk)
    return box.reshape(-1)
