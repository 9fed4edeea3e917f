"""Oracle restatement of the reference face geometry (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/trihalo/geometry.py:
  * regions in units of the fine spacing h, cells x-fastest   (geometry.py:26-30, 79-122)
  * reference frame: normal -> axis 0, tangential axes keep world order,
    only the normal axis is mirrored, when the coarse side is positive
                                                              (geometry.py:180-190)
  * frame application to (nz, ny, nx, u) grids                (geometry.py:165-174)
  * reference regions                                          (geometry.py:202-228)
  * gather maps world -> mapped order                          (geometry.py:332-341)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

AXES = ("x", "y", "z")
SIDES = ("negative", "positive")


@dataclass(frozen=True)
class FaceCfg:
    normal_axis: str = "x"
    coarse_side: str = "negative"
    segment: int = 4
    p: int = 4
    k: int = 3
    u: int = 58


@dataclass(frozen=True)
class Region:
    """Box of cells: extents (nx, ny, nz), spacing, low-corner origin (geometry.py:79-122)."""

    extents: tuple
    spacing: float
    origin: tuple

    @property
    def n(self) -> int:
        return int(self.extents[0] * self.extents[1] * self.extents[2])

    def lin(self, i, j, k2):
        nx, ny, _ = self.extents
        return (k2 * ny + j) * nx + i

    def unlin(self, r):
        nx, ny, _ = self.extents
        return r % nx, (r // nx) % ny, r // (nx * ny)

    def centre(self, idx, h=1.0):
        return tuple(h * (self.origin[d] + (idx[d] + 0.5) * self.spacing) for d in range(3))

    def all_centres(self, h=1.0) -> np.ndarray:
        nx, ny, nz = self.extents
        k2, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        idx = np.stack([i.ravel(), j.ravel(), k2.ravel()], axis=1).astype(np.float64)
        return h * (np.asarray(self.origin, dtype=np.float64) + (idx + 0.5) * self.spacing)


@dataclass(frozen=True)
class Frame:
    """perm[d] = reference axis of world axis d; flips[d] mirrors world axis d (geometry.py:125-174)."""

    perm: tuple
    flips: tuple

    def inverse(self) -> "Frame":
        inv = [0, 0, 0]
        for d in range(3):
            inv[self.perm[d]] = d
        return Frame(tuple(inv), tuple(self.flips[inv[e]] for e in range(3)))

    def map_region(self, reg: Region) -> Region:
        ext = [0, 0, 0]
        org = [0.0, 0.0, 0.0]
        for d in range(3):
            e = self.perm[d]
            ext[e] = reg.extents[d]
            if self.flips[d]:
                org[e] = -(reg.origin[d] + reg.extents[d] * reg.spacing)
            else:
                org[e] = reg.origin[d]
        return Region(tuple(ext), reg.spacing, tuple(org))

    def map_grid(self, grid: np.ndarray) -> np.ndarray:
        # grid axes are (z, y, x, u): world axis d lives at array axis 2-d
        for d in range(3):
            if self.flips[d]:
                grid = np.flip(grid, axis=2 - d)
        inv = [0, 0, 0]
        for d in range(3):
            inv[self.perm[d]] = d
        return np.ascontiguousarray(grid.transpose(2 - inv[2], 2 - inv[1], 2 - inv[0], 3))


def frame_for(cfg: FaceCfg) -> Frame:
    n = AXES.index(cfg.normal_axis)
    t1, t2 = [d for d in range(3) if d != n]
    perm = [0, 0, 0]
    perm[n], perm[t1], perm[t2] = 0, 1, 2
    flips = [False, False, False]
    flips[n] = cfg.coarse_side == "positive"
    return Frame(tuple(perm), tuple(flips))


def inner_layers(k: int) -> int:
    return math.ceil(k / 2)


# reference regions (geometry.py:202-228)
def ref_interp_source(p, k):
    return Region((2 * k, p, p), 3.0, (-3.0 * k, 0.0, 0.0))


def ref_interp_target_full(p, k):
    return Region((k, 3 * p, 3 * p), 1.0, (0.0, 0.0, 0.0))


def ref_interp_target_segment(p, k, s):
    return Region((k, p, p), 1.0, (0.0, float((s % 3) * p), float((s // 3) * p)))


def ref_restrict_source(p, k):
    return Region((2 * k, 3 * p, 3 * p), 1.0, (-float(k), 0.0, 0.0))


def ref_restrict_target(p, k, half=None):
    if half is None:
        return Region((k, p, p), 3.0, (0.0, 0.0, 0.0))
    lo = inner_layers(k)
    if half == "inner":
        return Region((lo, p, p), 3.0, (0.0, 0.0, 0.0))
    if half == "outer":
        return Region((k - lo, p, p), 3.0, (3.0 * lo, 0.0, 0.0))
    raise ValueError(half)


def _world(cfg, ref):
    return frame_for(cfg).inverse().map_region(ref)


def interp_source_world(cfg):
    return _world(cfg, ref_interp_source(cfg.p, cfg.k))


def interp_target_world(cfg):
    return _world(cfg, ref_interp_target_segment(cfg.p, cfg.k, cfg.segment))


def restrict_source_world(cfg):
    return _world(cfg, ref_restrict_source(cfg.p, cfg.k))


def restrict_target_world(cfg, half=None):
    return _world(cfg, ref_restrict_target(cfg.p, cfg.k, half))


def gather_cells(frame: Frame, world: Region) -> np.ndarray:
    """mapped[r] = world[idx[r]] (geometry.py:332-341)."""
    nx, ny, nz = world.extents
    ids = np.arange(world.n, dtype=np.int64).reshape(nz, ny, nx, 1)
    return frame.map_grid(ids).reshape(-1)


def subregion_rows(full: Region, sub: Region) -> np.ndarray:
    """Linear ids in ``full`` of ``sub``'s cells, in ``sub`` order (csr.py:204-216)."""
    sh = [round((sub.origin[d] - full.origin[d]) / full.spacing) for d in range(3)]
    nx, ny, nz = sub.extents
    k2, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    fx, fy, _ = full.extents
    rows = ((k2 + sh[2]) * fy + (j + sh[1])) * fx + (i + sh[0])
    return rows.ravel().astype(np.int64)


def same_level_fill(pool: np.ndarray, p: int, k: int, src_ids, dst_ids, normals, sides) -> np.ndarray:
    """Same-level halo fill of a patch pool (the reference has no
    counterpart — it handles 3:1 faces only — so this restates the plain copy in world
    (z, y, x, u) grids, geometry.py:26-30 ordering).  ``pool`` is (n, E, E, E, u) with
    E = p + 2k; returns a filled copy.  Face i: side 0 -> halo normal layers [0, k) of
    dst <- interior [p, p + k) of src; side 1 -> halo [p + k, p + 2k) <- interior [k, 2k);
    tangential interior [k, k + p) only."""
    out = pool.copy()
    for s, d, nrm, sd in zip(src_ids, dst_ids, normals, sides):
        src_n = slice(p, p + k) if sd == 0 else slice(k, 2 * k)
        dst_n = slice(0, k) if sd == 0 else slice(p + k, p + 2 * k)
        tan = slice(k, k + p)
        ax = 2 - int(nrm)  # world axis x/y/z -> grid axis 2/1/0
        src_idx = [tan, tan, tan]
        dst_idx = [tan, tan, tan]
        src_idx[ax], dst_idx[ax] = src_n, dst_n
        out[(int(d), *dst_idx)] = pool[(int(s), *src_idx)]
    return out
