"""Face batches: th_face descriptors for many faces and their launch.

A face record (include/trihalo_b200.h ``th_face``) locates a face's source
and target cells by element offsets and per-world-axis strides, so one kernel
serves every storage layout.  Builders here cover the layouts the bench and
the drop-in use:

* ``slab``: each face's source / target is a contiguous world-layout box —
  exactly the reference's HaloBuffer for that face (geometry.py:244-265);
* ``pool``: patches stored with their halos, ``pool[patch][z][y][x][u]`` with
  E = p + 2k cells per axis, and faces pointing into it through patch ids
  (coarse patch for interpolation sources, the nine fine patches of a face
  for restriction sources).  The reference has no pool; the embedding of
  its face regions into patch storage is:
    interp source   coarse normal [p, p+2k) (coarse on the negative side) or
                    [0, 2k) (positive side), tangential [k, k+p)
    restrict source fine normal   [0, 2k) (coarse negative) or [p, p+2k)
                    (positive), tangential [k, k+p) per fine patch
    restrict target coarse normal [p+k, p+2k) or [0, k), tangential [k, k+p)
    interp target   fine normal   [k, 2k) or [p, p+k), tangential [k, k+p)
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ContractViolationError
from .geometry import half_layers

FACE_DTYPE = _native.FACE_DTYPE


def _tangential(normal: np.ndarray):
    t1 = np.where(normal == 0, 1, 0)
    t2 = np.where(normal == 2, 1, 2)
    return t1, t2


def world_box_strides(normal: np.ndarray, n_ext: int, t_ext: int, u: int) -> np.ndarray:
    """(n, 3) element strides of x-fastest world boxes with extent n_ext along the normal."""
    normal = np.asarray(normal, dtype=np.int64)
    ext = np.full((normal.size, 3), t_ext, dtype=np.int64)
    ext[np.arange(normal.size), normal] = n_ext
    st = np.empty_like(ext)
    st[:, 0] = u
    st[:, 1] = u * ext[:, 0]
    st[:, 2] = u * ext[:, 0] * ext[:, 1]
    return st


def box_sizes(role: str, p: int, k: int, half=None) -> tuple:
    """(source cells, target cells) of one face's world boxes."""
    if role == "interpolate":
        return 2 * k * p * p, k * p * p
    lo, hi = half_layers(k, half)
    return 2 * k * 9 * p * p, (hi - lo) * p * p


def _records(n: int) -> np.ndarray:
    return np.zeros(n, dtype=FACE_DTYPE)


def slab_faces(role: str, p: int, k: int, u: int, normals, sides, segments=None, half=None,
               src_offsets=None, dst_offsets=None) -> np.ndarray:
    """Faces whose source and target are contiguous world-layout boxes (reference HaloBuffers)."""
    normals = np.asarray(normals, dtype=np.int64).ravel()
    sides = np.asarray(sides, dtype=np.int64).ravel()
    n = normals.size
    src_cells, dst_cells = box_sizes(role, p, k, half)
    if src_offsets is None:
        src_offsets = np.arange(n, dtype=np.int64) * src_cells * u
    if dst_offsets is None:
        dst_offsets = np.arange(n, dtype=np.int64) * dst_cells * u
    rec = _records(n)
    rec["normal"], rec["side"] = normals, sides
    lo, hi = half_layers(k, half) if role == "restrict" else (0, k)
    if role == "interpolate":
        rec["segment"] = np.asarray(segments, dtype=np.int64).ravel() if segments is not None else 4
        ss = world_box_strides(normals, 2 * k, p, u)
        rec["src"][:, 0] = src_offsets
    else:
        rec["half"] = _native.HALF_CODES[half]
        ss = world_box_strides(normals, 2 * k, 3 * p, u)
        t1, t2 = _tangential(normals)
        rows = np.arange(n)
        for b in range(9):
            b1, b2 = b % 3, b // 3
            rec["src"][:, b] = src_offsets + b1 * p * ss[rows, t1] + b2 * p * ss[rows, t2]
    rec["src_stride"] = ss
    rec["dst_stride"] = world_box_strides(normals, hi - lo, p, u)
    rec["dst"] = dst_offsets
    return rec


def pool_geometry(p: int, k: int, u: int):
    """(E, patch element count, world strides) of the halo-padded patch pool."""
    E = p + 2 * k
    return E, E ** 3 * u, np.array([u, E * u, E * E * u], dtype=np.int64)


def _corner(normal, n_start, t_start, strides):
    """Element offset of the cell (normal index n_start, tangential t_start, t_start)."""
    t1, t2 = _tangential(normal)
    return n_start * strides[normal] + t_start * strides[t1] + t_start * strides[t2]


def pool_interp_faces(p: int, k: int, u: int, coarse_ids, normals, sides, segments,
                      dst_offsets=None, fine_ids=None) -> np.ndarray:
    """Interpolation faces reading the coarse patch pool.

    Targets are per-face slabs (k x p x p fine cells in world order, the reference output
    layout) unless ``fine_ids`` (the fine patch of each face's segment) is given: then the
    values are written into the pool at the reference's target cells, which are fine patch
    F's first k interior layers next to the coarse patch — normal [k, 2k) when the coarse
    side is "negative", [p, p + k) when "positive" — by F's tangential interior (SURVEY A13,
    geometry.py:202-265).  Those cells are also restriction inputs, so launch this after any
    restriction that reads them (stream order).
    """
    normals = np.asarray(normals, dtype=np.int64).ravel()
    sides = np.asarray(sides, dtype=np.int64).ravel()
    coarse_ids = np.asarray(coarse_ids, dtype=np.int64).ravel()
    n = normals.size
    _, patch, strides = pool_geometry(p, k, u)
    rec = _records(n)
    rec["normal"], rec["side"], rec["segment"] = normals, sides, np.asarray(segments).ravel()
    n_start = np.where(sides == 0, p, 0)
    rec["src"][:, 0] = coarse_ids * patch + _corner(normals, n_start, k, strides)
    rec["src_stride"] = strides
    if fine_ids is None:
        rec["dst_stride"] = world_box_strides(normals, k, p, u)
        rec["dst"] = np.arange(n, dtype=np.int64) * k * p * p * u if dst_offsets is None else dst_offsets
    else:
        fine_ids = np.asarray(fine_ids, dtype=np.int64).ravel()
        rec["dst_stride"] = strides
        rec["dst"] = fine_ids * patch + _corner(normals, np.where(sides == 0, k, p), k, strides)
    return rec


def pool_restrict_faces(p: int, k: int, u: int, fine_ids, normals, sides, half=None,
                        dst_offsets=None, coarse_ids=None) -> np.ndarray:
    """Restriction faces reading the nine fine patches of each face from the pool.

    ``fine_ids`` is (n, 9): fine patch of block (b1, b2) at column b1 + 3*b2.
    Targets are per-face slabs (world order) unless ``coarse_ids`` is given,
    in which case the result is written into the coarse patches' halos.
    """
    normals = np.asarray(normals, dtype=np.int64).ravel()
    sides = np.asarray(sides, dtype=np.int64).ravel()
    fine_ids = np.asarray(fine_ids, dtype=np.int64).reshape(-1, 9)
    n = normals.size
    _, patch, strides = pool_geometry(p, k, u)
    rec = _records(n)
    rec["normal"], rec["side"], rec["half"] = normals, sides, _native.HALF_CODES[half]
    n_start = np.where(sides == 0, 0, p)
    corner = _corner(normals, n_start, k, strides)
    rec["src"] = fine_ids * patch + corner[:, None]
    rec["src_stride"] = strides
    lo, hi = half_layers(k, half)
    if coarse_ids is None:
        rec["dst_stride"] = world_box_strides(normals, hi - lo, p, u)
        rec["dst"] = np.arange(n, dtype=np.int64) * (hi - lo) * p * p * u if dst_offsets is None else dst_offsets
    else:
        coarse_ids = np.asarray(coarse_ids, dtype=np.int64).ravel()
        rec["dst_stride"] = strides
        # halo layers of the coarse patch on the fine side; the half's box starts
        # `lo` layers away from the face
        d_start = np.where(sides == 0, p + k + lo, k - hi)
        rec["dst"] = coarse_ids * patch + _corner(normals, d_start, k, strides)
    return rec


def pool_face_blocks(p: int, k: int, u: int) -> np.ndarray:
    """The cells of a halo-padded patch that 3:1 face work can read, as copy blocks.

    Interpolation reads the coarse patch's normal layers [p, p + 2k) or [0, 2k) by [k, k + p)
    tangentially; restriction reads the same layers of each fine patch.  The union
    over the six faces (2,160 of 3,375 cells at p = 9, k = 3) is returned as blocks
    {first row, rows, first element, elements} with a row = one x-line of E cells (E u
    elements) and row index z E + y -- the format of th_copy_patch_blocks."""
    E = p + 2 * k
    need = np.zeros((E, E, E), dtype=bool)  # [z][y][x]
    t = slice(k, k + p)
    for n in range(3):
        for lo in (0, p):
            sl = [t, t, t]
            sl[2 - n] = slice(lo, lo + 2 * k)
            need[tuple(sl)] = True
    runs = {}
    for z in range(E):
        for y in range(E):
            x = 0
            while x < E:
                if need[z, y, x]:
                    s0 = x
                    while x < E and need[z, y, x]:
                        x += 1
                    runs.setdefault((z, s0, x - s0), []).append(y)
                else:
                    x += 1
    blocks = []
    for (z, x0, n), ys in sorted(runs.items()):
        start = prev = ys[0]
        for y in ys[1:] + [None]:
            if y is None or y != prev + 1:
                blocks.append((z * E + start, prev - start + 1, x0 * u, n * u))
                start = y
            prev = y if y is not None else prev
    return np.array(blocks, dtype=np.int32)


def pool_same_level_faces(p: int, k: int, u: int, src_ids, dst_ids, normals, sides) -> np.ndarray:
    """Same-level halo faces of the patch pool.

    Face i fills the k halo layers of patch ``dst_ids[i]`` on its face (``normals[i]``,
    ``sides[i]``) from the k interior layers of the same-level neighbour ``src_ids[i]``
    next to the shared face, over the p x p tangential interior (pool layout as in
    ``pool_geometry``).  ``sides[i]`` = 0: the neighbour is on the destination's negative
    side, so halo normal layers [0, k) <- neighbour interior [p, p + k); 1: halo
    [p + k, p + 2k) <- neighbour interior [k, 2k).  Apply with ``copy_faces(pool, pool,
    rec, k, p, u)``; the boxes never overlap (halo vs interior cells).
    """
    from .geometry import validate_pk

    validate_pk(p, k)  # k <= p: the k interior source layers never reach the halo layers other faces write
    normals = np.asarray(normals, dtype=np.int64).ravel()
    sides = np.asarray(sides, dtype=np.int64).ravel()
    src_ids = np.asarray(src_ids, dtype=np.int64).ravel()
    dst_ids = np.asarray(dst_ids, dtype=np.int64).ravel()
    if src_ids.size and (src_ids.min() < 0 or dst_ids.min() < 0):
        raise ContractViolationError("patch ids must be >= 0")
    if not (normals.size == sides.size == src_ids.size == dst_ids.size):
        raise ContractViolationError("src_ids, dst_ids, normals and sides must have one entry per face")
    n = normals.size
    _, patch, strides = pool_geometry(p, k, u)
    rec = _records(n)
    rec["normal"], rec["side"] = normals, sides
    rec["src"][:, 0] = src_ids * patch + _corner(normals, np.where(sides == 0, p, k), k, strides)
    rec["dst"] = dst_ids * patch + _corner(normals, np.where(sides == 0, 0, p + k), k, strides)
    rec["src_stride"] = strides
    rec["dst_stride"] = strides
    return rec


def copy_faces(src, dst, records, n_ext: int, t_ext: int, u: int, stream=None) -> None:
    """Launch ``th_copy_faces`` over face records (numpy records or a device uint8 tensor
    holding them): each face copies an n_ext x t_ext x t_ext world box of cells."""
    import torch

    lib = _native.load()
    for t in (src, dst):
        if not (t.is_cuda and t.dtype == torch.float64):
            raise ContractViolationError("copy_faces needs float64 CUDA tensors")
    with torch.cuda.device(src.device):
        if isinstance(records, np.ndarray):
            records = torch.from_numpy(records.view(np.uint8).ravel().copy()).to(src.device)
        n = records.numel() // _native.FACE_DTYPE.itemsize
        if stream is None:
            s = torch.cuda.current_stream(src.device).cuda_stream
        else:  # the records (possibly a temporary) stay allocated until the copy on `stream` ran
            s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            if hasattr(stream, "cuda_stream"):
                records.record_stream(stream)
            else:
                records.record_stream(torch.cuda.ExternalStream(s, device=src.device))
        _native.check(lib.th_copy_faces(src.data_ptr(), dst.data_ptr(), records.data_ptr(), n, n_ext, t_ext, u, s))


class FaceBatch:
    """Device-resident face records of one (role, scheme) for repeated launches."""

    def __init__(self, operator, records: np.ndarray, u: int, device=None):
        import torch

        self.op = operator
        self.u = int(u)
        self.n = int(records.size)
        dev = torch.device("cuda", operator.device if device is None else device)
        raw = torch.from_numpy(np.ascontiguousarray(records).view(np.uint8).copy())
        self.records = raw.to(dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def launch(self, src, dst, stream=None, check_flag: bool = True) -> None:
        """Apply to all faces: src / dst are CUDA float64 tensors (element offsets index them)."""
        import torch

        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        flag = self.flag.data_ptr() if check_flag else None
        _native.check(_native.load().th_apply_faces(self.op.handle, src.data_ptr(), dst.data_ptr(),
                                                    self.records.data_ptr(), self.n, self.u, flag, s))

    def nonfinite(self) -> bool:
        """Reads (and clears) the device non-finite flag; synchronises."""
        bad = bool(self.flag.item())
        if bad:
            self.flag.zero_()
        return bad
