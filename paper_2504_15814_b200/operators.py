"""Operators: host construction in C++ (csrc/builder.cpp), upload to HBM,
and the reference-compatible CSR view.

Reference counterparts: OperatorKey / CsrOperator (csr.py:26-76),
OperatorCache / operator_cache_get (taylor.py:252-308),
build_reference_operator (schemes.py:56-70).  The device operator is keyed
by (role, scheme, p, k, device) only — segments and halves are selected per
face inside the kernels, so one upload serves all 9 segments / 3 halves.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native, geometry
from .errors import ConfigurationError, ContractViolationError
from .geometry import RegionShape


@dataclass(frozen=True)
class OperatorKey:
    role: str
    scheme: str
    p: int
    k: int
    segment: int | None = None
    half: str | None = None


@dataclass(frozen=True, eq=False)
class CsrOperator:
    """Host CSR view of a row block of a device operator (same fields as the reference's)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray = field(repr=False)
    col_indices: np.ndarray = field(repr=False)
    values: np.ndarray = field(repr=False)
    scheme_tag: str
    built_for: OperatorKey | None = None
    source_region: RegionShape | None = None
    target_region: RegionShape | None = None
    max_condition: float = float("nan")
    condition_warnings: tuple = ()

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    def row_sums(self) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        return np.bincount(rows, weights=self.values, minlength=self.n_rows)

    def arrays_equal(self, other) -> bool:
        return (self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.values, other.values))


def _require_torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise _native.DeviceError("no CUDA device: the B200 halo path has no CPU fallback")
    return torch


class HostOperator:
    """Operator built by the C++ builder without a device upload (inspection / export only)."""

    on_device = False

    def __init__(self, role: str, scheme: str, p: int, k: int):
        self._create(role, scheme, p, k, _native.load().th_operator_create_host)

    def _create(self, role, scheme, p, k, creator):
        if role not in _native.ROLES:
            raise ConfigurationError(f"role must be 'interpolate' or 'restrict', got {role!r}")
        if scheme not in _native.SCHEME_CODES:
            raise ConfigurationError(f"unknown scheme {scheme!r}; expected one of {tuple(_native.SCHEME_CODES)}")
        self.role, self.scheme, self.p, self.k = role, scheme, p, k
        handle = ctypes.c_void_p()
        _native.check(creator(_native.ROLES[role], _native.SCHEME_CODES[scheme], p, k, ctypes.byref(handle)))
        self.handle = handle
        info = _native.OperatorInfo()
        _native.check(_native.load().th_operator_info_get(handle, ctypes.byref(info)))
        self.info = info

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _native._lib is not None:
            try:
                _native._lib.th_operator_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None

    def support_layers(self) -> tuple:
        """Reference normal source layers [lo, lo + count) the operator reads."""
        lo, cnt = ctypes.c_int32(), ctypes.c_int32()
        _native.check(_native.load().th_operator_support_layers(self.handle, ctypes.byref(lo), ctypes.byref(cnt)))
        return lo.value, cnt.value

    def source_box(self, selector: int) -> tuple:
        """(lo0, n0, lo1, n1, lo2, n2): reference source cells the kernels read for a segment
        (interpolation) or half code (restriction), along (normal, t1, t2)."""
        box = (ctypes.c_int32 * 6)()
        _native.check(_native.load().th_operator_source_box(self.handle, int(selector), box))
        return tuple(int(v) for v in box)

    @property
    def max_condition(self) -> float:
        return float(self.info.max_condition)

    def export_rows(self, selector: int):
        """(row_offsets, col_indices, values) of a segment (-1 = full face) / half code."""
        lib = _native.load()
        n_rows, nnz = ctypes.c_int64(), ctypes.c_int64()
        _native.check(lib.th_operator_export_rows(self.handle, selector, ctypes.byref(n_rows), ctypes.byref(nnz),
                                                  None, None, None))
        ro = np.zeros(n_rows.value + 1, dtype=np.int64)
        ci = np.zeros(nnz.value, dtype=np.int64)
        va = np.zeros(nnz.value, dtype=np.float64)
        _native.check(lib.th_operator_export_rows(self.handle, selector, ctypes.byref(n_rows), ctypes.byref(nnz),
                                                  ro.ctypes.data, ci.ctypes.data, va.ctypes.data))
        return ro, ci, va

    def csr(self, segment: int | None = None, half: str | None = None) -> CsrOperator:
        p, k = self.p, self.k
        if self.role == "interpolate":
            selector = -1 if segment is None else int(segment)
            src = geometry.ref_interp_source(p, k)
            tgt = (geometry.ref_interp_target_full(p, k) if segment is None
                   else geometry.ref_interp_target_segment(p, k, segment))
        else:
            selector = _native.HALF_CODES[half]
            src = geometry.ref_restrict_source(p, k)
            tgt = geometry.ref_restrict_target(p, k, half)
        ro, ci, va = self.export_rows(selector)
        return CsrOperator(int(ro.size - 1), src.cell_count, ro, ci, va, self.scheme,
                           OperatorKey(self.role, self.scheme, p, k, segment=segment, half=half),
                           src, tgt, self.max_condition)


class DeviceOperator(HostOperator):
    """One uploaded operator (handle to a th_operator on one CUDA device)."""

    on_device = True

    def __init__(self, role: str, scheme: str, p: int, k: int, device: int | None = None):
        torch = _require_torch_cuda()
        self.device = torch.cuda.current_device() if device is None else int(device)
        with torch.cuda.device(self.device):
            self._create(role, scheme, p, k, _native.load().th_operator_create)


class OperatorCache:
    """Memoised device operators, one per (role, scheme, p, k, device); insert under a lock."""

    def __init__(self):
        self._ops: dict = {}
        self._csr: dict = {}
        self._lock = threading.Lock()

    def device_operator(self, role: str, scheme: str, p: int, k: int) -> DeviceOperator:
        torch = _require_torch_cuda()
        key = (role, scheme, p, k, torch.cuda.current_device())
        op = self._ops.get(key)
        if op is None:
            built = DeviceOperator(role, scheme, p, k)
            with self._lock:
                op = self._ops.setdefault(key, built)
        return op

    def host_operator(self, role: str, scheme: str, p: int, k: int) -> HostOperator:
        """Host-built operator (no device upload): CSR views work without a GPU."""
        key = ("host", role, scheme, p, k)
        op = self._ops.get(key)
        if op is None:
            built = HostOperator(role, scheme, p, k)
            with self._lock:
                op = self._ops.setdefault(key, built)
        return op

    def get(self, key: OperatorKey) -> CsrOperator:
        """Reference-compatible: the CSR rows of the keyed row block (host; no GPU needed)."""
        if key.scheme == "tensor_linear":
            raise ConfigurationError("tensor_linear is applied per axis and has no matrix form")
        op = self._csr.get(key)
        if op is None:
            built = self.host_operator(key.role, key.scheme, key.p, key.k).csr(segment=key.segment, half=key.half)
            with self._lock:
                op = self._csr.setdefault(key, built)
        return op

    def clear(self) -> None:
        with self._lock:
            self._ops.clear()
            self._csr.clear()


DEFAULT_CACHE = OperatorCache()


def operator_cache_get(cfg, scheme: str, role: str = "interpolate", half=None, cache=None) -> CsrOperator:
    cache = cache or DEFAULT_CACHE
    if role == "interpolate":
        return cache.get(OperatorKey(role, scheme, cfg.p, cfg.k, segment=cfg.segment))
    return cache.get(OperatorKey(role, scheme, cfg.p, cfg.k, half=half))


def apply(op: CsrOperator, src, out=None):
    """csr.apply on the device (csr.py:159-173): reference-frame AoS source in, HaloBuffer out."""
    torch = _require_torch_cuda()
    from .geometry import HaloBuffer

    if src.region.cell_count != op.n_cols:
        raise ContractViolationError(f"operator expects {op.n_cols} source cells, buffer has {src.region.cell_count}")
    if not np.isfinite(src.values).all():
        raise ContractViolationError("source buffer contains non-finite values")
    dev = torch.device("cuda", torch.cuda.current_device())
    ro = torch.from_numpy(np.ascontiguousarray(op.row_offsets, dtype=np.int64)).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(op.col_indices, dtype=np.int64)).to(dev)
    va = torch.from_numpy(np.ascontiguousarray(op.values, dtype=np.float64)).to(dev)
    s = torch.from_numpy(np.ascontiguousarray(src.values)).to(dev)
    o = torch.empty(op.n_rows * src.u, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    _native.check(_native.load().th_csr_apply(ro.data_ptr(), ci.data_ptr(), va.data_ptr(), op.n_rows,
                                              s.data_ptr(), o.data_ptr(), src.u, stream))
    host = o.cpu().numpy()
    if out is not None:
        out[...] = host
        host = out
    region = op.target_region
    if region is None or region.cell_count != op.n_rows:
        region = RegionShape((op.n_rows, 1, 1), 1.0, (0.0, 0.0, 0.0))
    return HaloBuffer(region, src.u, host)
