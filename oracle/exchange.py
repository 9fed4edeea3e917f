"""Oracle per-face exchange (TEST INFRASTRUCTURE ONLY).

Restates ``HaloExchange`` (/root/reference/pkg/src/trihalo/schemes.py:119-202):
precomputed int64 gather/scatter maps ``cell*u + lane`` (schemes.py:147-151),
the reference-face operator (CSR, or the three axis matrices for
``tensor_linear``, schemes.py:155-176) and a ``run`` that checks finiteness,
gathers, applies, scatters (schemes.py:185-202).  The apply itself is the C
restatement in ``trihalo_oracle.c`` (the reference's Numba kernel).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import geometry as G
from . import operators as O

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Ex(ctypes.Structure):
    _fields_ = [
        ("row_offsets", _i64p), ("col_indices", _i64p), ("values", _f64p), ("n_rows", ctypes.c_int64),
        ("mx", _f64p), ("my", _f64p), ("mz", _f64p),
        ("ax", ctypes.c_int64), ("ay", ctypes.c_int64), ("az", ctypes.c_int64),
        ("nz", ctypes.c_int64), ("ny", ctypes.c_int64), ("nx", ctypes.c_int64),
        ("gather", _i64p), ("n_src", ctypes.c_int64),
        ("scatter", _i64p), ("n_out", ctypes.c_int64), ("u", ctypes.c_int64),
    ]


def build_native() -> str:
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "trihalo_oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_native())
        _lib.oracle_exchange_run.restype = ctypes.c_int
        _lib.oracle_exchange_run.argtypes = [ctypes.POINTER(_Ex), _f64p, _f64p, _f64p]
        _lib.oracle_exchange_scratch.restype = ctypes.c_int64
        _lib.oracle_exchange_scratch.argtypes = [ctypes.POINTER(_Ex)]
        _lib.oracle_exchange_many.restype = None
        _lib.oracle_exchange_many.argtypes = [ctypes.POINTER(ctypes.POINTER(_Ex)), ctypes.POINTER(_f64p),
                                              ctypes.POINTER(_f64p), ctypes.c_int64, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int)]
    return _lib


def _p64(a):
    return a.ctypes.data_as(_i64p)


def _pf(a):
    return a.ctypes.data_as(_f64p)


class NonFinite(Exception):
    pass


class OracleExchange:
    """Reusable oracle exchange for one (cfg, scheme, role, half)."""

    def __init__(self, cfg: G.FaceCfg, scheme: str, role: str, half=None):
        self.cfg, self.scheme, self.role, self.half = cfg, scheme, role, half
        p, k, u = cfg.p, cfg.k, cfg.u
        fr = G.frame_for(cfg)
        if role == "interpolate":
            ref_src, ref_tgt = G.ref_interp_source(p, k), G.ref_interp_target_segment(p, k, cfg.segment)
        else:
            ref_src, ref_tgt = G.ref_restrict_source(p, k), G.ref_restrict_target(p, k, half)
        self.source_region = fr.inverse().map_region(ref_src)
        self.target_region = fr.inverse().map_region(ref_tgt)
        src_cells = G.gather_cells(fr, self.source_region)
        tgt_cells = G.gather_cells(fr.inverse(), ref_tgt)
        lanes = np.arange(u, dtype=np.int64)
        self.gather = (src_cells[:, None] * u + lanes).ravel()
        self.scatter = (tgt_cells[:, None] * u + lanes).ravel()
        self.src_cells, self.tgt_cells = src_cells, tgt_cells
        ex = _Ex()
        ex.gather, ex.n_src = _p64(self.gather), self.gather.size
        ex.scatter, ex.n_out = _p64(self.scatter), self.scatter.size
        ex.u = u
        if scheme == "tensor_linear":
            self.op = None
            if role == "interpolate":
                ys, zs = O.segment_slices(p, cfg.segment)
                pt = O.axis_tangential(p)
                mats = (O.axis_normal(k), pt[ys], pt[zs])
            else:
                rt = O.restrict_axis_tangential(p)
                mats = (O.restrict_axis_normal(k)[O.half_slice(k, half)], rt, rt)
            self.mats = tuple(np.ascontiguousarray(m) for m in mats)
            nx, ny, nz = ref_src.extents
            ex.mx, ex.my, ex.mz = (_pf(m) for m in self.mats)
            ex.ax, ex.ay, ex.az = (m.shape[0] for m in self.mats)
            ex.nz, ex.ny, ex.nx = nz, ny, nx
        else:
            self.op = O.build_operator(scheme, role, p, k,
                                       segment=cfg.segment if role == "interpolate" else None,
                                       half=half if role == "restrict" else None)
            ex.row_offsets, ex.col_indices = _p64(self.op.row_offsets), _p64(self.op.col_indices)
            ex.values, ex.n_rows = _pf(self.op.values), self.op.n_rows
        self._ex = ex
        self._scratch = np.empty(max(1, lib().oracle_exchange_scratch(ctypes.byref(ex))))

    @property
    def n_src(self):
        return self.gather.size

    @property
    def n_out(self):
        return self.scatter.size

    def run(self, src: np.ndarray, out: np.ndarray) -> None:
        src = np.ascontiguousarray(src, dtype=np.float64)
        assert src.size == self.n_src and out.size == self.n_out and out.flags.c_contiguous
        rc = lib().oracle_exchange_run(ctypes.byref(self._ex), _pf(src), _pf(out), _pf(self._scratch))
        if rc != 0:
            raise NonFinite("source buffer contains non-finite values")


def run_many(exchanges, srcs, outs, nthreads: int) -> np.ndarray:
    """Run many (exchange, src, out) triples over nthreads OpenMP threads."""
    n = len(exchanges)
    exs = (ctypes.POINTER(_Ex) * n)(*[ctypes.pointer(e._ex) for e in exchanges])
    sp = (_f64p * n)(*[_pf(s) for s in srcs])
    op = (_f64p * n)(*[_pf(o) for o in outs])
    status = np.zeros(n, dtype=np.int32)
    lib().oracle_exchange_many(exs, sp, op, n, int(nthreads), status.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return status


_EX_CACHE: dict = {}


def exchange_for(cfg: G.FaceCfg, scheme: str, role: str, half=None) -> OracleExchange:
    key = (cfg, scheme, role, half)
    ex = _EX_CACHE.get(key)
    if ex is None:
        ex = _EX_CACHE[key] = OracleExchange(cfg, scheme, role, half)
    return ex


def interpolate(cfg: G.FaceCfg, scheme: str, src: np.ndarray) -> np.ndarray:
    ex = exchange_for(cfg, scheme, "interpolate")
    out = np.empty(ex.n_out)
    ex.run(src, out)
    return out


def restrict(cfg: G.FaceCfg, scheme: str, src: np.ndarray, half=None) -> np.ndarray:
    ex = exchange_for(cfg, scheme, "restrict", half)
    out = np.empty(ex.n_out)
    ex.run(src, out)
    return out
