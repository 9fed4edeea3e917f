"""Reference-side binding of the B200 path: a ctypes stub a `trihalo` maintainer would add.

It talks to the C ABI (include/trihalo_b200.h) and to the CUDA runtime through ctypes only --
no torch, no paper_2504_15814_b200 import -- so it can live inside the reference package as
``trihalo/_b200.py``.  Two entry points:

* ``B200Exchange(cfg, scheme, role, half=None)`` with ``.run(src_values, out_values)`` -- the
  contract of ``trihalo.schemes.HaloExchange.run`` (schemes.py:185-202): world-layout float64
  numpy buffers, ``out`` written in place, ContractViolationError-style ValueError on a size
  mismatch or non-finite source (checked before ``out`` is touched).
* ``patch_reference(trihalo)`` -- makes an imported reference package dispatch every
  ``HaloExchange.run`` to the B200 path (its __init__, regions and buffers stay the
  reference's own), e.g. behind an environment flag in ``trihalo/__init__.py``:

      if os.environ.get("TRIHALO_B200"):
          from . import _b200; _b200.patch_reference(sys.modules[__name__])

Library lookup: TRIHALO_B200_LIB, else the in-tree build next to this file's repository.
"""

from __future__ import annotations

import ctypes
import ctypes.util
import glob
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("TRIHALO_B200_LIB",
                     os.path.join(_HERE, "..", "paper_2504_15814_b200", "_lib", "libtrihalo_b200.so"))

ROLE = {"interpolate": 0, "restrict": 1}
SCHEME = {"tensor_linear": 0, "matrix_linear": 1, "order2": 2, "order3": 3}
HALF = {None: 0, "inner": 1, "outer": 2}
AXES = ("x", "y", "z")
SIDES = ("negative", "positive")

# struct th_face (144 bytes)
FACE = np.dtype([("src", "<i8", (9,)), ("dst", "<i8"), ("src_stride", "<i8", (3,)), ("dst_stride", "<i8", (3,)),
                 ("normal", "<i4"), ("side", "<i4"), ("segment", "<i4"), ("half", "<i4")])

_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64


def _cudart():
    cands = [os.environ.get("TRIHALO_CUDART", "")]
    cands += [ctypes.util.find_library("cudart") or ""]
    cands += sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))
    for site in __import__("site").getsitepackages():
        cands += sorted(glob.glob(os.path.join(site, "nvidia", "cuda_runtime", "lib", "libcudart.so*")))
    for c in cands:
        if c:
            try:
                return ctypes.CDLL(c)
            except OSError:
                pass
    raise OSError("libcudart not found (set TRIHALO_CUDART)")


_th = None
_rt = None


def _libs():
    global _th, _rt
    if _th is None:
        _rt = _cudart()
        _rt.cudaMalloc.argtypes = [ctypes.POINTER(_vp), ctypes.c_size_t]
        _rt.cudaFree.argtypes = [_vp]
        _rt.cudaMemcpy.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int]
        _rt.cudaMemset.argtypes = [_vp, ctypes.c_int, ctypes.c_size_t]
        _rt.cudaDeviceSynchronize.argtypes = []
        th = ctypes.CDLL(LIB)
        th.th_last_error.restype = ctypes.c_char_p
        th.th_operator_create.argtypes = [_i32, _i32, _i32, _i32, ctypes.POINTER(_vp)]
        th.th_operator_destroy.argtypes = [_vp]
        th.th_apply_faces.argtypes = [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]
        th.th_check_finite.argtypes = [_vp, _i64, _vp, _vp]
        _th = th
    return _th, _rt


def _check(rc):
    if rc:
        raise RuntimeError(f"trihalo_b200: {_libs()[0].th_last_error().decode()} (status {rc})")


def _cuda(rc, what):
    if rc:
        raise RuntimeError(f"CUDA {what} failed ({rc})")


class _Device:
    """One device allocation (cudaMalloc / cudaFree)."""

    def __init__(self, nbytes):
        self.nbytes = max(int(nbytes), 8)
        self.ptr = _vp()
        _cuda(_libs()[1].cudaMalloc(ctypes.byref(self.ptr), self.nbytes), "cudaMalloc")

    def put(self, a: np.ndarray):
        _cuda(_libs()[1].cudaMemcpy(self.ptr, a.ctypes.data, a.nbytes, 1), "cudaMemcpy H2D")

    def get(self, a: np.ndarray):
        _cuda(_libs()[1].cudaMemcpy(a.ctypes.data, self.ptr, a.nbytes, 2), "cudaMemcpy D2H")

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value and _rt is not None:
            _rt.cudaFree(self.ptr)


def _world_strides(normal, n_ext, t_ext, u):
    ext = [t_ext, t_ext, t_ext]
    ext[normal] = n_ext
    return np.array([u, u * ext[0], u * ext[0] * ext[1]], dtype=np.int64)


def face_record(role, normal, side, segment, half, p, k, u) -> np.ndarray:
    """th_face of one face whose source / target are the reference's contiguous world buffers
    (geometry.py:244-265): x-fastest boxes, the source extent 2k along the normal."""
    rec = np.zeros(1, dtype=FACE)
    rec["normal"], rec["side"] = normal, side
    if role == "interpolate":
        rec["segment"] = segment
        rec["src_stride"] = _world_strides(normal, 2 * k, p, u)
        n_tgt = k
    else:
        rec["half"] = HALF[half]
        ss = _world_strides(normal, 2 * k, 3 * p, u)
        rec["src_stride"] = ss
        t1 = 1 if normal == 0 else 0
        t2 = 1 if normal == 2 else 2
        for b in range(9):  # low corners of the nine fine blocks
            rec["src"][0, b] = (b % 3) * p * ss[t1] + (b // 3) * p * ss[t2]
        inner = (k + 1) // 2
        n_tgt = {None: k, "inner": inner, "outer": k - inner}[half]
    rec["dst_stride"] = _world_strides(normal, n_tgt, p, u)
    return rec


class B200Exchange:
    """HaloExchange.run on the B200 (schemes.py:185-202)."""

    def __init__(self, cfg, scheme, role, half=None):
        th, _ = _libs()
        self.u, p, k = int(cfg.u), int(cfg.p), int(cfg.k)
        normal, side = AXES.index(cfg.normal_axis), SIDES.index(cfg.coarse_side)
        self.op = _vp()
        _check(th.th_operator_create(ROLE[role], SCHEME[scheme], p, k, ctypes.byref(self.op)))
        if role == "interpolate":
            self.n_src, self.n_out = 2 * k * p * p * self.u, k * p * p * self.u
        else:
            inner = (k + 1) // 2
            rows = {None: k, "inner": inner, "outer": k - inner}[half]
            self.n_src, self.n_out = 2 * k * 9 * p * p * self.u, rows * p * p * self.u
        rec = face_record(role, normal, side, cfg.segment, half, p, k, self.u)
        self._rec = _Device(rec.nbytes)
        self._rec.put(rec)
        self._src, self._out, self._flag = _Device(self.n_src * 8), _Device(self.n_out * 8), _Device(4)
        self._host_flag = np.zeros(1, dtype=np.int32)

    def run(self, src_values, out_values) -> None:
        th, rt = _libs()
        src = np.ascontiguousarray(src_values, dtype=np.float64).reshape(-1)
        out = np.asarray(out_values).reshape(-1)
        if src.size != self.n_src or out.size != self.n_out:
            raise ValueError(f"source / output need {self.n_src} / {self.n_out} values, got {src.size} / {out.size}")
        self._src.put(src)
        _cuda(rt.cudaMemset(self._flag.ptr, 0, 4), "cudaMemset")
        _check(th.th_check_finite(self._src.ptr, self.n_src, self._flag.ptr, None))
        _check(th.th_apply_faces(self.op, self._src.ptr, self._out.ptr, self._rec.ptr, 1, self.u, None, None))
        self._flag.get(self._host_flag)  # synchronous: the apply finished
        if self._host_flag[0]:
            raise ValueError("source buffer contains non-finite values")
        result = np.empty(self.n_out)
        self._out.get(result)
        out[:] = result

    def __del__(self):
        if getattr(self, "op", None) is not None and self.op.value and _th is not None:
            _th.th_operator_destroy(self.op)


def patch_reference(trihalo) -> None:
    """Route the reference's HaloExchange.run through the B200 path (the reference's own
    ContractViolationError is raised for bad buffers)."""
    HX = trihalo.schemes.HaloExchange
    errors = trihalo.errors
    if getattr(HX, "_b200_patched", False):
        return
    original_init = HX.__init__

    def __init__(self, cfg, scheme, role, half=None, cache=None):
        original_init(self, cfg, scheme, role, half=half, cache=cache)
        self._b200 = B200Exchange(cfg, scheme, role, half=half if role == "restrict" else None)

    def run(self, src_values, out_values):
        try:
            self._b200.run(src_values, out_values)
        except ValueError as exc:
            raise errors.ContractViolationError(str(exc)) from exc

    HX.__init__, HX.run, HX._b200_patched = __init__, run, True
