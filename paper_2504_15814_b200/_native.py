"""ctypes binding of the C ABI (include/trihalo_b200.h) in _lib/libtrihalo_b200.so.

There is no CPU fallback: if the shared library is missing or fails to load,
every hot-path call raises DeviceError.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or
``python -m paper_2504_15814_b200.build``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    ConfigurationError,
    ContractViolationError,
    DeviceError,
    SingularFitError,
    StencilInfeasibleError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libtrihalo_b200.so")
# A/B builds of the same ABI (tools/ab_build.sh): TH_LIBPATH points at another copy of the library
LIB_PATH = os.environ.get("TH_LIBPATH", LIB_PATH)

TH_OK, TH_ERR_CONFIG, TH_ERR_INFEASIBLE, TH_ERR_CONTRACT, TH_ERR_SINGULAR, TH_ERR_CUDA = range(6)
ROLES = {"interpolate": 0, "restrict": 1}
SCHEME_CODES = {"tensor_linear": 0, "matrix_linear": 1, "order2": 2, "order3": 3}
HALF_CODES = {None: 0, "inner": 1, "outer": 2}

# numpy mirror of struct th_face (144 bytes)
FACE_DTYPE = np.dtype([
    ("src", "<i8", (9,)),
    ("dst", "<i8"),
    ("src_stride", "<i8", (3,)),
    ("dst_stride", "<i8", (3,)),
    ("normal", "<i4"),
    ("side", "<i4"),
    ("segment", "<i4"),
    ("half", "<i4"),
])
assert FACE_DTYPE.itemsize == 144

# numpy mirror of struct th_box (80 bytes)
BOX_DTYPE = np.dtype([
    ("src", "<i8"),
    ("dst", "<i8"),
    ("src_stride", "<i8", (3,)),
    ("dst_stride", "<i8", (3,)),
    ("ext", "<i4", (3,)),
    ("pad", "<i4"),
])
assert BOX_DTYPE.itemsize == 80


class OperatorInfo(ctypes.Structure):
    _fields_ = [
        ("role", ctypes.c_int32), ("scheme", ctypes.c_int32), ("p", ctypes.c_int32), ("k", ctypes.c_int32),
        ("n_src_cells", ctypes.c_int32), ("n_tgt_cells_full", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
        ("max_items_per_face", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
        ("max_condition", ctypes.c_double), ("n_condition_warnings", ctypes.c_int32), ("kernel", ctypes.c_int32),
    ]


EXPORTED = (
    "th_abi_version", "th_last_error", "th_last_error_column", "th_scheme_feasible", "th_operator_create",
    "th_operator_create_host",
    "th_operator_destroy", "th_operator_info_get", "th_operator_export_rows", "th_apply_faces",
    "th_check_finite", "th_csr_apply", "th_operator_support_layers", "th_copy_box_layers", "th_copy_faces",
    "th_copy_boxes", "th_operator_source_box", "th_memcpy_async", "th_pseudoinverse_rows",
    "th_copy_patch_blocks", "th_pool_blocks",
)

_lib = None
_load_error = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


def load():
    """Load the shared library (raises DeviceError when it is not built)."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"CUDA extension not built: {LIB_PATH} is missing (run __graft_entry__.build())")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        _load_error = exc
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    lib.th_abi_version.restype = _i32
    lib.th_last_error.restype = ctypes.c_char_p
    lib.th_last_error_column.restype = _i32
    lib.th_scheme_feasible.restype = _i32
    lib.th_scheme_feasible.argtypes = [_i32, _i32, _i32, _i32]
    lib.th_operator_create.restype = _i32
    lib.th_operator_create.argtypes = [_i32, _i32, _i32, _i32, ctypes.POINTER(_vp)]
    lib.th_operator_create_host.restype = _i32
    lib.th_operator_create_host.argtypes = [_i32, _i32, _i32, _i32, ctypes.POINTER(_vp)]
    lib.th_operator_destroy.restype = None
    lib.th_operator_destroy.argtypes = [_vp]
    lib.th_operator_info_get.restype = _i32
    lib.th_operator_info_get.argtypes = [_vp, ctypes.POINTER(OperatorInfo)]
    lib.th_operator_export_rows.restype = _i32
    lib.th_operator_export_rows.argtypes = [_vp, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _vp, _vp, _vp]
    lib.th_apply_faces.restype = _i32
    lib.th_apply_faces.argtypes = [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]
    lib.th_check_finite.restype = _i32
    lib.th_check_finite.argtypes = [_vp, _i64, _vp, _vp]
    lib.th_operator_support_layers.restype = _i32
    lib.th_operator_support_layers.argtypes = [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
    lib.th_copy_box_layers.restype = _i32
    lib.th_copy_box_layers.argtypes = [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp]
    lib.th_copy_faces.restype = _i32
    lib.th_copy_faces.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp]
    lib.th_copy_boxes.restype = _i32
    lib.th_copy_boxes.argtypes = [_vp, _vp, _vp, _i64, _i32, _vp]
    lib.th_operator_source_box.restype = _i32
    lib.th_operator_source_box.argtypes = [_vp, _i32, ctypes.POINTER(_i32)]
    lib.th_memcpy_async.restype = _i32
    lib.th_memcpy_async.argtypes = [_vp, _vp, _i64, _i32, _vp]
    lib.th_pseudoinverse_rows.restype = _i32
    lib.th_pseudoinverse_rows.argtypes = [_vp, _i32, _i32, _vp, ctypes.POINTER(ctypes.c_double)]
    lib.th_copy_patch_blocks.restype = _i32
    lib.th_copy_patch_blocks.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i32, _i32, _vp]
    lib.th_pool_blocks.restype = _i32
    lib.th_pool_blocks.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _i32, _vp]
    lib.th_csr_apply.restype = _i32
    lib.th_csr_apply.argtypes = [_vp, _vp, _vp, _i64, _vp, _vp, _i32, _vp]
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Translate a TH_* status into the reference exception classes."""
    if rc == TH_OK:
        return
    lib = load()
    msg = lib.th_last_error().decode("utf-8", "replace")
    if rc == TH_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == TH_ERR_INFEASIBLE:
        raise StencilInfeasibleError(msg)
    if rc == TH_ERR_CONTRACT:
        raise ContractViolationError(msg)
    if rc == TH_ERR_SINGULAR:
        raise SingularFitError(int(lib.th_last_error_column()), msg)
    raise DeviceError(msg)
