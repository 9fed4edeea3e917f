"""Drop-in operator API on the B200 path.

Same names, arguments and error behaviour as trihalo.schemes
(/root/reference/pkg/src/trihalo/schemes.py):
  scheme_feasible / require_feasible  schemes.py:23-53
  build_reference_operator            schemes.py:56-70
  interpolate_halo / restrict_halo    schemes.py:73-101
  apply_scheme                        schemes.py:104-116
  HaloExchange(...).run(src, out)     schemes.py:119-202
Every apply runs the sm_100a kernels through the C ABI; host arrays are
copied to the device and back, CUDA tensors are used in place.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import _native, faces, geometry
from .errors import ConfigurationError, ContractViolationError, StencilInfeasibleError
from .geometry import FaceConfig, HaloBuffer
from .operators import DEFAULT_CACHE, CsrOperator, OperatorCache, OperatorKey

SCHEMES = ("tensor_linear", "matrix_linear", "order2", "order3")
MATRIX_SCHEMES = ("matrix_linear", "order2", "order3")
ROLES = ("interpolate", "restrict")


def _validate(scheme: str, role: str) -> None:
    if scheme not in SCHEMES:
        raise ConfigurationError(f"unknown scheme {scheme!r}; expected one of {SCHEMES}")
    if role not in ROLES:
        raise ConfigurationError(f"role must be 'interpolate' or 'restrict', got {role!r}")


def scheme_feasible(scheme: str, role: str, p: int, k: int) -> tuple:
    _validate(scheme, role)
    geometry.validate_pk(p, k)
    lib = _native.load()
    rc = lib.th_scheme_feasible(_native.ROLES[role], _native.SCHEME_CODES[scheme], p, k)
    if rc == _native.TH_OK:
        return True, ""
    if rc == _native.TH_ERR_INFEASIBLE:
        return False, lib.th_last_error().decode()
    _native.check(rc)
    return False, "unreachable"


def require_feasible(scheme: str, role: str, p: int, k: int) -> None:
    ok, why = scheme_feasible(scheme, role, p, k)
    if not ok:
        raise StencilInfeasibleError(why)


def build_reference_operator(scheme: str, role: str, p: int, k: int, segment=None, half=None,
                             cache: OperatorCache | None = None) -> CsrOperator:
    if scheme == "tensor_linear":
        raise ConfigurationError("tensor_linear is applied per axis and has no matrix form")
    require_feasible(scheme, role, p, k)
    return (cache or DEFAULT_CACHE).get(OperatorKey(role, scheme, p, k, segment=segment, half=half))


def _half_code(role: str, half):
    if role == "interpolate":
        return None
    if half not in (None, "inner", "outer"):
        raise ConfigurationError(f"half must be 'inner', 'outer' or None, got {half!r}")
    return half


class HaloExchange:
    """Reusable single-face exchange: face record, operator and device buffers built once."""

    def __init__(self, cfg: FaceConfig, scheme: str, role: str, half=None, cache: OperatorCache | None = None):
        import torch

        _validate(scheme, role)
        require_feasible(scheme, role, cfg.p, cfg.k)
        self.cfg, self.scheme, self.role = cfg, scheme, role
        self.half = _half_code(role, half)
        p, k, u = cfg.p, cfg.k, cfg.u
        if role == "interpolate":
            ref_src, ref_tgt = geometry.ref_interp_source(p, k), geometry.ref_interp_target_segment(p, k, cfg.segment)
        else:
            ref_src, ref_tgt = geometry.ref_restrict_source(p, k), geometry.ref_restrict_target(p, k, self.half)
        inv = geometry.reference_frame(cfg).inverse()
        self.source_region = inv.map_region(ref_src)
        self.target_region = inv.map_region(ref_tgt)
        self.n_src = self.source_region.cell_count * u
        self.n_out = self.target_region.cell_count * u
        self.op = (cache or DEFAULT_CACHE).device_operator(role, scheme, p, k)
        rec = faces.slab_faces(role, p, k, u, [cfg.normal], [cfg.side],
                               segments=[cfg.segment] if role == "interpolate" else None, half=self.half)
        self.batch = faces.FaceBatch(self.op, rec, u)
        dev = torch.device("cuda", self.op.device)
        self._src = torch.empty(max(self.n_src, 1), dtype=torch.float64, device=dev)
        self._out = torch.empty(max(self.n_out, 1), dtype=torch.float64, device=dev)
        # page-locked staging for host callers: one H2D, two kernels, one D2H of the result and
        # the non-finite flag, ONE synchronisation per run
        self._h_src = torch.empty(max(self.n_src, 1), dtype=torch.float64, pin_memory=True)
        self._h_out = torch.empty(max(self.n_out, 1), dtype=torch.float64, pin_memory=True)
        self._h_flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._h_src_np, self._h_out_np = self._h_src.numpy(), self._h_out.numpy()

    def make_buffers(self, rng: np.random.Generator | None = None):
        src = rng.standard_normal(self.n_src) if rng is not None else np.zeros(self.n_src)
        return src, np.zeros(self.n_out)

    def _device_check(self, t, n: int, what: str) -> None:
        import torch

        if t.dtype != torch.float64 or not t.is_contiguous() or t.device != self._src.device:
            raise ContractViolationError(f"{what} must be a contiguous float64 tensor on {self._src.device}, got "
                                         f"{t.dtype} on {t.device} (contiguous={t.is_contiguous()})")
        if t.numel() != n:
            raise ContractViolationError(f"{what} needs {n} values, got {t.numel()}")

    def run(self, src_values, out_values) -> None:
        """out_values[:] = operator(src_values); numpy arrays or CUDA tensors (world layout).

        Like the reference (schemes.py:185-202) the source is checked for non-finite values
        before anything is written: the result is computed into the exchange's own buffer and
        copied into ``out_values`` only after the check passed."""
        import torch

        out_dev = isinstance(out_values, torch.Tensor) and out_values.is_cuda
        src_dev = isinstance(src_values, torch.Tensor) and src_values.is_cuda
        if out_dev:
            self._device_check(out_values, self.n_out, "output")
        elif np.asarray(out_values).size != self.n_out:
            raise ContractViolationError(f"output needs {self.n_out} values, got {np.asarray(out_values).size}")
        if src_dev:
            self._device_check(src_values, self.n_src, "source")
        if not src_dev and not out_dev:
            return self._run_host(src_values, out_values)
        if src_dev:
            src_t = src_values
        else:
            src_np = np.asarray(src_values, dtype=np.float64)
            if src_np.size != self.n_src:
                raise ContractViolationError(f"source needs {self.n_src} values, got {src_np.size}")
            self._src.copy_(torch.from_numpy(np.ascontiguousarray(src_np).reshape(-1)))
            src_t = self._src
        if self.n_out == 0:
            return
        # whole-source finiteness, as the reference checks before applying (schemes.py:186)
        stream = torch.cuda.current_stream().cuda_stream
        _native.check(_native.load().th_check_finite(src_t.data_ptr(), self.n_src, self.batch.flag.data_ptr(), stream))
        self.batch.launch(src_t, self._out, check_flag=False)
        if self.batch.nonfinite():
            raise ContractViolationError("source buffer contains non-finite values")
        if out_dev:
            out_values.copy_(self._out[: self.n_out])
        else:
            np.copyto(np.asarray(out_values).reshape(-1), self._out[: self.n_out].cpu().numpy())

    def _run_host(self, src_values, out_values) -> None:
        """Host arrays in and out: staged through page-locked buffers, one sync."""
        import torch

        src_np = np.asarray(src_values, dtype=np.float64).reshape(-1)
        if src_np.size != self.n_src:
            raise ContractViolationError(f"source needs {self.n_src} values, got {src_np.size}")
        if self.n_out == 0:
            return
        lib = _native.load()
        stream = torch.cuda.current_stream(self._src.device)
        s = stream.cuda_stream
        np.copyto(self._h_src_np[: self.n_src], src_np)
        _native.check(lib.th_memcpy_async(self._src.data_ptr(), self._h_src.data_ptr(), self.n_src * 8, 0, s))
        flag = self.batch.flag
        _native.check(lib.th_check_finite(self._src.data_ptr(), self.n_src, flag.data_ptr(), s))
        self.batch.launch(self._src, self._out, stream=s, check_flag=False)
        _native.check(lib.th_memcpy_async(self._h_out.data_ptr(), self._out.data_ptr(), self.n_out * 8, 1, s))
        _native.check(lib.th_memcpy_async(self._h_flag.data_ptr(), flag.data_ptr(), 4, 1, s))
        stream.synchronize()
        if int(self._h_flag_np()[0]):
            flag.zero_()
            raise ContractViolationError("source buffer contains non-finite values")
        np.copyto(np.asarray(out_values).reshape(-1), self._h_out_np[: self.n_out])

    def _h_flag_np(self):
        return self._h_flag.numpy()


_EXCHANGES: dict = {}          # exchanges built with the default cache
_EXCHANGES_BY_CACHE = None     # weak: an OperatorCache's exchanges die with it
_EXCHANGE_LIMIT = 4096         # per cache: (orientation x segment / half x scheme x role) fits easily


def _exchange(cfg, scheme, role, half, cache) -> HaloExchange:
    global _EXCHANGES_BY_CACHE
    import weakref

    if cache is None:
        table = _EXCHANGES
    else:
        if _EXCHANGES_BY_CACHE is None:
            _EXCHANGES_BY_CACHE = weakref.WeakKeyDictionary()
        table = _EXCHANGES_BY_CACHE.setdefault(cache, {})
    key = (cfg, scheme, role, half)
    ex = table.get(key)
    if ex is None:
        if len(table) >= _EXCHANGE_LIMIT:
            table.clear()
        ex = table[key] = HaloExchange(cfg, scheme, role, half=half, cache=cache)
    return ex


def interpolate_halo(cfg: FaceConfig, scheme: str, coarse: HaloBuffer, cache: OperatorCache | None = None) -> HaloBuffer:
    """Fill cfg.segment's fine block from the coarse source (any scheme) on the GPU."""
    _validate(scheme, "interpolate")
    require_feasible(scheme, "interpolate", cfg.p, cfg.k)
    if coarse.region != geometry.interp_source_shape(cfg):
        raise ContractViolationError(f"buffer region {coarse.region} is not the interpolation source of {cfg}")
    cfg = dataclasses.replace(cfg, u=coarse.u)  # like the reference, the buffer's u rules
    ex = _exchange(cfg, scheme, "interpolate", None, cache)
    out = np.empty(ex.n_out)
    ex.run(coarse.values, out)
    return HaloBuffer(ex.target_region, cfg.u, out)


def restrict_halo(cfg: FaceConfig, scheme: str, fine: HaloBuffer, half=None,
                  cache: OperatorCache | None = None) -> HaloBuffer:
    """Fill the coarse halo (or one half of its depth) from the fine source on the GPU."""
    _validate(scheme, "restrict")
    half = _half_code("restrict", half)
    require_feasible(scheme, "restrict", cfg.p, cfg.k)
    if fine.region != geometry.restrict_source_shape(cfg):
        raise ContractViolationError(f"buffer region {fine.region} is not the restriction source of {cfg}")
    cfg = dataclasses.replace(cfg, u=fine.u)
    ex = _exchange(cfg, scheme, "restrict", half, cache)
    out = np.empty(ex.n_out)
    ex.run(fine.values, out)
    return HaloBuffer(ex.target_region, cfg.u, out)


def apply_scheme(cfg: FaceConfig, scheme: str, role: str, src: HaloBuffer, half=None,
                 cache: OperatorCache | None = None) -> HaloBuffer:
    if role == "interpolate":
        return interpolate_halo(cfg, scheme, src, cache=cache)
    if role == "restrict":
        return restrict_halo(cfg, scheme, src, half=half, cache=cache)
    raise ConfigurationError(f"role must be 'interpolate' or 'restrict', got {role!r}")
