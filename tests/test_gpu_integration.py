"""The reference-side ctypes binding (integration/trihalo_b200_ctypes.py) on
a B200: B200Exchange against the oracle for every scheme, role and half, and -- when the
reference is installed next to the repo (baseline/_ref, git-ignored) -- the unmodified
reference's own HaloExchange patched to dispatch to the B200, against its own CPU results."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
CASES = [(s, r, h) for s in ("tensor_linear", "matrix_linear", "order2", "order3")
         for r, h in (("interpolate", None), ("restrict", None), ("restrict", "inner"), ("restrict", "outer"))]


@pytest.fixture(scope="module")
def binding():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from integration import trihalo_b200_ctypes as B

    return B


@pytest.mark.parametrize("scheme,role,half", CASES)
def test_binding_matches_oracle(binding, scheme, role, half):
    import paper_2504_15814_b200 as th
    from oracle import exchange as OE
    from oracle import geometry as OG

    rng = np.random.default_rng(7)
    for normal, side, seg in (("x", "negative", 0), ("y", "positive", 4), ("z", "positive", 8)):
        cfg = th.FaceConfig(normal, side, seg, 9, 3, 59)
        ex = binding.B200Exchange(cfg, scheme, role, half=half)
        src = rng.standard_normal(ex.n_src)
        out = np.full(ex.n_out, np.nan)
        ex.run(src, out)
        want = np.empty(ex.n_out)
        OE.exchange_for(OG.FaceCfg(normal, side, seg, 9, 3, 59), scheme, role, half=half).run(src, want)
        assert np.abs(out - want).max() <= 1e-12 * np.abs(want).max(), (scheme, role, half, normal)
    src[3] = np.inf
    keep = out.copy()
    with pytest.raises(ValueError):
        ex.run(src, out)
    assert np.array_equal(out, keep, equal_nan=True)  # nothing written before the check


def test_patched_reference_matches_its_cpu_path(binding):
    if not os.path.isdir(os.path.join(REF, "trihalo")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import trihalo
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(3)
    cfgs = [trihalo.FaceConfig(n, s, seg, 9, 3, 59) for n, s, seg in (("x", "positive", 2), ("z", "negative", 6))]
    wants = []
    for cfg in cfgs:
        for scheme, role, half in CASES:
            ex = trihalo.HaloExchange(cfg, scheme, role, half=half)
            src, out = ex.make_buffers(rng)
            ex.run(src, out)
            wants.append((cfg, scheme, role, half, src, out.copy()))
    binding.patch_reference(trihalo)
    try:
        for cfg, scheme, role, half, src, want in wants:
            ex = trihalo.HaloExchange(cfg, scheme, role, half=half)
            out = np.empty_like(want)
            ex.run(src, out)
            assert np.abs(out - want).max() <= 1e-12 * np.abs(want).max(), (scheme, role, half)
        bad = src.copy()
        bad[0] = np.nan
        with pytest.raises(trihalo.errors.ContractViolationError):
            ex.run(bad, out)
    finally:
        sys.modules.pop("trihalo", None)
