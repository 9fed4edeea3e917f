"""CPU oracle for the halo interpolation / restriction hot path.

TEST INFRASTRUCTURE ONLY.  This package restates the reference
``trihalo`` algorithm (``/root/reference/pkg/src/trihalo``) on the host so
that the B200 product path can be checked against it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it, and only as the checker or as the
timed CPU reference.  The product package ``paper_2504_15814_b200`` never
imports it: the product has its own host-side operator builder (C++) and
its own CUDA kernels.

Pinning: the restatement is checked against golden vectors produced by the
real reference in the build container (``tests/golden/make_golden.py`` ->
``tests/golden/*.npz``) and against the reference's own known-answer tests
(``pkg/tests/test_csr.py:185-194`` GOLDEN_P1K1, ``test_linear.py:19-75``,
``test_linalg.py:54-61``, ``test_taylor.py:45-117``, ``test_geometry.py:148-165``).

Layout:
  geometry.py   regions, reference frames, gather maps       (geometry.py)
  operators.py  CSR canonicalisation, linear + Taylor builds (csr.py, linear.py, taylor.py, linalg.py)
  exchange.py   the per-face HaloExchange pipeline (schemes.py) over the C
                restatement in trihalo_oracle.c of the reference's Numba CSR
                kernel and tensor contraction (built by oracle/Makefile)
"""

from .geometry import (  # noqa: F401
    FaceCfg,
    Region,
    Frame,
    frame_for,
    gather_cells,
    interp_source_world,
    interp_target_world,
    restrict_source_world,
    restrict_target_world,
)
from .operators import Csr, build_operator, full_face_operator  # noqa: F401
from .exchange import OracleExchange, interpolate, restrict  # noqa: F401
