"""B200-native halo interpolation / restriction for 3:1 AMR patch faces.

Drop-in for the hot path of the reference package ``trihalo``
(/root/reference/pkg/src/trihalo/__init__.py:6-53): the operator API
(interpolate_halo, restrict_halo, apply_scheme, HaloExchange,
scheme_feasible, build_reference_operator, operator caches), its geometry
types and its exception classes.  The arithmetic runs in sm_100a CUDA
kernels behind the C ABI of include/trihalo_b200.h; operators are built on
the host in C++ and uploaded once per (role, scheme, p, k).  Batched,
device-resident faces go through ``faces.FaceBatch``.
"""

from .errors import (
    ConfigurationError,
    ContractViolationError,
    DeviceError,
    SingularFitError,
    StencilInfeasibleError,
    TrihaloError,
)
from .geometry import (
    DEFAULT_UNKNOWNS,
    FaceConfig,
    HaloBuffer,
    RegionShape,
    ReferenceFrame,
    from_reference,
    gather_cell_indices,
    interp_source_shape,
    interp_target_shape,
    reference_frame,
    restrict_source_shape,
    restrict_target_shape,
    to_reference,
)
from .operators import CsrOperator, DeviceOperator, OperatorCache, OperatorKey, apply, operator_cache_get
from .schemes import (
    MATRIX_SCHEMES,
    SCHEMES,
    HaloExchange,
    apply_scheme,
    build_reference_operator,
    interpolate_halo,
    require_feasible,
    restrict_halo,
    scheme_feasible,
)
from .faces import FaceBatch, copy_faces, pool_interp_faces, pool_restrict_faces, pool_same_level_faces, slab_faces
from .construction import (
    AxisOperator,
    DerivativeFit,
    StencilSpec,
    TaylorBasis,
    apply_tensor_interpolate,
    apply_tensor_restrict,
    build_axis_normal,
    build_axis_tangential,
    build_derivative_fit,
    build_interpolation,
    build_restriction,
    collapse_to_matrix,
    nearest_source_cell,
    select_stencil,
    taylor_basis,
)
from .csrio import dump_operator, dumps_operator, extract_half, extract_segment, from_triplets, load_operator
from .harness import (
    BenchReport,
    ConvergenceReport,
    run_bench,
    run_consistency_suite,
    run_convergence,
    run_unit_oracle,
    sample_field,
)

__version__ = "0.1.0"
