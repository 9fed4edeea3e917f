"""Error taxonomy of the B200 halo path.

The class names are the reference's (trihalo/errors.py:4-25) so callers can
catch the same exceptions after switching; the C ABI's integer status codes
(include/trihalo_b200.h, TH_ERR_*) are translated into them by
``_native.check``.
"""


class TrihaloError(Exception):
    """Root of every error raised by this package."""


class ConfigurationError(TrihaloError):
    """Bad face / scheme / role / half arguments (TH_ERR_CONFIG)."""


class ContractViolationError(TrihaloError):
    """Buffer shape, region or finiteness contract broken (TH_ERR_CONTRACT)."""


class SingularFitError(TrihaloError):
    """Rank-deficient least-squares fit during operator construction (TH_ERR_SINGULAR)."""

    def __init__(self, column: int, message: str):
        super().__init__(message)
        self.column = column


class StencilInfeasibleError(TrihaloError):
    """Scheme cannot place its stencil on this (p, k) (TH_ERR_INFEASIBLE)."""


class DeviceError(TrihaloError):
    """CUDA extension missing or a device call failed (TH_ERR_CUDA)."""
