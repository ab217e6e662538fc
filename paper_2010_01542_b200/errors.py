"""Exception taxonomy of the reference (errors.py:4-33), kept verbatim in
meaning so callers' ``except`` clauses keep working.  C-ABI status codes map
onto these: PGX_EINVAL -> ConfigError, anything else -> ExecutionError."""


class PregeliteError(Exception):
    """Base class for all package-specific errors."""


class GraphLoadError(PregeliteError):
    """An edge list or graph cache cannot be parsed / is invalid."""


class ConfigError(PregeliteError):
    """Invalid run configuration, or a program with no device lowering."""


class ValidationError(PregeliteError):
    """A result fails comparison against its reference implementation."""


class ExecutionError(PregeliteError):
    """A device-side failure during a run (CUDA / NCCL error)."""


class PhaseError(PregeliteError):
    """Kept for API compatibility: sends are phase-correct by construction
    on the device (a kernel boundary / grid barrier separates phases)."""
