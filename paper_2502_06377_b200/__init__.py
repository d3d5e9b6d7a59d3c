"""B200-native IBMI sweep (iterative block matrix inversion, arXiv 2502.06377).

Drop-in for the reference package's solver path: the names re-exported here
follow ``ibmi/__init__.py:11-79``: the solver, partition, exception, dense-core
(``linalg``), diagnostics (``analysis``) and matrix-file (``matio``) surfaces.  Not
re-exported, out of scope: the covariance-kernel generators
(``kernel_matrix``, ``KernelSpec``, ``PointSet``, ``grid_1d/2d``, ``FAMILIES``), the
CSV experiment harness (``run_experiment`` …) and the public ``ldlt``.  All arithmetic runs in ``libibmi_b200.so`` (FP64 DMMA kernels for
sm_100a, C ABI in ``include/ibmi_b200.h``); there is no CPU fallback.
"""

from .exceptions import (  # noqa: F401
    DeviceError,
    DimensionMismatch,
    DuplicateWithinSet,
    IndexOutOfRange,
    InvalidHyperparameter,
    InvalidOverlap,
    IoError,
    NoConvergenceWarning,
    NotPerfectSquare,
    NotPositiveDefinite,
    OutOfMemoryBudget,
    TooManyBlocks,
    UncoveredIndices,
    ZeroPivot,
)
from .analysis import (  # noqa: F401
    CostBreakdown,
    condition_number_2,
    contraction_factor,
    flop_cost,
    lemma_error_recurrence_check,
    newton_schultz,
    spectral_radius_condition,
)
from .linalg import (  # noqa: F401
    CholeskyFactor,
    chol_solve,
    cholesky,
    gather,
    matmul,
    scatter_add_assign,
    spd_inverse,
    two_norm,
)
from .matio import load_csv, load_ibmi, load_matrix, save_csv, save_ibmi, save_matrix  # noqa: F401
from .partition import (  # noqa: F401
    Partition,
    complement,
    contiguous_partition,
    load_partition_json,
    overlap_depth,
    red_black_partition,
    validate,
)
from .solver import (  # noqa: F401
    GUESS_CHOICES,
    IbmiConfig,
    SolveReport,
    block_update,
    error_estimate,
    initial_guess_identity,
    initial_guess_local_inverse,
    initial_guess_monte_carlo,
    initial_guess_takahashi,
    make_initial_guess,
    solve,
)

__version__ = "0.1.0"


def load_library():
    """Load libibmi_b200.so now (raises if it is missing)."""
    from . import _abi

    return _abi.lib()


def release_cached_memory(device: int = -1) -> None:
    """Return the device blocks the library keeps between solves to the driver
    (``device < 0``: every device).  See ``ibmi_release_cached_memory``."""
    from . import _abi

    _abi.check(_abi.lib().ibmi_release_cached_memory(int(device)), "release_cached_memory")


def cached_bytes(device: int = -1) -> int:
    """Bytes of device memory held in the library's block cache."""
    import ctypes

    from . import _abi

    out = ctypes.c_int64()
    _abi.check(_abi.lib().ibmi_cached_bytes(int(device), ctypes.byref(out)), "cached_bytes")
    return int(out.value)
