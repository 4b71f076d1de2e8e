"""B200-native SPD-KFAC optimizer step (arxiv 2107.06533), drop-in for the
reference `kfacsched` package's optimizer path.

Host policy (plans, cost models) is pure Python; all arithmetic runs in
hand-written sm_100a CUDA kernels reached through the C-ABI library
`lib/libspdkfac.so` (see include/spdkfac.h).  There is no CPU fallback:
importing the GPU-facing modules without the built library raises.
"""

from .perfmodel import (  # noqa: F401
    AllReduceParams, BcastParams, InverseParams, MarginalInverseParams, BenchSample, PerfParams,
    allreduce_time, bcast_time, inverse_time, fit_linear, fit_exponential,
    nct_threshold, read_params, write_params,
)
from .planner import (  # noqa: F401
    FactorKind, FactorTask, FusionPlan, FusionPolicy, InvTask, PlacementPlan,
    plan_fusion, lbp_place, seq_place, local_place, placement_makespan,
)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-facing API is loaded lazily so that host planning works on CPU-only
    # machines; touching it without the CUDA library fails loudly.
    if name in ("compute_factor_A", "compute_factor_G", "damped_inverse", "precondition",
                "pack_upper", "unpack_upper", "NotPositiveDefiniteError", "compute_factor_A_conv"):
        from . import linalg
        return getattr(linalg, name)
    if name in ("SPDKFAC",):
        from .optimizer import SPDKFAC
        return SPDKFAC
    raise AttributeError(name)
