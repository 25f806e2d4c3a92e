"""B200-native L1 phase unwrapper (IRLS + PCG, arXiv 2401.09961).

Drop-in for the reference package's hot path `phaseirls.unwrap`
(irls.py:132-224): same signature, dataclasses and trace, with every array
operation executed by hand-written sm_100a CUDA kernels in
`_lib/libpu_unwrap.so` (C ABI: include/pu_unwrap.h).  There is no CPU
fallback; calling into the solver without the library or a GPU raises.
"""

from . import band
from .band import unwrap_rows
from .irls import unwrap, unwrap_device, unwrap_many
from .objective import (IrlsWeights, arc_count, candidate_step, eval_f, eval_h_delta,
                        update_weights)
from .operators import DiagonalWeights, SystemVector, apply_system, build_rhs
from .params import (BudgetDecision, IrlsParams, IrlsTrace, IterationRecord, ModelParams, UnwrapResult,
                     cg_budget_update, lipschitz_constant, relative_improvement)
from .pcg import NumericalBreakdown, PcgOutcome, pcg_solve
from .phase import (TWO_PI, ErrorReport, GradientField, WeightField, as_phase_grid, center_mean_zero,
                    congruent_round, shift_error, validate_wrapped, wrap_to_principal)
from .preconditioner import apply_preconditioner, neumann_eigenvalues, sylvester_solve
from .synth import SceneSpec, add_phase_noise, config_scene, generate_scene, wrap_scene
from .wrapped import wrapped_gradients

__version__ = "0.1.0"


def release_workspaces():
    """Free the cached per-size device workspaces (single-grid, concurrent and
    row-sharded solvers); the next unwrap of a size plans it again."""
    import gc
    from .band import RowSharded
    from .device import Workspace
    Workspace.release_all()
    RowSharded._cache.clear()
    gc.collect()
