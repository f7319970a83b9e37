"""B200-native PipeOffload runtime: the ``ppoff`` planner API plus a measured executor.

Planner names are those of the reference package's public surface
(``pkg/src/ppoff/__init__.py:3-65``), re-implemented here; ``execute`` (``runner.py``,
``simulate``'s signature) replaces the reference's ``simulate`` as the pipeline runner
and returns a ``SimTrace`` of CUDA-measured times (``runner(**opts)`` binds it into a
``simulate``-compatible callable).  The CUDA side lives in the
in-tree C-ABI library ``libppo_b200.so`` (``include/ppo_b200.h``).
"""

from .costs import (
    HardwareSpec,
    ModelSpec,
    PassCosts,
    activation_bytes_per_layer,
    compute_k,
    estimate_pass_costs,
    layer_output_ratio,
    measured_pass_costs,
    offload_round_trip,
)
from .ir import (
    BuildingBlock,
    InfeasibleIntervalError,
    MemoryTimeline,
    Pass,
    PassKind,
    Schedule,
    ScheduleError,
    Violation,
    emit_schedule,
    interleave_compose,
    lifespan,
    memory_timeline,
    parse_schedule,
    stage_contribution_at_peak,
    uniform_repeat,
    validate,
)
from .builders import (
    BUILDERS,
    build_1f1b,
    build_1f1b_full_offload,
    build_gis,
    build_gis_g,
    build_gis_h,
    build_interleaved_1f1b,
    build_po,
    extract_block,
    po_block,
)
from .offload import (
    HostBufferLayout,
    NodeAssignment,
    OffloadPlan,
    Transfer,
    apply_topology_sync,
    assign_ranks_to_nodes,
    pack_host_bins,
    plan_slots,
    select_offload_stages,
)
from .sim import (
    ContentionModel,
    DeadlockError,
    SimTrace,
    bubble_time,
    host_peak_memory,
    peak_memory,
    simulate,
)
from .runner import MeasuredTrace, config_from_spec, execute, runner

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
