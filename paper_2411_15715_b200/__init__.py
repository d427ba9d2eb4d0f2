"""B200-native sliced-weight FFN / MoE-expert execution (ScheInfer, arXiv 2411.15715).

Drop-in for the reference package ``sliceplan`` on its hot path: the same
partition API (slicing rates, the edge-point rate solver, the greedy GPU-memory
assignment, the prompt token split and the four-stream cost model) and the
same operator API (``slice_weights`` / ``mlp_forward_sliced`` /
``execution_tags``), with the forward executed by libsliced on a B200:

* GG block   -- HBM-resident weights, sm_100a GEMV / GEMM kernels
* CG block   -- pinned host weights streamed through a 3-slot HBM ring on a
                copy stream, consumed chunk by chunk on the compute stream
* CC block   -- pinned host weights computed on host threads (AVX-512)
* merge      -- one kernel sums the partials, applies the MoE gates, casts

Import names mirror /root/reference/pkg/src/sliceplan/__init__.py:11-73.
"""

from .costs import (
    GemmCoeffs,
    HardwareProfile,
    OpClass,
    PerfCoeffs,
    Precision,
    ProfileSample,
    fit_launch,
    fit_linear,
    fit_profile,
    generate_samples,
    load_profile,
    predict,
    profile_from_dict,
    profile_to_dict,
    read_samples_csv,
    save_profile,
    write_samples_csv,
)
from .errors import (
    DegenerateSamples,
    EmptySamples,
    MixedOpClass,
    NativeError,
    NonIncreasingStep,
    SchemaViolation,
    ShapeMismatch,
    TokenCountOutOfRange,
)
from .planner import (
    MemoryPlan,
    PlanStep,
    RateSolution,
    TokenPlan,
    edge_points,
    greedy_assign,
    grid_scan,
    importance,
    lipschitz_bound,
    prompt_speedup,
    solve_ng,
    solve_ng_layer,
    prompt_layer_busy,
    solve_rates_grid,
    solve_rcg,
)
from .schedule import (
    CaseLabel,
    LayerSpec,
    Phase,
    SlicingRates,
    StageTimes,
    Timeline,
    Workload,
    cc_result_transfer_time,
    classify_case,
    evaluate_recurrence,
    simulate_streams,
    stage_times_generation,
    stage_times_prompt,
    timeline_records,
)
from .sliced import (
    Activation,
    ExecutorTask,
    SlicedFFN,
    SlicedMoE,
    SlicedWeights,
    execution_tags,
    max_recombination_error,
    mlp_forward_reference,
    mlp_forward_sliced,
    slice_weights,
)
from .store import load_mixtral_moe, load_safetensors, load_store, save_safetensors, save_store

__version__ = "0.1.0"
