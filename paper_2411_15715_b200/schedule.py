"""Stage-time model and four-stream completion recurrence of one sliced layer.

A layer runs ``n_gemms`` GEMMs through four serial resources: CPU compute
(Stream-A), kernel launch (Stream-B), host-to-device copy (Stream-C) and GPU
compute (Stream-D).  This module restates
/root/reference/pkg/src/sliceplan/pipeline.py term for term -- the planner's
answers must be bit-identical -- and is the *predicted* side of the measured
timelines the runtime emits in the same Gantt schema (``timeline_records``).
"""

from __future__ import annotations

import enum
import heapq
from dataclasses import dataclass

import numpy as np

from .costs import HardwareProfile, Precision
from .errors import TokenCountOutOfRange

#: Rates at or below this are exactly zero: empty slices pay no startup (pipeline.py:22-24).
SGN_EPS = 1e-12
#: Recurrence / simulator agreement bound (pipeline.py:26-27).
TFIN_EQUIV_TOL = 1e-12

TRANSFER_LITERAL = "literal"
TRANSFER_RATE_SCALED = "rate_scaled"
_TRANSFER_MODELS = (TRANSFER_LITERAL, TRANSFER_RATE_SCALED)


class Phase(enum.Enum):
    PROMPT = "prompt"
    GENERATION = "generation"


class CaseLabel(enum.Enum):
    CASE1 = "case1"  # copy-paced GPU chain
    CASE2 = "case2"  # GPU-kernel-paced
    CASE3 = "case3"  # launch-paced
    CPU_BOUND = "cpu_bound"
    DEGENERATE = "degenerate"


@dataclass(frozen=True)
class LayerSpec:
    """Shape of one layer's sliced GEMMs (pipeline.py:47-72).

    For a MoE decode step ``n_gemms`` = top_k * G (G = 2 plain MLP, 3 SwiGLU),
    the reference's own modelling convention.
    """

    model_dim: int
    hidden_dim: int
    n_gemms: int
    precision: Precision

    def __post_init__(self) -> None:
        if min(self.model_dim, self.hidden_dim, self.n_gemms) < 1:
            raise ValueError("model_dim, hidden_dim and n_gemms must all be >= 1")

    @property
    def weight_bytes(self) -> float:
        return self.model_dim * self.hidden_dim * self.precision.bytes_per_param

    @property
    def layer_bytes(self) -> float:
        return self.n_gemms * self.weight_bytes

    def gemm_units(self, tokens: int) -> float:
        return float(tokens) * self.model_dim * self.hidden_dim


@dataclass(frozen=True)
class Workload:
    tokens: int
    phase: Phase

    def __post_init__(self) -> None:
        if self.tokens < 1:
            raise ValueError(f"tokens must be >= 1, got {self.tokens}")


@dataclass(frozen=True)
class SlicingRates:
    """Column fractions (CPU-resident/CPU-run, CPU-resident/GPU-run, GPU-resident).

    Tiny negatives (>= -1e-12) snap to zero and the sum must be 1 within 1e-12
    (pipeline.py:85-105).
    """

    cc: float
    cg: float
    gg: float

    def __post_init__(self) -> None:
        for name in ("cc", "cg", "gg"):
            value = getattr(self, name)
            if value < 0.0:
                if value < -SGN_EPS:
                    raise ValueError(f"rate {name} must be >= 0, got {value}")
                object.__setattr__(self, name, 0.0)
        total = self.cc + self.cg + self.gg
        if abs(total - 1.0) > SGN_EPS:
            raise ValueError(f"rates must sum to 1 within {SGN_EPS}, got {total}")

    @classmethod
    def from_cg(cls, cg: float, gg: float) -> "SlicingRates":
        return cls(cc=1.0 - cg - gg, cg=cg, gg=gg)


@dataclass(frozen=True)
class StageTimes:
    launch_s: float
    transfer_s: float
    gpu_s: float
    cpu_s: float

    def __post_init__(self) -> None:
        for name in ("launch_s", "transfer_s", "gpu_s", "cpu_s"):
            if getattr(self, name) < 0.0:
                raise ValueError(f"{name} must be >= 0")


@dataclass(frozen=True)
class Timeline:
    """Per-stream completion stamps; index 0 is the origin."""

    launch_done: np.ndarray
    transfer_done: np.ndarray
    gpu_done: np.ndarray
    cpu_done: np.ndarray
    t_fin: float
    case_label: CaseLabel


def _on(x: float) -> float:
    return 1.0 if x > SGN_EPS else 0.0


def _live(x: float) -> float:
    return x if x > SGN_EPS else 0.0


def _coeffs(profile: HardwareProfile, layer: LayerSpec):
    return profile.gemm_for(layer.precision), profile.require_pcie(), profile.require_launch()


def stage_times_generation(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, rates: SlicingRates
) -> StageTimes:
    """Decode stage times (Eq. 1-4; pipeline.py:143-167)."""
    units = layer.gemm_units(workload.tokens)
    gemm, pcie, launch = _coeffs(profile, layer)
    cc, cg, gg = _live(rates.cc), _live(rates.cg), _live(rates.gg)
    s_cc, s_cg, s_gg = _on(cc), _on(cg), _on(gg)
    return StageTimes(
        launch_s=(2.0 * s_cg + s_gg) * launch.alpha,
        transfer_s=s_cg * (pcie.alpha + cg * layer.weight_bytes * pcie.beta),
        gpu_s=gemm.gpu.alpha * (s_cg + s_gg) + (cg + gg) * units * gemm.gpu.beta,
        cpu_s=gemm.cpu.alpha * s_cc + cc * units * gemm.cpu.beta,
    )


def stage_times_prompt(
    profile: HardwareProfile,
    layer: LayerSpec,
    workload: Workload,
    rates: SlicingRates,
    n_g: int,
    transfer_model: str = TRANSFER_LITERAL,
) -> StageTimes:
    """Prompt stage times with ``n_g`` tokens diverted to the GPU (pipeline.py:170-212)."""
    if workload.phase is not Phase.PROMPT:
        raise ValueError("stage_times_prompt requires a prompt-phase workload")
    if transfer_model not in _TRANSFER_MODELS:
        raise ValueError(f"transfer_model must be one of {_TRANSFER_MODELS}")
    tokens = workload.tokens
    if n_g < 0 or n_g > tokens:
        raise TokenCountOutOfRange(f"n_g must lie in [0, {tokens}], got {n_g}")

    mh = float(layer.model_dim) * layer.hidden_dim
    gemm, pcie, launch = _coeffs(profile, layer)
    cc, cg, gg = _live(rates.cc), _live(rates.cg), _live(rates.gg)
    s_cc, s_cg, s_gg = _on(cc), _on(cg), _on(gg)

    if transfer_model == TRANSFER_LITERAL:
        copy_s = pcie.alpha * (s_cg + s_cc) + layer.weight_bytes * pcie.beta
    else:
        copy_s = pcie.alpha * (s_cg + s_cc) + (cg + cc) * layer.weight_bytes * pcie.beta
    kept = tokens - n_g
    return StageTimes(
        launch_s=(2.0 * s_cg + 2.0 * s_cc + s_gg) * launch.alpha,
        transfer_s=copy_s,
        gpu_s=gemm.gpu.alpha * (s_cg + s_gg + s_cc)
        + (tokens * (cg + gg) + n_g * cc) * mh * gemm.gpu.beta,
        cpu_s=gemm.cpu.alpha * _on(cc * kept) + kept * cc * mh * gemm.cpu.beta,
    )


def classify_case(stage: StageTimes) -> CaseLabel:
    """Which stage paces the GPU chain; ties fall to the later case (pipeline.py:215-226)."""
    t_l, t_c2g, t_g = stage.launch_s, stage.transfer_s, stage.gpu_s
    copy_beats_launch = t_l < t_c2g
    if copy_beats_launch and t_g < t_c2g:
        return CaseLabel.CASE1
    if copy_beats_launch or t_l < t_g:
        return CaseLabel.CASE2
    return CaseLabel.CASE3


def _label(stage: StageTimes, gpu_final: float, cpu_final: float) -> CaseLabel:
    if stage.launch_s == 0.0 and stage.transfer_s == 0.0 and stage.gpu_s == 0.0:
        return CaseLabel.DEGENERATE
    if cpu_final > gpu_final:
        return CaseLabel.CPU_BOUND
    return classify_case(stage)


def _timeline(stamps: list[list[float]], stage: StageTimes) -> Timeline:
    arrays = [np.array(s, dtype=float) for s in stamps]
    gpu_final, cpu_final = float(arrays[2][-1]), float(arrays[3][-1])
    return Timeline(
        launch_done=arrays[0],
        transfer_done=arrays[1],
        gpu_done=arrays[2],
        cpu_done=arrays[3],
        t_fin=max(gpu_final, cpu_final),
        case_label=_label(stage, gpu_final, cpu_final),
    )


def evaluate_recurrence(stage: StageTimes, n_gemms: int) -> Timeline:
    """Eq. 5: launch -> copy -> kernel chain plus the independent CPU chain."""
    if n_gemms < 1:
        raise ValueError(f"n_gemms must be >= 1, got {n_gemms}")
    t_l, t_c2g, t_g, t_c = stage.launch_s, stage.transfer_s, stage.gpu_s, stage.cpu_s
    lau, cpy, gpu, cpu = [0.0], [0.0], [0.0], [0.0]
    for _ in range(n_gemms):
        lau.append(lau[-1] + t_l)
        cpy.append(max(lau[-1], cpy[-1]) + t_c2g)
        gpu.append(max(cpy[-1], gpu[-1]) + t_g)
        cpu.append(cpu[-1] + t_c)
    return _timeline([lau, cpy, gpu, cpu], stage)


STREAM_NAMES = ("launch", "transfer", "gpu", "cpu")
_LAUNCH, _COPY, _KERNEL, _CPU = range(4)
# Upstream dependencies inside one GEMM: the copy and the kernel wait for the
# launch, the kernel also waits for the copy (pipeline.py:268-283).
_NEEDS = {_LAUNCH: (), _COPY: (_LAUNCH,), _KERNEL: (_LAUNCH, _COPY), _CPU: ()}


def simulate_streams(stage: StageTimes, n_gemms: int) -> Timeline:
    """Discrete-event run of the four FIFO streams; an independent check of
    ``evaluate_recurrence``.

    Each stream executes its GEMM tasks in order.  A task is dispatched when
    its stream is idle and every upstream task of the same GEMM has finished;
    events are processed in time order off a heap.
    """
    if n_gemms < 1:
        raise ValueError(f"n_gemms must be >= 1, got {n_gemms}")
    dur = (stage.launch_s, stage.transfer_s, stage.gpu_s, stage.cpu_s)
    finished = [[None] * n_gemms for _ in range(4)]  # finish stamp per (stream, gemm)
    head = [0, 0, 0, 0]  # next GEMM index each stream will run
    idle_at = [0.0, 0.0, 0.0, 0.0]
    running = [False] * 4
    events: list[tuple[float, int, int, int]] = []  # (time, seq, stream, gemm)
    seq = 0

    def dispatch(s: int) -> None:
        nonlocal seq
        i = head[s]
        if running[s] or i >= n_gemms:
            return
        upstream = [finished[u][i] for u in _NEEDS[s]]
        if any(f is None for f in upstream):
            return
        start = max([idle_at[s]] + upstream)
        end = start + dur[s]
        running[s] = True
        head[s] += 1
        idle_at[s] = end
        heapq.heappush(events, (end, seq, s, i))
        seq += 1

    for s in range(4):
        dispatch(s)
    while events:
        end, _, s, i = heapq.heappop(events)
        finished[s][i] = end
        running[s] = False
        for t in range(4):
            dispatch(t)

    stamps = [[0.0] + [float(v) for v in finished[s]] for s in range(4)]
    return _timeline(stamps, stage)


def timeline_records(stage: StageTimes, timeline: Timeline) -> list[dict]:
    """Gantt rows ``{gemm_index (1-based), stream, start_s, end_s}``, stream-major."""
    dur = (stage.launch_s, stage.transfer_s, stage.gpu_s, stage.cpu_s)
    stamps = (timeline.launch_done, timeline.transfer_done, timeline.gpu_done, timeline.cpu_done)
    n = len(timeline.launch_done) - 1
    return [
        {"gemm_index": i, "stream": STREAM_NAMES[s], "start_s": float(stamps[s][i]) - dur[s],
         "end_s": float(stamps[s][i])}
        for s in range(4)
        for i in range(1, n + 1)
    ]


def cc_result_transfer_time(
    profile: HardwareProfile,
    layer: LayerSpec,
    workload: Workload,
    rates: SlicingRates,
    bytes_per_activation: float = 2.0,
) -> float:
    """Y_cc host-to-device copy after the pipeline drains; excluded from t_fin
    (pipeline.py:367-383).  The runtime measures the real copy separately."""
    if _on(rates.cc) == 0.0:
        return 0.0
    pcie = profile.require_pcie()
    return pcie.alpha + workload.tokens * layer.model_dim * bytes_per_activation * pcie.beta


# ---------------------------------------------------------------------------
# Vectorised twins for grid oracles; same expression trees as the scalar forms
# so both round identically (pipeline.py:391-461).


def _recurrence_tfin_vec(t_l, t_c2g, t_g, t_c, n_gemms: int) -> np.ndarray:
    lau = np.zeros_like(t_l)
    cpy = np.zeros_like(t_l)
    gpu = np.zeros_like(t_l)
    for _ in range(n_gemms):
        lau = lau + t_l
        cpy = np.maximum(lau, cpy) + t_c2g
        gpu = np.maximum(cpy, gpu) + t_g
    return np.maximum(gpu, n_gemms * t_c)


def _stage_arrays_generation(profile, layer, workload, cg_values: np.ndarray, r_gg: float):
    units = layer.gemm_units(workload.tokens)
    gemm, pcie, launch = _coeffs(profile, layer)
    gg = _live(r_gg)
    s_gg = _on(gg)
    cc_values = 1.0 - cg_values - r_gg
    cg = np.where(cg_values > SGN_EPS, cg_values, 0.0)
    cc = np.where(cc_values > SGN_EPS, cc_values, 0.0)
    s_cg = np.where(cg > SGN_EPS, 1.0, 0.0)
    s_cc = np.where(cc > SGN_EPS, 1.0, 0.0)
    launch_t = (2.0 * s_cg + s_gg) * launch.alpha
    transfer = s_cg * (pcie.alpha + cg * layer.weight_bytes * pcie.beta)
    gpu = gemm.gpu.alpha * (s_cg + s_gg) + (cg + gg) * units * gemm.gpu.beta
    cpu = gemm.cpu.alpha * s_cc + cc * units * gemm.cpu.beta
    return launch_t, transfer, gpu, cpu


def _stage_arrays_prompt(
    profile, layer, workload, rates: SlicingRates, ng_values: np.ndarray,
    transfer_model: str = TRANSFER_LITERAL,
):
    tokens = workload.tokens
    mh = float(layer.model_dim) * layer.hidden_dim
    gemm, pcie, launch = _coeffs(profile, layer)
    cc, cg, gg = _live(rates.cc), _live(rates.cg), _live(rates.gg)
    s_cc, s_cg, s_gg = _on(cc), _on(cg), _on(gg)
    ones = np.ones_like(ng_values, dtype=float)
    launch_t = ((2.0 * s_cg + 2.0 * s_cc + s_gg) * launch.alpha) * ones
    if transfer_model == TRANSFER_LITERAL:
        transfer = (pcie.alpha * (s_cg + s_cc) + layer.weight_bytes * pcie.beta) * ones
    else:
        transfer = (pcie.alpha * (s_cg + s_cc) + (cg + cc) * layer.weight_bytes * pcie.beta) * ones
    gpu = gemm.gpu.alpha * (s_cg + s_gg + s_cc) + (
        tokens * (cg + gg) + ng_values * cc
    ) * mh * gemm.gpu.beta
    s_cpu = np.where(cc * (tokens - ng_values) > SGN_EPS, 1.0, 0.0)
    cpu = gemm.cpu.alpha * s_cpu + (tokens - ng_values) * cc * mh * gemm.cpu.beta
    return launch_t, transfer, gpu, cpu
