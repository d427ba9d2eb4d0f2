"""Partition API: optimal CG rate, greedy GPU-memory budget, prompt token split.

These decide *where* each hidden column of a layer lives and who runs it --
the inputs of the sliced execution in ``sliced.py``.  All three solvers
restate the reference with identical floating-point expression trees so the
chosen rates and token counts are bit-exact:

* affine edge-point machinery   -- /root/reference/pkg/src/sliceplan/_piecewise.py:13-92
* ``solve_rcg`` and grid oracle -- /root/reference/pkg/src/sliceplan/rate_solver.py:40-166
* ``greedy_assign``             -- /root/reference/pkg/src/sliceplan/memory_assigner.py:37-122
* ``solve_ng``                  -- /root/reference/pkg/src/sliceplan/token_assigner.py:33-148
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .costs import HardwareProfile
from .errors import NonIncreasingStep
from .schedule import (
    SGN_EPS,
    TRANSFER_LITERAL,
    TRANSFER_RATE_SCALED,
    LayerSpec,
    Phase,
    SlicingRates,
    Workload,
    _recurrence_tfin_vec,
    _stage_arrays_generation,
    evaluate_recurrence,
    stage_times_generation,
    stage_times_prompt,
)

#: One-sided probe just past the jump where the CG slice turns on (rate_solver.py:29-30).
EDGE_EPS = 1e-9


# ---------------------------------------------------------------------------
# affine pieces


@dataclass(frozen=True)
class Affine:
    """``a + b * u`` in the decision variable u (a rate or a token count)."""

    a: float
    b: float

    def at(self, u: float) -> float:
        return self.a + self.b * u

    def __add__(self, other: "Affine") -> "Affine":
        return Affine(self.a + other.a, self.b + other.b)

    def scaled(self, k: float) -> "Affine":
        return Affine(k * self.a, k * self.b)


def intersect(p: Affine, q: Affine) -> float | None:
    slope_gap = p.b - q.b
    return None if slope_gap == 0.0 else (q.a - p.a) / slope_gap


def gpu_finish_affine(case: int, t_l: Affine, t_c2g: Affine, t_g: Affine, n_gemms: int) -> Affine:
    """Closed-form GPU-chain finish when the copy (1), kernel (2) or launch (3) paces."""
    n = float(n_gemms)
    if case == 1:
        return t_l + t_c2g.scaled(n) + t_g
    if case == 2:
        return t_l + t_c2g + t_g.scaled(n)
    if case == 3:
        return t_l.scaled(n) + t_c2g + t_g
    raise ValueError(f"case must be 1, 2 or 3, got {case}")


def boundary_roots(
    t_l: Affine, t_c2g: Affine, t_g: Affine, t_c: Affine, n_gemms: int,
    lo: float, hi: float, tol: float = 1e-12,
) -> list[tuple[float, str]]:
    """In-range roots of the six equalities where t_fin can bend, clamped to [lo, hi]."""
    cpu_done = t_c.scaled(float(n_gemms))
    equalities = [("launch=transfer", t_l, t_c2g), ("gpu=transfer", t_g, t_c2g), ("launch=gpu", t_l, t_g)]
    equalities += [
        (f"gpu_finish[case{c}]=cpu_finish", gpu_finish_affine(c, t_l, t_c2g, t_g, n_gemms), cpu_done)
        for c in (1, 2, 3)
    ]
    found: list[tuple[float, str]] = []
    for label, p, q in equalities:
        u = intersect(p, q)
        if u is not None and lo - tol <= u <= hi + tol:
            found.append((min(max(u, lo), hi), label))
    return found


def dedupe_sorted(values: list[float], tol: float = 1e-12) -> list[float]:
    kept: list[float] = []
    for v in sorted(values):
        if not kept or v - kept[-1] > tol:
            kept.append(v)
    return kept


# ---------------------------------------------------------------------------
# CG rate at a fixed GG rate


@dataclass(frozen=True)
class RateSolution:
    rates: SlicingRates
    t_fin: float
    candidates: tuple[tuple[float, float], ...]


def _generation_affines(profile, layer: LayerSpec, workload: Workload, r_gg: float):
    """Stage times as affines in r_CG with both CC and CG live (rate_solver.py:40-55)."""
    units = layer.gemm_units(workload.tokens)
    gemm = profile.gemm_for(layer.precision)
    pcie, launch = profile.require_pcie(), profile.require_launch()
    gg = r_gg if r_gg > SGN_EPS else 0.0
    s_gg = 1.0 if gg > 0.0 else 0.0
    return (
        Affine((2.0 + s_gg) * launch.alpha, 0.0),
        Affine(pcie.alpha, layer.weight_bytes * pcie.beta),
        Affine(gemm.gpu.alpha * (1.0 + s_gg) + gg * units * gemm.gpu.beta, units * gemm.gpu.beta),
        Affine(gemm.cpu.alpha + (1.0 - gg) * units * gemm.cpu.beta, -units * gemm.cpu.beta),
    )


def edge_candidates(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, r_gg: float,
    eps: float = EDGE_EPS,
) -> list[tuple[float, str]]:
    if not 0.0 <= r_gg <= 1.0:
        raise ValueError(f"r_gg must lie in [0, 1], got {r_gg}")
    hi = 1.0 - r_gg
    points: list[tuple[float, str]] = [(0.0, "endpoint"), (hi, "endpoint")]
    if 0.0 < eps < hi:
        points.append((eps, "zero-jump probe"))
    if hi > 0.0:
        points += boundary_roots(*_generation_affines(profile, layer, workload, r_gg),
                                 layer.n_gemms, 0.0, hi)
    return sorted(points, key=lambda p: p[0])


def edge_points(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, r_gg: float,
    eps: float = EDGE_EPS,
) -> list[float]:
    return dedupe_sorted([v for v, _ in edge_candidates(profile, layer, workload, r_gg, eps)])


def _tfin(profile, layer, workload, rates: SlicingRates) -> float:
    return evaluate_recurrence(stage_times_generation(profile, layer, workload, rates), layer.n_gemms).t_fin


def solve_rcg(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, r_gg: float
) -> RateSolution:
    """Best r_CG at fixed r_GG; every edge point is scored by the full recurrence
    and ties keep the smaller r_CG (rate_solver.py:90-117)."""
    scored = [(cg, _tfin(profile, layer, workload, SlicingRates.from_cg(cg, r_gg)))
              for cg in edge_points(profile, layer, workload, r_gg)]
    best_cg, best_t = 0.0, float("inf")
    for cg, t in scored:
        if t < best_t:
            best_cg, best_t = cg, t
    return RateSolution(SlicingRates.from_cg(best_cg, r_gg), best_t, tuple(scored))


def grid_scan(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, r_gg: float, grid_n: int
) -> tuple[np.ndarray, np.ndarray]:
    if grid_n < 2:
        raise ValueError(f"grid_n must be >= 2, got {grid_n}")
    if not 0.0 <= r_gg <= 1.0:
        raise ValueError(f"r_gg must lie in [0, 1], got {r_gg}")
    cg_values = np.linspace(0.0, 1.0 - r_gg, grid_n)
    stages = _stage_arrays_generation(profile, layer, workload, cg_values, r_gg)
    return cg_values, _recurrence_tfin_vec(*stages, layer.n_gemms)


def solve_rates_grid(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, r_gg: float, grid_n: int
) -> RateSolution:
    cg_values, t_fin = grid_scan(profile, layer, workload, r_gg, grid_n)
    rates = SlicingRates.from_cg(float(cg_values[int(np.argmin(t_fin))]), r_gg)
    return RateSolution(
        rates=rates,
        t_fin=_tfin(profile, layer, workload, rates),
        candidates=tuple(zip(cg_values.tolist(), t_fin.tolist())),
    )


def lipschitz_bound(profile: HardwareProfile, layer: LayerSpec, workload: Workload) -> float:
    units = layer.gemm_units(workload.tokens)
    gemm, pcie = profile.gemm_for(layer.precision), profile.require_pcie()
    return layer.n_gemms * (units * (gemm.gpu.beta + gemm.cpu.beta) + layer.weight_bytes * pcie.beta)


# ---------------------------------------------------------------------------
# GPU-memory budget across layers


@dataclass(frozen=True)
class PlanStep:
    iteration: int
    layer_index: int
    rgg: float
    importance: float


@dataclass(frozen=True)
class MemoryPlan:
    per_layer_rgg: tuple[float, ...]
    bytes_used: float
    budget: float
    iterations: int
    trace: tuple[PlanStep, ...]


def importance(
    profile: HardwareProfile, layer: LayerSpec, workload: Workload, v_prev: float, v_i: float
) -> float:
    """Seconds saved per extra resident byte (memory_assigner.py:37-56)."""
    if not (0.0 <= v_prev <= 1.0 and 0.0 <= v_i <= 1.0):
        raise ValueError("resident fractions must lie in [0, 1]")
    if v_i <= v_prev:
        raise NonIncreasingStep(f"v_i must exceed v_prev, got {v_i} <= {v_prev}")
    gain = solve_rcg(profile, layer, workload, v_prev).t_fin - solve_rcg(profile, layer, workload, v_i).t_fin
    return gain / ((v_i - v_prev) * layer.layer_bytes)


def greedy_assign(
    profile: HardwareProfile,
    layers: Sequence[LayerSpec],
    workload: Workload,
    budget: float,
    n_steps: int = 16,
) -> MemoryPlan:
    """Spend ``budget`` bytes on per-layer r_GG in {i/n_steps}, best seconds-per-byte
    first; strict improvement only, ties to the lowest layer then smallest
    fraction (memory_assigner.py:59-122)."""
    if budget < 0.0:
        raise ValueError(f"budget must be >= 0, got {budget}")
    if n_steps < 1:
        raise ValueError(f"n_steps must be >= 1, got {n_steps}")

    memo: dict[tuple, float] = {}

    def tfin_at(layer: LayerSpec, v: float) -> float:
        key = (layer.model_dim, layer.hidden_dim, layer.n_gemms, layer.precision, v)
        if key not in memo:
            memo[key] = solve_rcg(profile, layer, workload, v).t_fin
        return memo[key]

    resident = [0.0] * len(layers)
    used = 0.0
    steps: list[PlanStep] = []
    while True:
        pick: tuple[int, float, float] | None = None
        pick_score = 0.0
        for j, layer in enumerate(layers):
            now = tfin_at(layer, resident[j])
            for i in range(1, n_steps + 1):
                v = i / n_steps
                if v <= resident[j]:
                    continue
                extra = (v - resident[j]) * layer.layer_bytes
                if used + extra > budget:
                    continue
                score = (now - tfin_at(layer, v)) / extra
                if score > pick_score:
                    pick, pick_score = (j, v, extra), score
        if pick is None:
            break
        j, v, extra = pick
        resident[j] = v
        used += extra
        steps.append(PlanStep(iteration=len(steps) + 1, layer_index=j, rgg=v, importance=pick_score))
    return MemoryPlan(tuple(resident), used, budget, len(steps), tuple(steps))


# ---------------------------------------------------------------------------
# prompt-token diversion at frozen rates


@dataclass(frozen=True)
class TokenPlan:
    n_g: int
    t_fin_prompt: float
    baseline_t_fin: float
    candidates: tuple[tuple[int, float], ...]

    @property
    def speedup(self) -> float:
        return 1.0 if self.t_fin_prompt <= 0.0 else self.baseline_t_fin / self.t_fin_prompt


def _prompt_affines(profile, layer: LayerSpec, tokens: int, rates: SlicingRates, transfer_model: str):
    """Interior stage times as affines in n_g (token_assigner.py:47-82)."""
    mh = float(layer.model_dim) * layer.hidden_dim
    gemm = profile.gemm_for(layer.precision)
    pcie, launch = profile.require_pcie(), profile.require_launch()
    cc, cg, gg = (r if r > SGN_EPS else 0.0 for r in (rates.cc, rates.cg, rates.gg))
    s_cc, s_cg, s_gg = (1.0 if r > 0.0 else 0.0 for r in (cc, cg, gg))
    if transfer_model == TRANSFER_LITERAL:
        copy_a = pcie.alpha * (s_cg + s_cc) + layer.weight_bytes * pcie.beta
    elif transfer_model == TRANSFER_RATE_SCALED:
        copy_a = pcie.alpha * (s_cg + s_cc) + (cg + cc) * layer.weight_bytes * pcie.beta
    else:
        raise ValueError(f"unknown transfer_model '{transfer_model}'")
    return (
        Affine((2.0 * s_cg + 2.0 * s_cc + s_gg) * launch.alpha, 0.0),
        Affine(copy_a, 0.0),
        Affine(gemm.gpu.alpha * (s_cg + s_gg + s_cc) + tokens * (cg + gg) * mh * gemm.gpu.beta,
               cc * mh * gemm.gpu.beta),
        Affine(gemm.cpu.alpha * s_cc + tokens * cc * mh * gemm.cpu.beta, -cc * mh * gemm.cpu.beta),
    )


def _integer_candidates(profile, layer, tokens: int, rates, transfer_model: str) -> list[int]:
    picks = {0, tokens, max(tokens - 1, 0)}
    affines = _prompt_affines(profile, layer, tokens, rates, transfer_model)
    for root, _ in boundary_roots(*affines, layer.n_gemms, 0.0, float(tokens)):
        picks.update(int(v) for v in (math.floor(root), math.ceil(root)) if 0 <= v <= tokens)
    return sorted(picks)


def solve_ng(
    profile: HardwareProfile,
    layer: LayerSpec,
    tokens: int,
    rates: SlicingRates,
    transfer_model: str = TRANSFER_LITERAL,
) -> TokenPlan:
    """Best number of prompt tokens to run on the GPU against the CC columns;
    ties to the smaller count (token_assigner.py:104-137)."""
    workload = Workload(tokens=tokens, phase=Phase.PROMPT)
    scored: list[tuple[int, float]] = []
    for ng in _integer_candidates(profile, layer, tokens, rates, transfer_model):
        stage = stage_times_prompt(profile, layer, workload, rates, ng, transfer_model)
        scored.append((ng, evaluate_recurrence(stage, layer.n_gemms).t_fin))
    best_ng, best_t = 0, float("inf")
    for ng, t in scored:
        if t < best_t:
            best_ng, best_t = ng, t
    baseline = dict(scored)[0]
    return TokenPlan(n_g=best_ng, t_fin_prompt=best_t, baseline_t_fin=baseline, candidates=tuple(scored))


@dataclass(frozen=True)
class LayerTokenPlan:
    n_g: tuple[int, ...]       # per expert of the layer
    link_s: float              # modelled host-link time of the layer
    cpu_s: float               # modelled host CC time of the layer


def _prompt_call_costs(profile: HardwareProfile, layer: LayerSpec, rates: SlicingRates, chunk_bytes: float):
    """(link(T_e, n_g), cpu(T_e, n_g)) seconds of one expert call in the prompt
    phase: the linear model solve_ng_layer plans with (docstring there)."""
    gemm, pcie = profile.gemm[layer.precision], profile.require_pcie()
    G = float(layer.n_gemms)
    W = float(layer.weight_bytes)
    mh = float(layer.model_dim) * layer.hidden_dim
    cc, cg = rates.cc, rates.cg

    def link(t: int, ng: int) -> float:
        nbytes = (cg + (cc if ng > 0 else 0.0)) * G * W
        return pcie.alpha * math.ceil(nbytes / chunk_bytes) + nbytes * pcie.beta if nbytes > 0 else 0.0

    def cpu(t: int, ng: int) -> float:
        kept = t - ng
        return G * (gemm.cpu.alpha + kept * cc * mh * gemm.cpu.beta) if kept > 0 and cc > 0 else 0.0

    return link, cpu


def prompt_layer_busy(
    profile: HardwareProfile, layer: LayerSpec, tokens: Sequence[int], n_g: Sequence[int], rates: SlicingRates,
    chunk_bytes: float = 8 << 20,
) -> tuple[float, float]:
    """EXTENSION: predicted (link busy, host CC busy) seconds of one MoE layer's
    prompt calls with the given per-expert splits -- any plan's, solve_ng's or
    solve_ng_layer's -- under solve_ng_layer's cost model.  Used to re-anchor
    the prompt profile on a box from a traced prefill."""
    link, cpu = _prompt_call_costs(profile, layer, rates, chunk_bytes)
    return (sum(link(int(t), int(n)) for t, n in zip(tokens, n_g)),
            sum(cpu(int(t), int(n)) for t, n in zip(tokens, n_g)))


def solve_ng_layer(
    profile: HardwareProfile, layer: LayerSpec, tokens: Sequence[int], rates: SlicingRates,
    chunk_bytes: float = 8 << 20,
) -> LayerTokenPlan:
    """EXTENSION (not in the reference): token split of a whole MoE layer.

    ``solve_ng`` (token_assigner.py:104-137, bit-exact above) plans one expert
    as if it had the host link and the host cores to itself.  The experts of
    a layer share both, and the runtime streams an expert's CC chunks only
    when some of its rows run on the GPU (n_g > 0).  Per expert this takes
    n_g in {T_e (every row on the GPU: CC chunks streamed, host idle),
    0 (every row on the host: only CG streamed)} and greedily moves experts to
    the host side while the layer's max(link, host) time drops:
        link_e = alpha_P * chunks + (cg + cc * [n_g > 0]) * G * W * beta_P
        cpu_e  = G * (alpha_C + (T_e - n_g) * cc * M * H * beta_C)
    (G GEMMs per expert = layer.n_gemms, W = layer.weight_bytes).  Ties go to
    the lower expert index; deterministic."""
    link, cpu = _prompt_call_costs(profile, layer, rates, chunk_bytes)
    ng = [int(t) for t in tokens]  # start: every row on the GPU

    def layer_time(plan):
        lk = sum(link(t, n) for t, n in zip(tokens, plan))
        cp = sum(cpu(t, n) for t, n in zip(tokens, plan))
        return max(lk, cp), lk, cp

    best, _, _ = layer_time(ng)
    while True:
        move, move_t = None, best
        for e, t in enumerate(tokens):
            if ng[e] == 0 or t == 0:
                continue
            trial = list(ng)
            trial[e] = 0
            tt, _, _ = layer_time(trial)
            if tt < move_t:
                move, move_t = e, tt
        if move is None:
            break
        ng[move] = 0
        best = move_t
    _, lk, cp = layer_time(ng)
    return LayerTokenPlan(n_g=tuple(ng), link_s=lk, cpu_s=cp)


def prompt_speedup(
    profile: HardwareProfile, layer: LayerSpec, tokens: int, rates: SlicingRates,
    transfer_model: str = TRANSFER_LITERAL,
) -> float:
    return solve_ng(profile, layer, tokens, rates, transfer_model).speedup
