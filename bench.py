#!/usr/bin/env python
"""Sliced-weight MoE FFN decode on B200 -- the BASELINE.json headline metric.

Default workload (BASELINE.json configs[1]): one Mixtral-8x7B MoE FFN layer
(model 4096, ffn 14336, 8 SwiGLU experts, top-2, bf16), decode, batch 1 token
per step per GPU, slicing rates chosen by the partition API on the re-fitted
B200 profile (profiles/b200_decode.json) under an explicit GPU byte budget
(default: half of every expert resident in HBM, the paper's limited-memory
regime).  A step = route the token(s), run every active expert's GG block
(HBM), stream its CG block over PCIe through the HBM ring, compute its CC block
on the host threads, merge (and all-reduce over ranks when N > 1).

``--config cfg1``: BASELINE configs[0] shapes (1024/3584, fp32, fixed rates
0.2/0.3/0.5) through the same runtime.

Keys of the JSON line (rank 0):
  value    tokens/s with x resident in HBM (SP_IO_DEVICE), CUDA events, max over ranks
  e2e      tokens/s through the public API with host x / y (SP_IO_HOST)
  roofline GG ffn_block launch (dominant HBM kernel) achieved GB/s vs MEASURED_PEAKS
  link     CG copy GB/s vs the measured link, and the step roofline
           t_roof = max(GG bytes / HBM, CG bytes / link) / measured step
           (north-star definition), plus the bound that includes the host:
           max(t_roof, CC bytes / fitted in-situ CC rate)
  cpu_baseline  the reference algorithm (oracle/sliced_forward.py, fp64 numpy,
           slicing_kernel.py:97-124) on the host cores, bounded sample

``--impl reference`` times that CPU reference alone on the same config.
Multi-GPU (torchrun): experts are sharded round-robin (expert_parallel.py),
one NCCL all-reduce per step; global batch = batch * world (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

UNIT = "tokens/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "model"])
    ap.add_argument("--moe", default="8x22b", choices=["phimoe", "8x22b"], help="cfg5 model")
    ap.add_argument("--layers", type=int, default=32, help="cfg3: layers per forward")
    ap.add_argument("--distinct-layers", type=int, default=8, help="cfg3: distinct weight sets cycled over the layers")
    ap.add_argument("--prompt", type=int, default=512, help="cfg3: prompt tokens")
    ap.add_argument("--decode-steps", type=int, default=128, help="cfg3: decode tokens after the prompt")
    ap.add_argument("--transfer-model", default="rate_scaled", choices=["literal", "rate_scaled"],
                    help="cfg3: solve_ng's prompt transfer model (pipeline.py:204-207).  rate_scaled charges the "
                         "(cg + cc) share of the weights -- exactly what the CG streamer moves when n_g > 0 (CG "
                         "chunks + the CC chunks for the diverted rows); literal charges the whole layer")
    ap.add_argument("--token-plan", default="solve_ng", choices=["solve_ng", "layer"],
                    help="cfg3: per-expert solve_ng (the reference's token assigner, default) or the layer-level "
                         "extension planner.solve_ng_layer (experts share the link and the host)")
    ap.add_argument("--ng-frac", type=float, default=-1.0,
                    help="cfg3 study only: n_g = round(frac * T_e) instead of solve_ng (landscape sweeps)")
    ap.add_argument("--prompt-profile", default="",
                    help="prompt-phase profile (default: profiles/b200_prompt.json, host CC sampled at 32 tokens, "
                         "for solve_ng; profiles/b200_prompt_t128.json, sampled at an expert's 128-token share, "
                         "for --token-plan layer)")
    ap.add_argument("--batch", type=int, default=1, help="decode tokens per step per GPU")
    ap.add_argument("--budget-frac", type=float, default=0.5,
                    help="GPU budget as a fraction of each expert's bytes (planner units)")
    ap.add_argument("--force-cc", type=float, default=-1.0,
                    help="probe only: override the planner's r_CC (r_CG = 1 - r_GG - r_CC); the line says so")
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--top-k", type=int, default=2)
    ap.add_argument("--profile", default=str(ROOT / "profiles" / "b200_decode.json"))
    ap.add_argument("--cpu-sample-steps", type=int, default=20, help="cpu_baseline: at least this many steps")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0, help="cpu_baseline: and at least this much CPU work")
    ap.add_argument("--dry-run", action="store_true",
                    help="spawn / rendezvous / barrier only (CPU test of the multi-rank launch path)")
    ap.add_argument("--trace-out", default="")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--calibrate", type=int, default=1,
                    help="rescale the profile's host CPU / link terms from traced steps on this box and re-solve")
    ap.add_argument("--calib-steps", type=int, default=16)
    ap.add_argument("--calib-rounds", type=int, default=1,
                    help="calibrate -> re-solve -> re-slice rounds; stops early once r_CC moves < --calib-tol")
    ap.add_argument("--calib-tol", type=float, default=0.005)
    args = ap.parse_args(argv)
    if args.config == "cfg1":
        args.model_dim, args.hidden_dim, args.dtype = 1024, 3584, "f32"
    elif args.config == "cfg4":  # LLaMA-2-70B dense FFN, column-sharded over the ranks
        args.model_dim, args.hidden_dim, args.dtype, args.experts, args.top_k = 8192, 28672, "bf16", 1, 1
    elif args.config == "cfg5":  # PhiMoE 16x(4096/6400) or Mixtral-8x22B 8x(6144/16384), top-2
        args.dtype = "bf16"
        args.model_dim, args.hidden_dim, args.experts = (4096, 6400, 16) if args.moe == "phimoe" else (6144, 16384, 8)
    else:
        args.model_dim, args.hidden_dim, args.dtype = 4096, 14336, "bf16"
    if args.config == "cfg3" and args.steps == 100:
        args.steps = 2  # prefill repetitions
    if args.config == "model" and args.steps == 100:
        args.steps = 16  # decoded tokens
    return args


def metric_name(args):
    if args.config == "model":
        return (f"decode tokens/s, {args.layers}-layer Mixtral-8x7B-shaped decoder (attention + KV cache in torch, "
                "sliced MoE FFN per layer), batch 1")
    if args.config == "cfg4":
        return "decode tokens/s, LLaMA-2-70B dense FFN layer (8192/28672) bf16, column-sharded, sliced CC/CG/GG"
    if args.config == "cfg5":
        name = "PhiMoE 16x(4096/6400)" if args.moe == "phimoe" else "Mixtral-8x22B 8x(6144/16384)"
        return f"decode tokens/s, {name} MoE FFN layer top-2, expert-parallel, batch {args.batch}/GPU"
    if args.config == "cfg3":
        plan = "n_g from solve_ng" if args.token_plan == "solve_ng" else "per-layer token plan"
        return (f"prefill tokens/s, Mixtral-8x7B {args.layers}-layer MoE FFN stack, {args.prompt}-token prompt "
                f"with the token-assignment split ({plan}), then {args.decode_steps} decode steps")
    if args.config == "cfg1":
        return "decode tokens/s, MoE FFN layer 1024/3584 (8 experts top-2) fp32, fixed CC/CG/GG 0.2/0.3/0.5"
    return "decode tokens/s, Mixtral-8x7B MoE FFN layer (4096/14336, 8 experts top-2), sliced CC/CG/GG"


# ---------------------------------------------------------------------------
# planning


# Host threads the committed profiles were measured with (the 1-GPU pool box:
# 16 vCPUs, all of them running the CC block).
PROFILE_HOST_THREADS = 16


def rank_host_threads() -> int:
    return int(os.environ.get("SP_HOST_THREADS", "0") or 0) or (os.cpu_count() or PROFILE_HOST_THREADS)


def prompt_profile_path(args):
    """--prompt-profile, else the fitted prompt profile the token plan uses
    (128-token fit for the per-layer plan, 32-token fit for solve_ng)."""
    if args.prompt_profile:
        return args.prompt_profile
    return str(ROOT / "profiles" / ("b200_prompt_t128.json" if args.token_plan == "layer" else "b200_prompt.json"))


def load_profile(path):
    """The fitted profile; with fewer host threads per rank than it was measured
    with (one process per GPU sharing the host), the CPU terms are scaled by
    the thread ratio -- the CC block runs on this rank's share of the cores."""
    from paper_2411_15715_b200 import costs
    from paper_2411_15715_b200.b200_profile import FALLBACK_DECODE

    p = Path(path) if path else None
    if p is not None and p.is_file():
        prof, src = costs.load_profile(p), str(p.relative_to(ROOT) if p.is_relative_to(ROOT) else p)
    else:
        prof, src = costs.profile_from_dict(FALLBACK_DECODE), "fallback (b200_profile.FALLBACK_DECODE)"
    threads = rank_host_threads()
    if threads < PROFILE_HOST_THREADS:
        doc = costs.profile_to_dict(prof)
        k = PROFILE_HOST_THREADS / threads
        for g in doc.get("gemm", {}).values():
            if "cpu" in g:
                g["cpu"]["alpha"] *= k
                g["cpu"]["beta"] *= k
        prof = costs.profile_from_dict(doc)
        src += f" (CPU terms x{k:g}: {threads} host threads per rank)"
    return prof, src


def sp_precision_fp16():
    from paper_2411_15715_b200.costs import Precision

    return Precision.FP16


def decode_profile_for(path, t_expert: int) -> str:
    """The decode profile measured closest below the per-expert token count
    (b200_decode_t<T>.json from ``b200_profile --tokens T``; T = 1 is the
    default file): the cost model is linear in T, the kernels are not."""
    p = Path(path)
    best = p
    for t in (2, 4, 8):
        q = p.with_name(f"{p.stem}_t{t}{p.suffix}")
        if t <= t_expert and q.exists():
            best = q
    return str(best)


def expected_active(experts: int, top_k: int, batch: int) -> float:
    """Expected distinct experts a batch of `batch` tokens touches with uniform top-k routing."""
    return experts * (1.0 - (1.0 - top_k / experts) ** batch)


def plan_rates(args, tokens_per_step):
    """greedy_assign under the budget picks r_GG, solve_rcg the best r_CG
    (config 1 uses the fixed rates of BASELINE.json configs[0]).

    MoE decode is modelled the reference's way, n_gemms = active experts x 3
    (PAPER.md:157), with the expected number of experts a batch activates and
    the tokens each of them sees (hard part 6).  Under
    expert parallelism (WORLD_SIZE > 1) every rank routes the global batch and
    plans for the experts it owns."""
    import math

    import paper_2411_15715_b200 as sp

    hidden = getattr(args, "shard_hidden", args.hidden_dim)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.experts > 1:
        # every rank routes the global batch; a rank runs only its own experts
        t_glob = tokens_per_step * world
        e_act = min(expected_active(args.experts, args.top_k, t_glob), args.experts)
        e_loc = args.experts / world * (1.0 - (1.0 - args.top_k / args.experts) ** t_glob)
        n_gemms = max(1, round(e_loc)) * 3
        t_expert = max(1, math.ceil(t_glob * args.top_k / max(e_act, 1.0)))
    else:
        n_gemms, t_expert = 3, max(1, tokens_per_step)
    profile, source = load_profile(decode_profile_for(args.profile, t_expert))
    # The reference's Precision has 2-byte and 4-bit weights only (perf_model.py:45-51).
    # fp32 weights (cfg1) are modelled as a twice-as-wide 2-byte layer: every term of
    # the decode model is bytes-bound (weight stream, CC rows, CG copies), so twice
    # the bytes per GEMM is twice the units at the same per-unit rates.
    layer = sp.LayerSpec(args.model_dim, hidden * (2 if args.dtype == "f32" else 1), n_gemms=n_gemms,
                         precision=sp.Precision.FP16)
    wl = sp.Workload(tokens=t_expert, phase=sp.Phase.GENERATION)
    args.plan_layer, args.plan_workload = layer, wl  # what predict_step() evaluates
    budget = args.budget_frac * layer.layer_bytes
    if args.config == "cfg1":
        return sp.SlicingRates(0.2, 0.3, 0.5), budget, "fixed 0.2/0.3/0.5 (BASELINE configs[0])", profile
    rates = solve_rates(args, profile, budget)
    if getattr(args, "force_cc", -1.0) >= 0.0:
        source += f" (r_CC forced to {args.force_cc}: probe, not the planner's split)"
    return rates, budget, source, profile


def solve_rates(args, profile, budget):
    """greedy_assign (memory_assigner.py:37-122) then solve_rcg (rate_solver.py:90-117)."""
    import paper_2411_15715_b200 as sp

    layer, wl = args.plan_layer, args.plan_workload
    mem = sp.greedy_assign(profile, [layer], wl, budget, n_steps=16)
    rates = sp.solve_rcg(profile, layer, wl, mem.per_layer_rgg[0]).rates
    if getattr(args, "force_cc", -1.0) >= 0.0:
        rates = sp.SlicingRates(args.force_cc, 1.0 - rates.gg - args.force_cc, rates.gg)
    return rates


def predict_step(args, rates, profile) -> dict:
    """The planner's own prediction of one step on the profile it planned with:
    stage times (pipeline.py:143-167), the Eq. 5 recurrence over the step's
    n_gemms GEMMs (pipeline.py:237-260) and its Gantt rows (pipeline.py:347-364),
    per stream busy time next to t_fin."""
    import paper_2411_15715_b200 as sp

    layer, wl = args.plan_layer, args.plan_workload
    stage = sp.stage_times_generation(profile, layer, wl, rates)
    tl = sp.evaluate_recurrence(stage, layer.n_gemms)
    return {"t_fin_s": tl.t_fin, "case": tl.case_label.value, "n_gemms": layer.n_gemms,
            "busy_s": {"transfer": stage.transfer_s * layer.n_gemms, "gpu": stage.gpu_s * layer.n_gemms,
                       "cpu": stage.cpu_s * layer.n_gemms, "launch": stage.launch_s * layer.n_gemms},
            "gantt": sp.timeline_records(stage, tl)}


def calibrate_host_terms(args, profile, rates, spans, steps) -> tuple:
    """Per-box recalibration of the host side of the cost model.

    The committed profile was fitted on one pool box; host DRAM bandwidth (the
    CC block) and the effective link rate under that load (the CG copies) vary
    box to box.  ``spans`` are the library trace of ``steps`` real decode steps
    at ``rates``: the measured CC busy time and copy busy time per step are
    divided by what the profile predicts for the same step
    (stage_times_generation, pipeline.py:143-167), and the profile's CPU GEMM
    and PCIe terms (alpha and beta) are scaled by those ratios -- the same
    linear model (perf_model.py:99-128), re-anchored on this box.  The caller
    re-runs solve_rcg on the result."""
    from paper_2411_15715_b200 import costs

    pred = predict_step(args, rates, profile)["busy_s"]
    meas_cpu = sum(s["end_s"] - s["start_s"] for s in spans if s["kind"] == "cc") / steps
    meas_link = sum(s["end_s"] - s["start_s"] for s in spans if s["kind"] == "copy") / steps
    k_cpu = meas_cpu / pred["cpu"] if pred["cpu"] > 0 and meas_cpu > 0 else 1.0
    k_link = meas_link / pred["transfer"] if pred["transfer"] > 0 and meas_link > 0 else 1.0
    doc = costs.profile_to_dict(profile)
    for g in doc.get("gemm", {}).values():
        if "cpu" in g:
            g["cpu"]["alpha"] *= k_cpu
            g["cpu"]["beta"] *= k_cpu
    if "pcie" in doc:
        doc["pcie"]["alpha"] *= k_link
        doc["pcie"]["beta"] *= k_link
    info = {"k_cpu": k_cpu, "k_link": k_link, "steps": steps,
            "cpu_busy_s": {"measured": meas_cpu, "predicted": pred["cpu"]},
            "transfer_busy_s": {"measured": meas_link, "predicted": pred["transfer"]}}
    return costs.profile_from_dict(doc), info


def calibrate_prompt_terms(profile, layer_spec, rates, plans, layers, spans) -> tuple:
    """The prompt-phase counterpart of calibrate_host_terms.  ``spans`` are the
    library trace of one prefill through ``layers`` layers cycling ``plans``:
    measured host CC busy and copy busy, over what the profile predicts for the
    same calls (planner.prompt_layer_busy), scale the profile's CPU GEMM and
    PCIe terms.  The caller re-plans the token split on the result."""
    import paper_2411_15715_b200 as sp
    from paper_2411_15715_b200 import costs

    pred_link = pred_cpu = 0.0
    for l in range(layers):
        calls = plans[l % len(plans)]
        lk, cp = sp.prompt_layer_busy(profile, layer_spec, [len(c.token_ids) for c in calls],
                                      [c.n_g for c in calls], rates)
        pred_link += lk
        pred_cpu += cp
    meas_cpu = sum(s["end_s"] - s["start_s"] for s in spans if s["kind"] == "cc")
    meas_link = sum(s["end_s"] - s["start_s"] for s in spans if s["kind"] == "copy")
    k_cpu = meas_cpu / pred_cpu if pred_cpu > 0 and meas_cpu > 0 else 1.0
    k_link = meas_link / pred_link if pred_link > 0 and meas_link > 0 else 1.0
    doc = costs.profile_to_dict(profile)
    for g in doc.get("gemm", {}).values():
        if "cpu" in g:
            g["cpu"]["alpha"] *= k_cpu
            g["cpu"]["beta"] *= k_cpu
    if "pcie" in doc:
        doc["pcie"]["alpha"] *= k_link
        doc["pcie"]["beta"] *= k_link
    info = {"k_cpu": k_cpu, "k_link": k_link, "layers": layers,
            "n_g_layer0_before": [c.n_g for c in plans[0]],
            "cpu_busy_s": {"measured": meas_cpu, "predicted": pred_cpu},
            "transfer_busy_s": {"measured": meas_link, "predicted": pred_link}}
    return costs.profile_from_dict(doc), info


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: NVML
    every 5 ms from a thread (a decode region lasts ~0.2-0.4 s, far below the
    100 ms granularity of ``nvidia-smi -lms``), nvidia-smi as the fallback."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    # nvmlClocksEventReason* bits, in NAMES order
    BITS = [0x8, 0x40, 0x20, 0x4]
    PERIOD_S = 0.005

    def __init__(self, device=0):
        self.rows, self.proc, self.device, self.armed = [], None, device, False
        self.first = threading.Event()
        self.nvml, self.handle, self.stop_ev, self.source = None, None, threading.Event(), "unsampled"

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            from paper_2411_15715_b200.placement import pci_bus_id

            bid = pci_bus_id(self.device)
            try:
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bid.encode() if bid else b"")
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml = pynvml
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.source = f"nvml every {self.PERIOD_S * 1e3:g} ms"
            threading.Thread(target=self._poll, daemon=True).start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            self.first.wait(timeout=10)
            self.source = "nvidia-smi -lms 100"
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        reason_fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_ev.is_set():
            if self.armed:
                try:
                    sm = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                    r = int(reason_fn(self.handle))
                    self.rows.append([str(sm), str(self.max_sm)] +
                                     ["Active" if r & b else "Not Active" for b in self.BITS])
                except Exception:
                    pass
            time.sleep(self.PERIOD_S)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.first.set()
                if self.armed:
                    self.rows.append(parts)

    def stop(self):
        self.stop_ev.set()
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "source": self.source}
        num = lambda v: float(v) if v.replace(".", "").isdigit() else None  # noqa: E731
        sm = [v for v in (num(r[0]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of slicing_kernel.py) -- baseline only


def blas_info() -> tuple[int, list]:
    """(BLAS threads, threadpoolctl.threadpool_info() BLAS entries)."""
    try:
        import threadpoolctl

        info = [{k: i.get(k) for k in ("user_api", "internal_api", "num_threads", "version", "architecture")}
                for i in threadpoolctl.threadpool_info() if i.get("user_api") == "blas"]
        return max((i["num_threads"] or 1 for i in info), default=os.cpu_count() or 1), info
    except Exception:
        return os.cpu_count() or 1, []


def cpu_reference_sample(args, rates, steps, warmup=1, tokens=None, min_s=0.0, max_steps=None):
    """fp64 numpy sliced forward (the reference algorithm, slicing_kernel.py:97-124)
    of `tokens` tokens (default: the global batch) through top-k SwiGLU experts;
    two fp64 expert weight sets (> L3) reused across steps.  Times at least
    `steps` steps and keeps going until `min_s` seconds of CPU work (bounded by
    `max_steps`).  Returns a dict: tokens/s over the whole sample, best and
    median per-step tokens/s, step times, threads and the BLAS pool."""
    import torch

    from oracle import sliced_forward as orc

    M, H = args.model_dim, args.hidden_dim
    tokens = tokens or args.batch
    torch.manual_seed(0)
    sets = [tuple((torch.randn(*s) / 64).double().numpy() for s in ((M, H), (M, H), (H, M)))
            for _ in range(min(2, args.top_k))]
    x = np.random.default_rng(0).standard_normal((tokens, M))
    gates = np.full(args.top_k, 1.0 / args.top_k)

    def step():
        y = np.zeros((tokens, M))
        for k in range(args.top_k):
            w1, w3, w2 = sets[k % len(sets)]
            y += gates[k] * orc.sliced_forward(x, w1, w2, "silu", rates.cc, rates.cg, w3)
        return y

    for _ in range(warmup):
        step()
    times = []
    t_all = time.perf_counter()
    while len(times) < steps or (time.perf_counter() - t_all < min_s and len(times) < (max_steps or 10 ** 9)):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = time.perf_counter() - t_all
    threads, info = blas_info()
    desc = (f"{len(times)} steps x {tokens} token(s) x {args.top_k} experts ({total:.1f} s of CPU work), fp64 "
            f"numpy/OpenBLAS (slicing_kernel.py:97-124 as written), rates cc={rates.cc:.4f} cg={rates.cg:.4f} "
            f"gg={rates.gg:.4f}, 2 fp64 expert weight sets")
    return {"value": tokens * len(times) / total, "best": tokens / min(times), "median": tokens / float(np.median(times)),
            "s_per_step": total / len(times), "steps": len(times), "threads": threads, "threadpool": info,
            "sample": desc}


# ---------------------------------------------------------------------------


def ncu_traffic(args):
    """dram__bytes_read.sum + dram__bytes_write.sum per GG launch from the
    committed ncu --set full capture of this workload (profiles/ncu_traffic.json)."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    if not f.exists():
        return None
    return json.loads(f.read_text()).get(f"{args.config}_gg_launch_bytes")


def rank_device(local_rank: int) -> int:
    """CUDA device of a local rank: one GPU per rank; every rank on cuda:0
    under SP_BENCH_ONE_GPU=1 (multi-rank plumbing on a one-GPU box)."""
    return 0 if os.environ.get("SP_BENCH_ONE_GPU") == "1" else local_rank


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def base_config(args, global_batch, world):
    """The config both arms print (identical dicts, so the driver's same-config
    check compares like with like).  The split the GPU arm executes (rates,
    block widths) is reported under its own ``split`` key: it is re-planned on
    each box, and the reference arm's fp64 forward computes all three blocks on
    the host whatever the split."""

    wl = {"cfg1": "cfg1-1024x3584-moe-ffn-decode", "cfg2": "mixtral-8x7b-moe-ffn-decode",
          "cfg4": "llama2-70b-dense-ffn-decode-colsharded",
          "cfg5": f"{'phimoe' if args.moe == 'phimoe' else 'mixtral-8x22b'}-moe-ffn-decode-ep"}.get(args.config, args.config)
    return {"workload": wl,
            "model_dim": args.model_dim, "hidden_dim": args.hidden_dim, "experts": args.experts,
            "top_k": args.top_k, "batch_per_gpu": args.batch, "global_batch": global_batch,
            "parallelism": (f"col{world}" if args.config == "cfg4" else f"ep{world}") if world > 1 else "single",
            "budget_frac": args.budget_frac,
            "l2": "inputs larger than L2: the experts' GG blocks (>1 GB) rotate with routing"}


def run_reference(args):
    """The reference arm: the reference's CPU algorithm (the oracle port of
    slicing_kernel.py:97-124, fp64 numpy, every host thread) on this arm's
    config -- the same global batch per step as the GPU arm at N ranks, planned
    with rank 0's rates.  Under torchrun only rank 0 runs and prints."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    from paper_2411_15715_b200.placement import bind_rank

    # plan exactly as rank 0 of the GPU arm does (its host-thread share), run on every core
    bind_rank(0, world, device_of=rank_device, apply=False)
    if args.config == "cfg4":
        from paper_2411_15715_b200.expert_parallel import column_shard

        lo, hi = column_shard(args.hidden_dim, 0, world)
        args.shard_hidden = hi - lo
    rates, _, _, _ = plan_rates(args, args.batch)
    global_batch = args.batch * world
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=os.cpu_count(), user_api="blas"):
        # the whole layer (every rank's experts / column shards) for the global batch
        r = cpu_reference_sample(args, rates, args.steps, warmup=args.warmup, tokens=global_batch)
    line = {
        "impl": "reference", "metric": metric_name(args), "value": r["value"], "unit": UNIT, "n_gpus": world,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["s_per_step"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": base_config(args, global_batch, world),
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port",
                         "sample": r["sample"], "best": r["best"], "median": r["median"], "threadpool": r["threadpool"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_experts(args, rates, owned, device, hidden=None):
    """Random-init experts (HF layout) placed by `rates`."""
    import torch

    from paper_2411_15715_b200.sliced import SlicedFFN

    M, H = args.model_dim, hidden or args.hidden_dim
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    experts = {}
    for e in owned:
        g = torch.Generator(device=device).manual_seed(1000 + e)
        w1t = (torch.randn(H, M, device=device, generator=g) / 64).to(tdt).cpu()
        w3t = (torch.randn(H, M, device=device, generator=g) / 64).to(tdt).cpu()
        w2t = (torch.randn(M, H, device=device, generator=g) / 120).to(tdt).cpu()
        experts[e] = SlicedFFN(w1t, w2t, rates, w3t=w3t, activation="silu", dtype=args.dtype, device=device.index)
        del w1t, w3t, w2t
    return experts


def run_ours(args):
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.expert_parallel import ExpertParallelMoE, local_experts

    from paper_2411_15715_b200.placement import bind_rank

    world, rank, local = dist_env()
    # SP_BENCH_ONE_GPU=1 (test plumbing): every rank on cuda:0 with gloo, so the
    # multi-rank bench path runs on a one-GPU box; production is one GPU per rank, NCCL
    one_gpu = os.environ.get("SP_BENCH_ONE_GPU") == "1"
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    dev_index = rank_device(local)
    device = torch.device("cuda", dev_index)
    torch.cuda.set_device(device)
    # this rank's share of its GPU's NUMA node (CPU mask + preferred memory),
    # before sp_init creates the CC pool and before any pinned weight is placed
    placement = bind_rank(local, local_world, device_of=rank_device)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist

        backend = "gloo" if one_gpu else "nccl"
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    nat.init(dev_index)

    B = args.batch
    global_batch = B * world
    if args.config == "cfg4":
        from paper_2411_15715_b200.expert_parallel import ColumnShardedFFN, column_shard

        lo, hi = column_shard(args.hidden_dim, rank, world)
        args.shard_hidden = hi - lo
    rates, budget, source, profile = plan_rates(args, B)
    fitted = profile  # the committed fit: link peak and in-situ CC rate for the roofline keys
    rng = np.random.default_rng(7)
    if args.config == "cfg4":
        experts = make_experts(args, rates, [rank], device, hidden=hi - lo)
        moe = ColumnShardedFFN(experts[rank])
    else:
        experts = make_experts(args, rates, local_experts(args.experts, rank, world), device)
        router = rng.standard_normal((args.model_dim, args.experts))
        moe = ExpertParallelMoE(experts, router, args.top_k, args.experts, out_dim=args.model_dim)
    pool = 64
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    xs_dev = [torch.from_numpy(rng.standard_normal((global_batch, args.model_dim)).astype(np.float32)).to(device, tdt)
              for _ in range(pool)]
    xs_host = [x.float().cpu().numpy() for x in xs_dev]  # routing sees the values the kernels see

    def step(i, host_io=False):
        # device I/O: routing reads x back from the GPU inside the timed region
        j = i % pool
        return moe(xs_host[j]) if host_io else moe(xs_dev[j])

    per_step_wall = []  # host wall ms of every step, per timed region (outlier check)

    def timed(n, host_io=False, trace=False):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        if trace:
            nat.trace_enable(True, gg_only=(trace == "gg"))
        l0 = nat.stats()["kernel_launches"]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        ticks = [t0]
        for i in range(n):
            step(i, host_io)
            ticks.append(time.perf_counter())
        b.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        per_step_wall.append(np.diff(ticks) * 1e3)
        launches = nat.stats()["kernel_launches"] - l0
        spans = nat.trace_fetch() if trace else []
        if trace:
            nat.trace_enable(False)
        ms = a.elapsed_time(b)
        if dist is not None:
            tt = torch.tensor([ms], device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms / n, wall / n, launches, spans

    for i in range(args.warmup):
        step(i)
        step(i, host_io=True)
    torch.cuda.synchronize()

    # ---- per-box recalibration of the host terms, then re-plan (before timing) ----
    calib = None
    if args.calibrate and args.config != "cfg1" and (args.experts > 1 or args.config == "cfg4"):
        # Fixed-point rounds: trace the step at the current split, rescale the
        # host terms by measured / predicted, re-solve, re-slice, repeat until
        # the split stops moving.  One round re-anchors the model at the OLD
        # split only; where the host's per-row CC cost depends on the split
        # itself (batched decode: CC block on the critical path or not, shared
        # host DRAM with the copies), the next round measures the new split.
        from dataclasses import asdict

        from paper_2411_15715_b200.sliced import split_boundaries

        t_cal = time.perf_counter()
        rates0, profile0 = rates, profile
        t_fin0 = predict_step(args, rates0, profile0)["t_fin_s"]
        rounds, k_cpu_tot, k_link_tot, resliced = [], 1.0, 1.0, False
        for _ in range(max(1, args.calib_rounds)):
            _, _, _, cspans = timed(args.calib_steps, trace="full")
            profile, info = calibrate_host_terms(args, profile, rates, cspans, args.calib_steps)
            k_cpu_tot *= info["k_cpu"]
            k_link_tot *= info["k_link"]
            new_rates = solve_rates(args, profile, budget)
            info.update(rates=asdict(rates), rates_next=asdict(new_rates))
            rounds.append(info)
            moved = abs(new_rates.cc - rates.cc) > args.calib_tol or abs(new_rates.cg - rates.cg) > args.calib_tol
            w0 = next(iter(experts.values())).block_widths if experts else None
            if experts and tuple(split_boundaries(w0[0] + w0[1] + w0[2], new_rates)) != (w0[0], w0[0] + w0[1]):
                new_experts = {e: ex.reslice(new_rates) for e, ex in experts.items()}
                for ex in experts.values():
                    ex.layer.release()
                experts = new_experts
                resliced = True
                if args.config == "cfg4":
                    moe = ColumnShardedFFN(experts[rank])
                else:
                    moe = ExpertParallelMoE(experts, router, args.top_k, args.experts, out_dim=args.model_dim)
                for i in range(args.warmup):
                    step(i)
                    step(i, host_io=True)
                torch.cuda.synchronize()
            rates = new_rates
            if not moved:
                break
        source += f" (host terms recalibrated on this box: CPU x{k_cpu_tot:.3f}, link x{k_link_tot:.3f})"
        calib = {"k_cpu": k_cpu_tot, "k_link": k_link_tot, "steps": args.calib_steps,
                 "cpu_busy_s": rounds[-1]["cpu_busy_s"], "transfer_busy_s": rounds[-1]["transfer_busy_s"],
                 "rounds": rounds, "rates_before": asdict(rates0), "rates_after": asdict(rates),
                 "resliced": resliced, "t_fin_pred_before_s": t_fin0, "seconds": time.perf_counter() - t_cal}

    clk = ClockSampler(local).start()
    clk.armed = True
    # the headline region records device events only around the GG launches (the
    # roofline kernel) plus host-clock CC spans: full tracing puts events on the
    # saturated copy stream and slows the step it measures
    ms_step, wall_step, launches, gg_spans = timed(args.steps, trace="gg")
    clk.armed = False
    clk.stop()
    clocks = clk.summary()
    # SP_BENCH_TRACE_E2E=path: also trace the e2e region (probe; the e2e number then carries the trace cost)
    e2e_trace = os.environ.get("SP_BENCH_TRACE_E2E", "")
    e2e_ms, _, _, e2e_spans = timed(args.steps, host_io=True, trace="full" if e2e_trace else False)
    if e2e_trace and rank == 0:
        Path(e2e_trace).write_text(json.dumps(e2e_spans))
    # a third region of the same steps, fully traced: per-stream busy time, copy
    # rates and the measured Gantt (analysis only; its own step time is reported)
    full_ms, _, _, spans = timed(args.steps, trace="full")
    value = global_batch / (ms_step * 1e-3)
    e2e_value = global_batch / (e2e_ms * 1e-3)

    # ---- kernel-level roofline from the trace (CUDA events on the library's compute stream) ----
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    gg = [s for s in gg_spans if s["kind"] == "gg"]
    cp = [s for s in spans if s["kind"] == "copy"]
    cc = [s for s in spans if s["kind"] == "cc"]
    gg_bytes = float(np.mean([s["bytes"] for s in gg])) if gg else 0.0
    gg_dt = float(np.mean([s["end_s"] - s["start_s"] for s in gg])) if gg else 0.0
    gg_gbs = gg_bytes / gg_dt / 1e9 if gg_dt else 0.0
    # the same launches timed on the device itself (first CTA start -> last CTA
    # end, %globaltimer).  A timing event recorded while copy-engine H2D traffic
    # saturates the link costs ~23 us of stream time (scripts/probes/event_span.cu),
    # which is why the grouped GG launch runs behind the last chunk kernel.
    gg_dev = [s["dev_s"] for s in gg if s.get("dev_s", 0) > 0]
    gg_dev_dt = float(np.mean(gg_dev)) if gg_dev else 0.0
    cp_bytes = sum(s["bytes"] for s in cp)
    cp_busy = sum(s["end_s"] - s["start_s"] for s in cp)
    link_peak = 1.0 / fitted.pcie.beta / 1e9 if fitted.pcie and fitted.pcie.beta else 55.5
    step_s = ms_step * 1e-3
    gg_step_bytes = sum(s["bytes"] for s in spans if s["kind"] == "gg") / args.steps
    cg_step_bytes = cp_bytes / args.steps
    t_roof = max(gg_step_bytes / (hbm_peak * 1e9), cg_step_bytes / (link_peak * 1e9))
    cc_busy = sum(s["end_s"] - s["start_s"] for s in cc) / args.steps
    # the host side of the step: CC bytes at the profile's fitted (in-situ) CC rate
    cc_step_bytes = sum(s["bytes"] for s in cc) / args.steps
    g16 = fitted.gemm.get(sp_precision_fp16()) if fitted.gemm else None
    cc_rate = 2.0 / g16.cpu.beta if g16 is not None and g16.cpu and g16.cpu.beta else None
    t_host = max(t_roof, cc_step_bytes / cc_rate) if cc_rate else None
    if args.trace_out and rank == 0:
        keep = int(os.environ.get("SP_TRACE_KEEP_CALLS", "4"))
        Path(args.trace_out).write_text(json.dumps([s for s in spans if s["call"] < keep], indent=0))

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(limits=os.cpu_count(), user_api="blas"):
            r = cpu_reference_sample(args, rates, args.cpu_sample_steps, min_s=args.cpu_sample_s, max_steps=2000)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port", "sample": r["sample"],
               "best": r["best"], "median": r["median"], "threadpool": r["threadpool"]}

    first = next(iter(experts.values())) if experts else None
    xel = 2 if args.dtype == "bf16" else 4
    from paper_2411_15715_b200.sliced import split_boundaries

    config = base_config(args, global_batch, world)
    hidden = getattr(args, "shard_hidden", args.hidden_dim)
    b1, b2 = split_boundaries(hidden, rates)
    split = {"rates": {"cc": rates.cc, "cg": rates.cg, "gg": rates.gg}, "block_widths": [b1, b2 - b1, hidden - b2]}
    assert first is None or list(first.block_widths) == split["block_widths"]
    pred = predict_step(args, rates, profile) if args.experts > 1 or args.config == "cfg4" else None
    meas_busy = {"transfer": cp_busy / args.steps, "cpu": cc_busy,
                 "gpu": sum(s["end_s"] - s["start_s"] for s in spans if s["stream"] == "gpu") / args.steps}
    line = {
        "metric": metric_name(args), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (random-init weights, seeded)",
        "config": config,
        "split": split,
        "calibration": calib,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": global_batch * args.model_dim * xel,
                "d2h_bytes_per_step": global_batch * args.model_dim * 4},
        "roofline": {"bound": "hbm", "kernel": "ffn_block_kernel on the GG block (fused up+gate+down, TMA bulk ring)",
                     "achieved": gg_gbs, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": gg_gbs / hbm_peak if hbm_peak else None, "traffic": ncu_traffic(args),
                     "algorithmic_bytes_per_launch": gg_bytes, "mean_launch_us": gg_dt * 1e6,
                     "device_span_us": gg_dev_dt * 1e6,
                     "achieved_device_span": gg_bytes / gg_dev_dt / 1e9 if gg_dev_dt else None,
                     "frac_device_span": gg_bytes / gg_dev_dt / 1e9 / hbm_peak if gg_dev_dt and hbm_peak else None,
                     "timing": "achieved/frac: CUDA events on the library compute stream around each GG launch "
                               "in the timed region; *_device_span: the same launches, in-kernel %globaltimer"},
        "link": {"cg_copy_GBps_while_busy": cp_bytes / cp_busy / 1e9 if cp_busy else None,
                 "cg_GBps_over_step": cg_step_bytes / step_s / 1e9, "link_peak_GBps": link_peak,
                 "frac_over_step": (cg_step_bytes / step_s / 1e9) / link_peak if link_peak else None,
                 "step_roofline_s": t_roof, "step_roofline_frac": t_roof / step_s if step_s else None,
                 "cc_host_s_per_step": cc_busy,
                 "cc_rate_GBps_fitted": cc_rate / 1e9 if cc_rate else None,
                 "step_bound_with_cc_s": t_host,
                 "step_bound_with_cc_frac": t_host / step_s if t_host and step_s else None},
        "model_vs_measured": None if pred is None else {
            "t_fin_pred_s": pred["t_fin_s"], "step_meas_s": step_s, "meas_over_pred": step_s / pred["t_fin_s"],
            "case": pred["case"], "n_gemms": pred["n_gemms"],
            "busy_pred_s": pred["busy_s"], "busy_meas_s": meas_busy,
            "gantt_pred": pred["gantt"],
            "step_full_trace_s": full_ms * 1e-3,
            "note": "planner prediction (stage_times_generation + evaluate_recurrence, pipeline.py:143-167,237-260, "
                    "Gantt rows :347-364) on the profile that chose the rates, vs the measured step and per-stream "
                    "busy time (library trace of a separate, fully traced region of the same steps, rank 0; "
                    "step_full_trace_s is that region's own step time)"},
        "plan": {"gpu_budget_bytes": budget, "profile": source,
                 "placed_bytes_per_expert": first.layer.placed_bytes() if first else {}},
        "placement": placement.summary(),
        "collective": None if world == 1 else {
            "backend": backend, "op": "all_reduce(sum) of fp32 partial outputs, one per step",
            "bytes_per_step": global_batch * args.model_dim * 4},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "wall_ms_per_step": wall_step * 1e3,
        "step_wall_ms": {name: {"p50": float(np.percentile(w, 50)), "p90": float(np.percentile(w, 90)),
                                "max": float(np.max(w))}
                         for name, w in zip(("value", "e2e"), per_step_wall)},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_prefill_decode(args):
    """BASELINE configs[2]: L MoE FFN layers, a P-token prompt routed top-2 per
    layer, each expert's share T_e split by the token assigner (solve_ng on the
    prompt-phase B200 profile, rates frozen from decode): the last n_g rows run
    the CC columns on the GPU (streamed CC chunks), the rest on host threads;
    then decode steps through the same layers."""
    import torch

    import paper_2411_15715_b200 as sp
    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.sliced import CallSpec, forward_calls, moe_route

    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("cfg3 runs on one GPU")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    nat.init(local)
    rates, budget, source, _ = plan_rates(args, 1)
    args.prompt_profile = prompt_profile_path(args)
    p_profile, p_source = load_profile(args.prompt_profile)
    if p_source.startswith("fallback"):
        p_profile, p_source = load_profile(args.profile)
    layer_spec = sp.LayerSpec(args.model_dim, args.hidden_dim, n_gemms=3, precision=sp.Precision.FP16)
    D = min(args.distinct_layers, args.layers)
    sets = [make_experts(args, rates, range(args.experts), device) for _ in range(D)]
    rng = np.random.default_rng(11)
    routers = [rng.standard_normal((args.model_dim, args.experts)) for _ in range(D)]
    xp = torch.from_numpy(rng.standard_normal((args.prompt, args.model_dim)).astype(np.float32)).to(device, torch.bfloat16)
    xp_host = xp.float().cpu().numpy()
    xd = [torch.from_numpy(rng.standard_normal((1, args.model_dim)).astype(np.float32)).to(device, torch.bfloat16)
          for _ in range(16)]
    xd_host = [x.float().cpu().numpy() for x in xd]
    ng_cache: dict[int, int] = {}

    def n_g_for(t_e: int) -> int:
        if t_e not in ng_cache:
            ng_cache[t_e] = (int(round(args.ng_frac * t_e)) if args.ng_frac >= 0
                             else sp.solve_ng(p_profile, layer_spec, t_e, rates,
                                              transfer_model=args.transfer_model).n_g)
        return ng_cache[t_e]

    layer_plans = []

    def plan(d, x_host, split):
        ids, gates = moe_route(x_host.astype(np.float32), routers[d], args.top_k)
        routed = []
        for e, ffn in sets[d].items():
            rows, slots = np.nonzero(ids == e)
            if rows.size:
                routed.append((ffn, rows, slots))
        if split and args.token_plan == "layer":
            # extension: the layer's experts planned together (planner.solve_ng_layer)
            lp = sp.solve_ng_layer(p_profile, layer_spec, [r.size for _, r, _ in routed], rates)
            layer_plans.append(lp)
            ngs = list(lp.n_g)
        else:
            ngs = [n_g_for(r.size) if split else 0 for _, r, _ in routed]
        return [CallSpec(ffn.layer, rows.astype(np.int32), gates[rows, slots].astype(np.float32), ng)
                for (ffn, rows, slots), ng in zip(routed, ngs)]

    prompt_plans = [plan(d, xp_host, True) for d in range(D)]
    decode_plans = [[plan(d, xh, False) for xh in xd_host] for d in range(D)]
    out_p = torch.empty_like(xp)
    out_d = torch.empty_like(xd[0])

    def prefill():
        for l in range(args.layers):
            forward_calls(prompt_plans[l % D], xp, out=out_p)

    # ---- per-box recalibration of the prompt profile's host terms, then re-plan ----
    pcalib = None
    if args.calibrate:
        prefill()  # staging / workspaces at prompt size
        torch.cuda.synchronize()
        nat.trace_enable(True)
        prefill()
        torch.cuda.synchronize()
        cspans = nat.trace_fetch()
        nat.trace_enable(False)
        p_profile, pcalib = calibrate_prompt_terms(p_profile, layer_spec, rates, prompt_plans, args.layers, cspans)
        p_source += (f" (host terms recalibrated on this box: CPU x{pcalib['k_cpu']:.3f}, "
                     f"link x{pcalib['k_link']:.3f})")
        ng_cache.clear()
        layer_plans.clear()
        prompt_plans = [plan(d, xp_host, True) for d in range(D)]
        pcalib["n_g_layer0_after"] = [c.n_g for c in prompt_plans[0]]

    def decode():
        for i in range(args.decode_steps):
            for l in range(args.layers):
                forward_calls(decode_plans[l % D][i % 16], xd[i % 16], out=out_d)

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e-3

    for _ in range(max(1, args.warmup)):
        prefill()
    clk = ClockSampler(local).start()
    clk.armed = True
    l0 = nat.stats()["kernel_launches"]
    t_p = min(timed(prefill) for _ in range(max(1, args.steps)))
    t_d = timed(decode)
    launches = nat.stats()["kernel_launches"] - l0
    clk.armed = False
    clk.stop()
    ng_used = {t: n for t, n in sorted(ng_cache.items())}
    t_e_prompt = sorted({len(c.token_ids) for c in prompt_plans[0]})
    # one traced prefill: the Y_cc transfer measured next to the reference's model of it
    nat.trace_enable(True)
    prefill()
    torch.cuda.synchronize()
    pspans = nat.trace_fetch()
    nat.trace_enable(False)
    ycc = [s for s in pspans if s["kind"] == "ycc"]
    ycc_meas = sum(s["end_s"] - s["start_s"] for s in ycc) / args.layers
    # the GG blocks of the traced prefill: tcgen05 chains (~128 tokens per expert)
    ggs = [s for s in pspans if s["kind"] == "gg" and s["bytes"] > 0]
    gg_b = sum(s["bytes"] for s in ggs)
    gg_t = sum(s["end_s"] - s["start_s"] for s in ggs)
    gg_d = sum(s["dev_s"] for s in ggs if s["dev_s"] > 0)
    peaks_doc = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks_doc.get("hbm_gbs")
    ycc_model = sum(sp.cc_result_transfer_time(p_profile, layer_spec,
                                               sp.Workload(tokens=len(c.token_ids) - c.n_g, phase=sp.Phase.PROMPT),
                                               rates, bytes_per_activation=4.0)
                    for c in prompt_plans[0] if len(c.token_ids) > c.n_g)
    if args.trace_out:
        nat.trace_enable(True)
        prefill()
        torch.cuda.synchronize()
        Path(args.trace_out).write_text(json.dumps([s for s in nat.trace_fetch() if s["call"] < 4], indent=0))
        nat.trace_enable(False)
        # the same through the host-I/O public API (x / y in host memory), after
        # two untraced host-I/O layers (staging and workspaces at host-I/O sizes)
        for l in range(min(2, args.layers)):
            forward_calls(prompt_plans[l % D], xp_host)
        torch.cuda.synchronize()
        nat.trace_enable(True)
        t0 = time.perf_counter()
        for l in range(min(4, args.layers)):
            forward_calls(prompt_plans[l % D], xp_host)
        torch.cuda.synchronize()
        host_wall = (time.perf_counter() - t0) / min(4, args.layers)
        Path(args.trace_out.replace(".json", "_hostio.json")).write_text(
            json.dumps([s for s in nat.trace_fetch() if s["call"] < 4], indent=0))
        nat.trace_enable(False)
        print(f"host-I/O prefill layer wall: {host_wall * 1e3:.1f} ms", flush=True)
    # host-I/O prefill through the public API (one untimed pass first: the host
    # staging and device workspace grow to the host-I/O sizes once)
    for l in range(min(2, args.layers)):
        forward_calls(prompt_plans[l % D], xp_host)
    t_e2e = timed(lambda: [forward_calls(prompt_plans[l % D], xp_host) for l in range(args.layers)])
    line = {
        "metric": metric_name(args), "value": args.prompt / t_p, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_p * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (random-init weights, seeded)",
        "decode_tokens_per_s": args.decode_steps / t_d, "decode_ms_per_token": t_d / args.decode_steps * 1e3,
        "config": {"workload": f"mixtral-8x7b-{args.layers}layer-prefill{args.prompt}-decode{args.decode_steps}",
                   "layers": args.layers,
                   "distinct_weight_sets": D, "prompt_tokens": args.prompt, "decode_steps": args.decode_steps,
                   "model_dim": args.model_dim, "hidden_dim": args.hidden_dim, "experts": args.experts,
                   "top_k": args.top_k, "rates": {"cc": rates.cc, "cg": rates.cg, "gg": rates.gg},
                   "gpu_budget_frac": args.budget_frac, "decode_profile": source, "prompt_profile": p_source,
                   "tokens_per_expert_layer0": t_e_prompt, "n_g_by_expert_tokens": ng_used,
                   "solve_ng_transfer_model": args.transfer_model, "token_plan": args.token_plan,
                   "layer_plan_n_g_layer0": list(layer_plans[0].n_g) if layer_plans else None,
                   "l2": f"{D} distinct layers x 8 experts ({D * 2.8:.0f} GB) cycled, >> L2"},
        "e2e": {"value": args.prompt / t_e2e, "unit": UNIT, "h2d_bytes_per_step": args.prompt * args.model_dim * 2 * args.layers,
                "d2h_bytes_per_step": args.prompt * args.model_dim * 4 * args.layers},
        "gpu_launches": launches, "clocks": clk.summary(), "prompt_calibration": pcalib,
        "roofline": {"bound": "hbm", "kernel": "tcgen05 GG chains (CTA-pair up GEMM + down GEMM) of one traced prefill",
                     "achieved": gg_b / gg_t / 1e9 if gg_t else None, "peak": hbm, "unit": "GB/s",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else None,
                     "frac": gg_b / gg_t / 1e9 / hbm if gg_t and hbm else None, "traffic": None,
                     "algorithmic_bytes_per_launch": gg_b / len(ggs) if ggs else None,
                     "mean_launch_us": gg_t / len(ggs) * 1e6 if ggs else None,
                     "frac_device_span": gg_b / gg_d / 1e9 / hbm if gg_d and hbm else None,
                     "blocks": len(ggs),
                     "timing": "per GG block: CUDA events on the compute stream (frac) and the chain's in-kernel "
                               "%globaltimer span (frac_device_span); the GG work is ~2 % of a prefill layer, its blocks "
                               "(half an expert, ~128 tokens, split K) share the SMs with the CG chunk kernels and "
                               "their events sit under a saturated host link"},
        "ycc_transfer": {"measured_ms_per_layer": ycc_meas * 1e3,
                         "model_ms_per_layer": ycc_model * 1e3 if ycc_model is not None else None,
                         "note": "CC partials host->HBM (pipeline.py:367-383 cc_result_transfer_time, fp32 "
                                 "partials); excluded from t_fin like the reference, overlapped with chunk kernels"},
    }
    print(json.dumps(line), flush=True)


def run_model(args):
    """the sliced MoE FFN inside a whole decoder loop
    (model.py): RMSNorm + GQA attention with RoPE over a static KV cache
    (torch SDPA), then the sliced MoE, per layer; batch-1 decode after a
    synthetic --prompt-token context."""
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral

    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("--config model runs on one GPU")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    nat.init(local)
    rates, budget, source, _ = plan_rates(args, 1)
    cfg = DecoderConfig(layers=args.layers, distinct=min(args.distinct_layers, args.layers),
                        model_dim=args.model_dim, hidden_dim=args.hidden_dim, experts=args.experts, top_k=args.top_k,
                        max_seq=args.prompt + args.warmup + 2 * args.steps + 8)
    m = SlicedMixtral(cfg, rates, device=local)
    g = torch.Generator(device=device).manual_seed(5)
    # the context: a real prefill through every layer (attention + sliced MoE with
    # solve_ng's token split on the prompt-phase profile), timed
    import paper_2411_15715_b200 as sp

    p_profile, _ = load_profile(args.prompt_profile or str(ROOT / "profiles" / "b200_prompt.json"))
    layer_spec = sp.LayerSpec(args.model_dim, args.hidden_dim, n_gemms=3, precision=sp.Precision.FP16)
    ng_cache = {}

    def planner(t_e):
        if t_e not in ng_cache:
            ng_cache[t_e] = sp.solve_ng(p_profile, layer_spec, t_e, rates, transfer_model=args.transfer_model).n_g
        return ng_cache[t_e]

    xp = (torch.randn(args.prompt, args.model_dim, device=device, generator=g) * 0.5).to(torch.bfloat16)
    m.prefill(xp, planner)  # warm-up: workspace / staging growth, attention plans (KV overwritten below)
    torch.cuda.synchronize()
    pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pa.record()
    hp_out = m.prefill(xp, planner)
    pb.record()
    torch.cuda.synchronize()
    t_prefill = pa.elapsed_time(pb) * 1e-3
    x0 = hp_out[-1:].clone()
    pos = args.prompt
    # eager reference speed (per-op launches), then the CUDA-graph decode that is timed below
    torch.cuda.synchronize()
    te = time.perf_counter()
    for _ in range(args.warmup):
        x0 = m.decode_step(x0, pos)
        pos += 1
    torch.cuda.synchronize()
    eager_ms = (time.perf_counter() - te) * 1e3 / max(1, args.warmup)
    m.enable_graphs(x0)
    m.pos_dev.fill_(pos)
    for _ in range(2):
        x0 = m.decode_step_graph(x0).clone()
        pos += 1
    torch.cuda.synchronize()
    clk = ClockSampler(local).start()
    clk.armed = True
    l0 = nat.stats()["kernel_launches"]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = x0
    a.record()
    for _ in range(args.steps):
        x = m.decode_step_graph(x)
        pos += 1
    b.record()
    torch.cuda.synchronize()
    launches = nat.stats()["kernel_launches"] - l0
    clk.armed = False
    clk.stop()
    t = a.elapsed_time(b) * 1e-3 / args.steps
    # e2e: the step's input from pinned host memory and its output read back every token
    xh = x0.float().cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    torch.cuda.synchronize()
    a.record()
    for _ in range(args.steps):
        xd = xh.to(device, non_blocking=True).to(torch.bfloat16)
        yh.copy_(m.decode_step_graph(xd).float(), non_blocking=True)
        pos += 1
    b.record()
    torch.cuda.synchronize()
    t_e2e = a.elapsed_time(b) * 1e-3 / args.steps
    line = {
        "metric": metric_name(args), "value": 1.0 / t, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (random-init weights, seeded)",
        "config": {"workload": "mixtral-8x7b-decoder-decode", "layers": cfg.layers, "distinct_moe_sets": cfg.distinct,
                   "context_tokens": args.prompt, "context": "real prefill (attention + sliced MoE, solve_ng split)", "heads": cfg.heads, "kv_heads": cfg.kv_heads,
                   "model_dim": cfg.model_dim, "hidden_dim": cfg.hidden_dim, "experts": cfg.experts,
                   "top_k": cfg.top_k, "rates": {"cc": rates.cc, "cg": rates.cg, "gg": rates.gg},
                   "budget_frac": args.budget_frac, "profile": source,
                   "l2": f"{cfg.distinct} MoE weight sets x 8 experts cycled, >> L2",
                   "launch": "torch part of each layer replayed as a CUDA graph; sliced MoE native call"},
        "e2e": {"value": 1.0 / t_e2e, "unit": UNIT, "h2d_bytes_per_step": args.model_dim * 4,
                "d2h_bytes_per_step": args.model_dim * 4},
        "gpu_launches": launches, "clocks": clk.summary(),
        "eager_ms_per_step": eager_ms,
        "prefill_tokens_per_s": args.prompt / t_prefill,
        "prefill_ms": t_prefill * 1e3,
    }
    m.release()
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args) -> int:
    """``bench.py --gpus N`` started without a torchrun environment re-executes
    itself under torchrun: one process per GPU on this node, rendezvous on
    127.0.0.1, NCCL's communicator set-up logged (NCCL_DEBUG=INFO, INIT) to
    stderr so the run shows which transport the all-reduce uses."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def dry_run(args):
    """Rendezvous, one barrier and a max-over-ranks reduction over gloo, then
    rank 0 prints a JSON line: the launch path without GPUs."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(rank)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world, "gpus_arg": args.gpus,
                          "max_rank": world - 1, "local_world": int(os.environ.get("LOCAL_WORLD_SIZE", "1"))}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = dist_env()[0]
    if world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: the run uses {world} ranks", file=sys.stderr)
    if args.dry_run:
        return dry_run(args)
    if args.config == "model" and args.impl == "ours":
        return run_model(args)
    if args.config == "cfg3" and args.impl == "ours":
        return run_prefill_decode(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
