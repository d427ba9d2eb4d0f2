"""Re-fit the planner's cost model to MEASURED B200 / host-link / host-core rates.

The reference fits ``alpha + n * beta`` per op class from profiling samples
(perf_model.py:429-466, CSV schema :312-320) but only ever feeds it synthetic
samples (:387-426).  This module produces the real samples on the machine the
runtime executes on, through the runtime's own code paths:

* ``gpu_gemm_fp16`` -- the GG block of a bf16 SwiGLU layer (up + gated act +
  down) over hidden widths h, timed with CUDA events on the library's compute
  stream (trace spans), per GEMM = span / 3; n = T * M * h.  L2 is flushed
  between samples so the weights stream from HBM as they do in decode.
* ``cpu_gemm_fp16`` -- the CC block on the host thread pool (AVX-512), per
  GEMM = wall time / 3; n = T * M * h.  The L3 is flushed between samples.
* ``c2g``           -- the runtime's own pinned-host -> HBM chunk copies (copy
  stream trace spans) over chunk sizes 0.8 - 31 MB.
* ``launch``        -- host enqueue time per kernel launch of a forward.

The CC threads and the copy engine read the same host DRAM at the same time
in every sliced step (the CC block runs while the CG chunks stream), and the
GG kernels run while the copy engine saturates the host link (which delays
the end of their CUDA-event spans by ~15-20 us, scripts/probe_gg.py and
scripts/probes/launch_latency.cu -- the kernels themselves run at full rate).
By default (``--load concurrent``) every rate is therefore sampled under the
load the step puts next to it: CC blocks and chunk copies come from real
sliced steps (``insitu_samples``, decode at T tokens per expert), prompt-phase
CC blocks under background copies and copies under a background CC block, GG
blocks under background host -> HBM copies.  ``--load isolated`` samples each
rate alone (the round-1 method).

``python -m paper_2411_15715_b200.b200_profile --out profiles/`` writes the
CSV and the fitted profile JSON (per phase: the GPU term is far from linear in
T across decode and prefill, SURVEY.md section 7 hard part 3).
"""

from __future__ import annotations

import argparse
import json
import threading
import time
from pathlib import Path

import numpy as np

from . import _native as nat
from .costs import OpClass, Precision, ProfileSample, fit_profile, save_profile, write_samples_csv

# Measured on the pool's boxes before the first refit (round 1 probe): pinned
# H2D 55.5 GB/s, numpy fp64 GEMV 136 GB/s on 16 host cores, HBM copy 6550.7
# GB/s (MEASURED_PEAKS.json).  Used only when no fitted profile exists yet.
FALLBACK_DECODE = {
    "testbed": "b200-fallback",
    "launch": {"alpha": 5.0e-6, "sigma2": 1.0e-12},
    "pcie": {"alpha": 1.0e-5, "beta": 1.0 / 55.5e9, "r2": 1.0},
    "gemm": {
        "fp16": {
            "gpu": {"alpha": 5.0e-6, "beta": 2.0 / 6.0e12, "r2": 1.0},
            "cpu": {"alpha": 2.0e-5, "beta": 2.0 / 100e9, "r2": 1.0},
        }
    },
}


class BackgroundCopy:
    """Keeps pinned host -> HBM copies in flight on a side stream (the CG
    streamer's host-DRAM load) while the block runs."""

    def __init__(self, torch, nbytes=64 << 20):
        self.torch = torch
        self.host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        self.dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.stream = torch.cuda.Stream()
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        torch = self.torch
        while not self.stop.is_set():
            with torch.cuda.stream(self.stream):
                for _ in range(4):
                    self.dev.copy_(self.host, non_blocking=True)
            self.stream.synchronize()

    def __enter__(self):
        self.th.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join()


class BackgroundCC:
    """Keeps a 150 MB CC block running on the host threads (the CC block's
    host-DRAM load) while the chunk copies are sampled."""

    def __init__(self, model_dim=4096, hidden=6144, seed=5):
        from .sliced import NativeLayer

        rng = np.random.default_rng(seed)
        w = rng.standard_normal((hidden, model_dim), dtype=np.float32) / 64
        self.lay = NativeLayer(w, w, hidden, hidden, "silu", w, dtype="bf16")
        self.x = rng.standard_normal((1, model_dim))
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop.is_set():
            self.lay.cc_forward_host(self.x)

    def __enter__(self):
        self.th.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join()
        self.lay.release()


def _flush_l2(torch, scratch):
    scratch.add_(1.0)  # 256 MB > 126 MB L2


def _flush_host(buf: np.ndarray) -> None:
    buf += 1.0  # 256 MB > 60 MB L3


def gpu_gemm_samples(torch, tokens: int, widths, model_dim=4096, reps=5, seed=0):
    from .sliced import NativeLayer

    scratch = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(seed)
    out = []
    for h in widths:
        w1t = (torch.randn(h, model_dim, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()
        w3t = (torch.randn(h, model_dim, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()
        w2t = (torch.randn(model_dim, h, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()
        lay = NativeLayer(w1t, w2t.t().contiguous(), 0, 0, "silu", w3t, dtype="bf16")
        x = torch.randn(tokens, model_dim, device="cuda").to(torch.bfloat16)
        from .sliced import CallSpec, forward_calls

        for r in range(reps + 2):
            _flush_l2(torch, scratch)
            torch.cuda.synchronize()
            nat.trace_enable(True)
            forward_calls([CallSpec(lay)], x)
            spans = [s for s in nat.trace_fetch() if s["kind"] == "gg"]
            nat.trace_enable(False)
            if r >= 2:
                dt = sum(s["end_s"] - s["start_s"] for s in spans) / 3.0
                out.append(ProfileSample(OpClass.GPU_GEMM, float(tokens) * model_dim * h, dt, Precision.FP16))
        lay.release()
    return out


def cpu_gemm_samples(tokens: int, widths, model_dim=4096, reps=5, seed=0, threads=0):
    from .sliced import NativeLayer

    rng = np.random.default_rng(seed)
    flush = np.zeros(32 << 20)
    out = []
    for h in widths:
        w1t = (rng.standard_normal((h, model_dim), dtype=np.float32) / 64)
        w3t = (rng.standard_normal((h, model_dim), dtype=np.float32) / 64)
        w2 = (rng.standard_normal((h, model_dim), dtype=np.float32) / 64)
        lay = NativeLayer(w1t, w2, h, h, "silu", w3t, dtype="bf16")
        x = rng.standard_normal((tokens, model_dim))
        for r in range(reps + 1):
            _flush_host(flush)
            t0 = time.perf_counter()
            lay.cc_forward_host(x, threads=threads)
            dt = (time.perf_counter() - t0) / 3.0
            if r >= 1:
                out.append(ProfileSample(OpClass.CPU_GEMM, float(tokens) * model_dim * h, dt, Precision.FP16))
        lay.release()
    return out


def c2g_samples(torch, chunk_rows=(32, 64, 128, 320, 640, 1280), reps=3, model_dim=4096):
    """Host-to-HBM chunk copies of the runtime itself (cudaHostAlloc'd region,
    copy stream), sized by chunk_rows; one sample per copy span."""
    from .sliced import CallSpec, NativeLayer, forward_calls

    h = 2 * max(chunk_rows)
    g = torch.Generator().manual_seed(3)
    w1t = torch.randn(h, model_dim, generator=g).to(torch.bfloat16)
    w2 = torch.randn(h, model_dim, generator=g).to(torch.bfloat16)
    x = torch.randn(1, model_dim, device="cuda").to(torch.bfloat16)
    out = []
    for cr in chunk_rows:
        lay = NativeLayer(w1t, w2, 0, h, "silu", w1t, dtype="bf16", chunk_rows=cr)
        for r in range(reps + 1):
            torch.cuda.synchronize()
            nat.trace_enable(True)
            forward_calls([CallSpec(lay)], x)
            spans = [s for s in nat.trace_fetch() if s["kind"] == "copy"]
            nat.trace_enable(False)
            if r >= 1:
                out += [ProfileSample(OpClass.C2G, float(s["bytes"]), s["end_s"] - s["start_s"]) for s in spans]
        lay.release()
    return out


def insitu_samples(torch, cc_rates=(0.1, 0.2, 0.3, 0.4), r_gg=0.5, model_dim=4096, hidden=14336,
                   experts=2, reps=6, seed=11, tokens=1, n_g_list=(0,)):
    """CPU GEMM and chunk-copy samples taken from real sliced decode steps.

    For each CC rate, `experts` SwiGLU experts are placed with rates
    (cc, 1 - r_gg - cc, r_gg) and run as one batched decode forward (the
    top-2 MoE step): the CC blocks (host threads) and the CG chunk copies
    (copy engine) then share host DRAM exactly as they do in production.
    Every CC block's host span gives one ``cpu_gemm_fp16`` sample (n = T*M*b1
    per GEMM, span / 3) and every chunk copy one ``c2g`` sample.  ``n_g_list``
    (prompt phase) diverts the last n_g of the tokens to the GPU, as the token
    assigner does, so the CC block runs at T - n_g tokens while the CC chunks
    stream to the GPU next to it."""
    from .sliced import CallSpec, NativeLayer, forward_calls

    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
    weights = [(mk(hidden, model_dim), mk(hidden, model_dim), mk(hidden, model_dim)) for _ in range(experts)]
    x = torch.randn(tokens, model_dim, device="cuda").to(torch.bfloat16)
    out = []
    for cc in cc_rates:
        b1 = int(np.floor(cc * hidden))
        b2 = int(np.floor((1.0 - r_gg) * hidden))
        lays = [NativeLayer(w1t, w2, b1, b2, "silu", w3t, dtype="bf16") for (w1t, w3t, w2) in weights]
        for r in range((reps + 2) * len(n_g_list)):
            n_g = n_g_list[r % len(n_g_list)]
            torch.cuda.synchronize()
            nat.trace_enable(True)
            forward_calls([CallSpec(l, n_g=n_g) for l in lays], x)
            torch.cuda.synchronize()
            spans = nat.trace_fetch()
            nat.trace_enable(False)
            if r < 2 * len(n_g_list):
                continue
            for s_ in spans:
                dt = s_["end_s"] - s_["start_s"]
                if s_["kind"] == "cc":
                    out.append(ProfileSample(OpClass.CPU_GEMM, float(tokens - n_g) * model_dim * b1, dt / 3.0,
                                             Precision.FP16))
                elif s_["kind"] == "copy":
                    out.append(ProfileSample(OpClass.C2G, float(s_["bytes"]), dt))
        for l in lays:
            l.release()
    return out


def launch_samples(torch, reps=20):
    from .sliced import CallSpec, NativeLayer, forward_calls

    rng = np.random.default_rng(1)
    lay = NativeLayer(rng.standard_normal((256, 512), dtype=np.float32), rng.standard_normal((256, 512), dtype=np.float32),
                      0, 0, "silu", rng.standard_normal((256, 512), dtype=np.float32), dtype="bf16")
    x = torch.randn(1, 512, device="cuda").to(torch.bfloat16)
    out = []
    for r in range(reps + 3):
        torch.cuda.synchronize()
        before = nat.stats()["kernel_launches"]
        nat.trace_enable(True)
        forward_calls([CallSpec(lay)], x)
        spans = [s for s in nat.trace_fetch() if s["kind"] == "launch"]
        nat.trace_enable(False)
        n = nat.stats()["kernel_launches"] - before
        if r >= 3 and spans and n:
            out.append(ProfileSample(OpClass.LAUNCH, 1.0, (spans[0]["end_s"] - spans[0]["start_s"]) / n))
    lay.release()
    return out


def measure(phase: str = "decode", quick: bool = False, load: str = "concurrent",
            tokens: int = 1, prompt_insitu: bool = False, cpu_tokens: int = 32) -> list[ProfileSample]:
    """decode: ``tokens`` per expert everywhere (1 = single-token decode; 2..8
    for batched decode, where each active expert sees a few tokens).  prompt:
    the GPU GEMM at T = 128 tokens (an expert's share of a 512-token top-2
    prompt, tensor-core path) and the host GEMM at T = 32.  One profile per
    regime, because t_G = alpha + T*M*H*beta (pipeline.py:163) is linear in T
    while a weight-streaming GEMV (and the host CC block) costs nearly the same
    for 1 or 4 tokens."""
    import torch

    nat.init(0)
    gpu_tokens, cpu_tokens = (tokens, tokens) if phase == "decode" else (128, cpu_tokens)
    widths = [256, 1024, 2048, 4096, 7168, 10240, 14336]
    cpu_widths = [128, 256, 512, 1024, 2048, 4096] if phase == "decode" else [256, 1024, 2048, 4096]
    if quick:
        widths, cpu_widths = [1024, 4096, 14336], cpu_widths[:3]
    if load == "concurrent":
        # every rate under the load the step puts next to it: GG kernels while
        # the copy engine writes the ring, CC blocks and chunk copies from
        # real sliced steps (decode), copies under a running CC block (prompt)
        with BackgroundCopy(torch):
            samples = gpu_gemm_samples(torch, gpu_tokens, widths, reps=3 if quick else 5)
        if phase == "decode":
            samples += insitu_samples(torch, reps=3 if quick else 6, tokens=tokens)
        elif prompt_insitu:
            # real prompt steps: 128 tokens per expert (a 512-token top-2 prompt's
            # share), the CC block at 128 - n_g tokens while the chunks stream
            samples += insitu_samples(torch, cc_rates=(0.2, 0.35), reps=2 if quick else 3, tokens=128,
                                      n_g_list=(32, 48, 64, 80))
        else:
            # Default for the prompt phase: CC blocks at 32 tokens under background
            # copies, copies under a background CC block.  The in-situ line (above)
            # is the more faithful measurement, but the reference's cost model is
            # linear in T*M*H per GEMM and solve_ng plans one expert at a time
            # while all of a layer's experts share the host: with the in-situ
            # line it keeps every prompt row on the host (n_g = 0) and the layer
            # turns CPU bound (measured 405-456 vs 533 prefill tokens/s).
            with BackgroundCopy(torch):
                samples += cpu_gemm_samples(cpu_tokens, cpu_widths, reps=2 if quick else 4)
            with BackgroundCC():
                samples += c2g_samples(torch)
    else:
        samples = gpu_gemm_samples(torch, gpu_tokens, widths, reps=3 if quick else 5)
        samples += cpu_gemm_samples(cpu_tokens, cpu_widths, reps=2 if quick else 4)
        samples += c2g_samples(torch)
    samples += launch_samples(torch)
    return samples


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--phase", default="decode", choices=["decode", "prompt"])
    ap.add_argument("--prompt-insitu", action="store_true",
                    help="prompt phase: sample the CC block inside real prompt steps (see measure())")
    ap.add_argument("--tokens", type=int, default=1,
                    help="decode: tokens per expert (batched decode); writes b200_decode_t<T>.json for T > 1")
    ap.add_argument("--cpu-tokens", type=int, default=32,
                    help="prompt phase: tokens per host CC sample (32: the per-expert solve_ng profile; "
                         "128, an expert's share of a 512-token prompt: the layer planner's)")
    ap.add_argument("--tag", default="", help="file tag suffix (b200_<phase><tag>.json)")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--load", default="concurrent", choices=["concurrent", "isolated"],
                    help="sample the host-side rates under each other's host-DRAM load (default) or alone")
    args = ap.parse_args(argv)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    samples = measure(args.phase, args.quick, args.load, args.tokens, args.prompt_insitu, args.cpu_tokens)
    tag = (args.phase if args.phase == "prompt" or args.tokens == 1 else f"{args.phase}_t{args.tokens}") + args.tag
    write_samples_csv(samples, out / f"b200_samples_{tag}.csv")
    prof, warns = fit_profile(samples, f"b200-{tag}" + ("" if args.load == "concurrent" else "-isolated"))
    (out / f"b200_{tag}.json").write_bytes(save_profile(prof))
    g = prof.gemm[Precision.FP16]
    summary = {
        "gpu_gemm_effective_GBps": 2.0 / g.gpu.beta / 1e9 if g.gpu.beta else None,
        "cpu_gemm_effective_GBps": 2.0 / g.cpu.beta / 1e9 if g.cpu.beta else None,
        "c2g_GBps": 1.0 / prof.pcie.beta / 1e9 if prof.pcie and prof.pcie.beta else None,
        "launch_us": prof.launch.alpha * 1e6 if prof.launch else None,
        "warnings": warns,
    }
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
