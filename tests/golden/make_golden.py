"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (``sliceplan``) from
/root/reference/pkg/src and writes

* ``forward_golden.npz``  -- sliced / dense forwards, block widths and
  execution tags of slicing_kernel.py on seeded small inputs (the oracle and
  the GPU path are both pinned to these), and
* ``planner_golden.json`` -- rate solver, memory assigner, token assigner,
  stage times, recurrences, simulator, fits and profile/CSV bytes over the
  Table I testbeds plus seeded log-uniform jitters of them (the conftest
  ``random_profile`` recipe, /root/reference/pkg/tests/conftest.py:47-63).
  Floats are stored with ``float.hex`` so the parity tests can demand ``==``.

Nothing at test / bench time reads /root/reference; only these files travel.
"""

from __future__ import annotations

import copy
import io
import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

import sliceplan as sp  # noqa: E402  (the reference)
from sliceplan import slicing_kernel as sk  # noqa: E402
from sliceplan.testbeds import ALL_TESTBEDS  # noqa: E402


def hx(v: float) -> str:
    return float(v).hex()


def jitter_doc(rng: np.random.Generator, base: dict) -> dict:
    doc = copy.deepcopy(base)

    def j(value: float) -> float:
        return value * float(10.0 ** rng.uniform(-1.0, 1.0))

    for prec in doc["gemm"].values():
        for side in ("gpu", "cpu"):
            prec[side]["alpha"] = j(prec[side]["alpha"])
            prec[side]["beta"] = j(prec[side]["beta"])
    doc["pcie"]["alpha"] = j(doc["pcie"]["alpha"])
    doc["pcie"]["beta"] = j(doc["pcie"]["beta"])
    doc["launch"]["alpha"] = j(doc["launch"]["alpha"])
    return doc


# ---------------------------------------------------------------------------
# forward goldens


def forward_golden() -> None:
    rng = np.random.default_rng(20241115)
    arrays: dict[str, np.ndarray] = {}
    cases = []
    acts = list(sk.Activation)
    fixed_rates = [(0.2, 0.3, 0.5), (1 / 3, 1 / 3, 1 / 3), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                   (0.0, 0.0, 1.0), (0.5, 0.5, 0.0), (0.0, 0.5, 0.5), (0.4999999999999999, 0.25, 0.2500000000000001)]
    for i in range(48):
        t = int(rng.integers(1, 9))
        m = int(rng.integers(2, 65))
        h = int(rng.integers(2, 97))
        o = int(rng.integers(2, 65))
        x = rng.uniform(-1.0, 1.0, (t, m))
        w1 = rng.uniform(-1.0, 1.0, (m, h))
        w2 = rng.uniform(-1.0, 1.0, (h, o))
        if i < len(fixed_rates):
            cc, cg, gg = fixed_rates[i]
        else:
            raw = rng.uniform(0.0, 1.0, 3)
            raw /= raw.sum()
            cc, cg, gg = raw[0], raw[1], 1.0 - raw[0] - raw[1]
        rates = sp.SlicingRates(cc=cc, cg=cg, gg=gg)
        act = acts[i % len(acts)]
        n_g = int(rng.integers(0, t + 1))
        sliced = sk.slice_weights(w1, w2, rates)
        key = f"c{i}"
        arrays[f"{key}_x"], arrays[f"{key}_w1"], arrays[f"{key}_w2"] = x, w1, w2
        arrays[f"{key}_dense"] = sk.mlp_forward_reference(x, w1, w2, act)
        arrays[f"{key}_sliced"] = sk.mlp_forward_sliced(x, sliced, act, n_g)
        tags = [[tk.block, tk.executor, tk.row_start, tk.row_stop]
                for tk in sk.execution_tags(sliced, t, n_g)]
        cases.append({
            "key": key, "act": act.value, "rates": [hx(rates.cc), hx(rates.cg), hx(rates.gg)],
            "n_g": n_g, "boundaries": list(sliced.boundaries), "widths": list(sliced.block_widths),
            "tags": tags,
        })
    # the config-1 split the survey measured: 1024 x 3584 at 0.2/0.3/0.5
    wide = sk.slice_weights(np.zeros((2, 3584)), np.zeros((3584, 2)), sp.SlicingRates(0.2, 0.3, 0.5))
    meta = {"cases": cases, "cfg1_widths": list(wide.block_widths),
            "recombination_seed123_trials50": hx(sk.max_recombination_error(seed=123, trials=50))}
    arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "forward_golden.npz", **arrays)


# ---------------------------------------------------------------------------
# planner goldens


LAYERS = [
    (4096, 14336, 2, "fp16"),
    (4096, 14336, 6, "fp16"),
    (1024, 3584, 4, "fp16"),
    (8192, 28672, 3, "int4"),
    (128, 256, 1, "fp16"),
]


def layer_of(spec) -> "sp.LayerSpec":
    m, h, n, p = spec
    return sp.LayerSpec(model_dim=m, hidden_dim=h, n_gemms=n, precision=sp.Precision(p))


def stage_hex(st) -> list[str]:
    return [hx(st.launch_s), hx(st.transfer_s), hx(st.gpu_s), hx(st.cpu_s)]


def planner_golden() -> None:
    rng = np.random.default_rng(31337)
    docs = [dict(d) for d in ALL_TESTBEDS.values()]
    bases = list(ALL_TESTBEDS.values())
    for i in range(24):
        docs.append(jitter_doc(rng, bases[i % 3]))
    out: dict = {"profiles": docs, "layers": LAYERS, "solve_rcg": [], "edge_points": [],
                 "stages": [], "recurrence": [], "solve_ng": [], "greedy": [], "grid": [],
                 "misc": [], "fits": [], "importance": []}
    decode = sp.Workload(tokens=1, phase=sp.Phase.GENERATION)
    gen4 = sp.Workload(tokens=4, phase=sp.Phase.GENERATION)
    for pi, doc in enumerate(docs):
        prof = sp.profile_from_dict(doc)
        for li, spec in enumerate(LAYERS):
            layer = layer_of(spec)
            for wl in (decode, gen4):
                for r_gg in (0.0, 0.25, 0.5, 0.9375, 1.0, float(rng.uniform(0, 1))):
                    sol = sp.solve_rcg(prof, layer, wl, r_gg)
                    out["solve_rcg"].append({
                        "p": pi, "l": li, "T": wl.tokens, "r_gg": hx(r_gg),
                        "rates": [hx(sol.rates.cc), hx(sol.rates.cg), hx(sol.rates.gg)],
                        "t_fin": hx(sol.t_fin),
                        "cands": [[hx(c), hx(t)] for c, t in sol.candidates],
                    })
                    if pi % 4 == 0:
                        out["edge_points"].append({"p": pi, "l": li, "T": wl.tokens, "r_gg": hx(r_gg),
                                                   "pts": [hx(v) for v in sp.edge_points(prof, layer, wl, r_gg)]})
            # stage times + recurrence + simulator on solver and fixed rates
            for rates in ((0.2, 0.3, 0.5), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0), (0.5, 0.5, 0.0)):
                r = sp.SlicingRates(*rates)
                st = sp.stage_times_generation(prof, layer, decode, r)
                rec = sp.evaluate_recurrence(st, layer.n_gemms)
                sim = sp.simulate_streams(st, layer.n_gemms)
                out["stages"].append({"p": pi, "l": li, "kind": "gen", "rates": [hx(v) for v in rates],
                                      "stage": stage_hex(st)})
                out["recurrence"].append({
                    "stage": stage_hex(st), "n": layer.n_gemms, "t_fin": hx(rec.t_fin),
                    "label": rec.case_label.value, "sim_t_fin": hx(sim.t_fin), "sim_label": sim.case_label.value,
                    "gpu_done": [hx(v) for v in rec.gpu_done], "cpu_done": [hx(v) for v in rec.cpu_done],
                    "records": [[d["gemm_index"], d["stream"], hx(d["start_s"]), hx(d["end_s"])]
                                for d in sp.timeline_records(st, rec)],
                })
                for tokens, n_g in ((64, 0), (64, 17), (257, 257), (512, 401)):
                    for tm in ("literal", "rate_scaled"):
                        stp = sp.stage_times_prompt(prof, layer, sp.Workload(tokens, sp.Phase.PROMPT), r, n_g, tm)
                        out["stages"].append({"p": pi, "l": li, "kind": "prompt", "rates": [hx(v) for v in rates],
                                              "T": tokens, "n_g": n_g, "tm": tm, "stage": stage_hex(stp)})
            # token assignment at decode-solved rates
            rates = sp.solve_rcg(prof, layer, decode, 0.0).rates
            for tokens in (1, 2, 64, 257, 512):
                for tm in ("literal", "rate_scaled"):
                    plan = sp.solve_ng(prof, layer, tokens, rates, tm)
                    out["solve_ng"].append({
                        "p": pi, "l": li, "T": tokens, "tm": tm,
                        "rates": [hx(rates.cc), hx(rates.cg), hx(rates.gg)],
                        "n_g": plan.n_g, "t": hx(plan.t_fin_prompt), "base": hx(plan.baseline_t_fin),
                        "cands": [[n, hx(t)] for n, t in plan.candidates],
                    })
            out["misc"].append({
                "p": pi, "l": li,
                "lipschitz": hx(sp.lipschitz_bound(prof, layer, decode)),
                "cc_result": hx(sp.cc_result_transfer_time(prof, layer, gen4, sp.SlicingRates(0.2, 0.3, 0.5))),
            })
            if pi % 6 == 0:
                cg, tf = sp.grid_scan(prof, layer, decode, 0.25, 257)
                g = sp.solve_rates_grid(prof, layer, decode, 0.25, 257)
                out["grid"].append({"p": pi, "l": li, "cg": [hx(v) for v in cg], "t": [hx(v) for v in tf],
                                    "rates": [hx(g.rates.cc), hx(g.rates.cg), hx(g.rates.gg)], "t_fin": hx(g.t_fin)})
                out["importance"].append({"p": pi, "l": li,
                                          "v": hx(sp.importance(prof, layer, decode, 0.25, 0.5))})
        # memory plans
        for layer_ids, budget_frac, steps in (([0, 0], 1.0, 4), ([0, 1, 2], 0.7, 16), ([2] * 8, 3.3, 16),
                                              ([0, 4, 1, 4], 0.0, 16), ([1, 0], 100.0, 8)):
            layers = [layer_of(LAYERS[i]) for i in layer_ids]
            budget = budget_frac * layers[0].layer_bytes
            plan = sp.greedy_assign(prof, layers, decode, budget, n_steps=steps)
            out["greedy"].append({
                "p": pi, "layers": layer_ids, "budget": hx(budget), "steps": steps,
                "rgg": [hx(v) for v in plan.per_layer_rgg], "used": hx(plan.bytes_used), "iters": plan.iterations,
                "trace": [[s.iteration, s.layer_index, hx(s.rgg), hx(s.importance)] for s in plan.trace],
            })
        # fits, serialisation
        if pi < 9:
            samples = sp.generate_samples(prof, points=9, noise=0.02 * (pi % 3), seed=pi)
            buf = io.StringIO()
            sp.write_samples_csv(samples, buf)
            fitted, warns = sp.fit_profile(samples, f"fit-{pi}")
            out["fits"].append({
                "p": pi, "csv": buf.getvalue(), "profile_json": sp.save_profile(fitted).decode(),
                "warnings": warns, "saved_input": sp.save_profile(prof).decode(),
            })
    (OUT / "planner_golden.json").write_text(json.dumps(out, separators=(",", ":")))


if __name__ == "__main__":
    assert os.environ.get("PYTHONDONTWRITEBYTECODE") == "1" or sys.dont_write_bytecode
    forward_golden()
    planner_golden()
    for name in ("forward_golden.npz", "planner_golden.json"):
        print(name, (OUT / name).stat().st_size, "bytes")
