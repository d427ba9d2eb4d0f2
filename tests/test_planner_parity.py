"""Partition API is bit-exact with the reference.

Fixtures in tests/golden/planner_golden.json were produced by the reference
itself (tests/golden/make_golden.py); every float is compared with ``==`` via
its hex form.  When /root/reference is present (the build container) a live
differential test also draws fresh random profiles and compares both packages
call by call.
"""

from __future__ import annotations

import io
import json
import sys

import numpy as np
import pytest

import paper_2411_15715_b200 as sp
from conftest import GOLDEN, REFERENCE_SRC, random_profile

G = json.loads((GOLDEN / "planner_golden.json").read_text())
PROFILES = [sp.profile_from_dict(d) for d in G["profiles"]]
DECODE = sp.Workload(tokens=1, phase=sp.Phase.GENERATION)


def fx(h: str) -> float:
    return float.fromhex(h)


def layer(i: int) -> sp.LayerSpec:
    m, h, n, p = G["layers"][i]
    return sp.LayerSpec(model_dim=m, hidden_dim=h, n_gemms=n, precision=sp.Precision(p))


def hexes(values) -> list[str]:
    return [float(v).hex() for v in values]


def test_solve_rcg_bit_exact():
    assert len(G["solve_rcg"]) > 1000
    for case in G["solve_rcg"]:
        wl = sp.Workload(tokens=case["T"], phase=sp.Phase.GENERATION)
        sol = sp.solve_rcg(PROFILES[case["p"]], layer(case["l"]), wl, fx(case["r_gg"]))
        assert hexes([sol.rates.cc, sol.rates.cg, sol.rates.gg]) == case["rates"], case
        assert sol.t_fin.hex() == case["t_fin"]
        assert [[c.hex(), t.hex()] for c, t in sol.candidates] == case["cands"]


def test_edge_points_bit_exact():
    for case in G["edge_points"]:
        wl = sp.Workload(tokens=case["T"], phase=sp.Phase.GENERATION)
        pts = sp.edge_points(PROFILES[case["p"]], layer(case["l"]), wl, fx(case["r_gg"]))
        assert hexes(pts) == case["pts"]


def test_stage_times_bit_exact():
    for case in G["stages"]:
        prof, lay = PROFILES[case["p"]], layer(case["l"])
        rates = sp.SlicingRates(*(fx(v) for v in case["rates"]))
        if case["kind"] == "gen":
            st = sp.stage_times_generation(prof, lay, DECODE, rates)
        else:
            wl = sp.Workload(case["T"], sp.Phase.PROMPT)
            st = sp.stage_times_prompt(prof, lay, wl, rates, case["n_g"], case["tm"])
        assert hexes([st.launch_s, st.transfer_s, st.gpu_s, st.cpu_s]) == case["stage"]


def test_recurrence_simulator_records_bit_exact():
    for case in G["recurrence"]:
        st = sp.StageTimes(*(fx(v) for v in case["stage"]))
        rec = sp.evaluate_recurrence(st, case["n"])
        sim = sp.simulate_streams(st, case["n"])
        assert rec.t_fin.hex() == case["t_fin"] and rec.case_label.value == case["label"]
        assert sim.t_fin.hex() == case["sim_t_fin"] and sim.case_label.value == case["sim_label"]
        assert hexes(rec.gpu_done) == case["gpu_done"] and hexes(rec.cpu_done) == case["cpu_done"]
        recs = [[r["gemm_index"], r["stream"], r["start_s"].hex(), r["end_s"].hex()]
                for r in sp.timeline_records(st, rec)]
        assert recs == case["records"]


def test_solve_ng_bit_exact():
    for case in G["solve_ng"]:
        rates = sp.SlicingRates(*(fx(v) for v in case["rates"]))
        plan = sp.solve_ng(PROFILES[case["p"]], layer(case["l"]), case["T"], rates, case["tm"])
        assert plan.n_g == case["n_g"]
        assert plan.t_fin_prompt.hex() == case["t"] and plan.baseline_t_fin.hex() == case["base"]
        assert [[n, t.hex()] for n, t in plan.candidates] == case["cands"]


def test_greedy_assign_bit_exact():
    for case in G["greedy"]:
        layers = [layer(i) for i in case["layers"]]
        plan = sp.greedy_assign(PROFILES[case["p"]], layers, DECODE, fx(case["budget"]), n_steps=case["steps"])
        assert hexes(plan.per_layer_rgg) == case["rgg"]
        assert plan.bytes_used.hex() == case["used"] and plan.iterations == case["iters"]
        assert [[s.iteration, s.layer_index, s.rgg.hex(), s.importance.hex()] for s in plan.trace] == case["trace"]


def test_grid_and_misc_bit_exact():
    for case in G["grid"]:
        cg, tf = sp.grid_scan(PROFILES[case["p"]], layer(case["l"]), DECODE, 0.25, 257)
        assert hexes(cg) == case["cg"] and hexes(tf) == case["t"]
        g = sp.solve_rates_grid(PROFILES[case["p"]], layer(case["l"]), DECODE, 0.25, 257)
        assert hexes([g.rates.cc, g.rates.cg, g.rates.gg]) == case["rates"] and g.t_fin.hex() == case["t_fin"]
    for case in G["importance"]:
        v = sp.importance(PROFILES[case["p"]], layer(case["l"]), DECODE, 0.25, 0.5)
        assert v.hex() == case["v"]
    gen4 = sp.Workload(tokens=4, phase=sp.Phase.GENERATION)
    for case in G["misc"]:
        prof, lay = PROFILES[case["p"]], layer(case["l"])
        assert sp.lipschitz_bound(prof, lay, DECODE).hex() == case["lipschitz"]
        got = sp.cc_result_transfer_time(prof, lay, gen4, sp.SlicingRates(0.2, 0.3, 0.5))
        assert got.hex() == case["cc_result"]


def test_fits_and_serialisation_byte_exact():
    for case in G["fits"]:
        prof = PROFILES[case["p"]]
        assert sp.save_profile(prof).decode() == case["saved_input"]
        samples = sp.generate_samples(prof, points=9, noise=0.02 * (case["p"] % 3), seed=case["p"])
        buf = io.StringIO()
        sp.write_samples_csv(samples, buf)
        assert buf.getvalue() == case["csv"]
        fitted, warns = sp.fit_profile(sp.read_samples_csv(io.StringIO(case["csv"])), f"fit-{case['p']}")
        assert sp.save_profile(fitted).decode() == case["profile_json"]
        assert warns == case["warnings"]


# ---------------------------------------------------------------------------
# live differential against the reference (build container only)


@pytest.fixture(scope="module")
def ref():
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted (GPU box / CI)")
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REFERENCE_SRC))
    import sliceplan

    return sliceplan


def test_live_differential_random_profiles(ref):
    rng = np.random.default_rng(99)
    for i in range(150):
        prof = random_profile(rng)
        rprof = ref.profile_from_dict(sp.profile_to_dict(prof))
        m = int(rng.choice([1024, 4096, 6144, 8192]))
        h = int(rng.choice([3584, 6400, 14336, 16384, 28672]))
        n = int(rng.integers(1, 9))
        p = "fp16" if i % 3 else "int4"
        ours = sp.LayerSpec(m, h, n, sp.Precision(p))
        theirs = ref.LayerSpec(m, h, n, ref.Precision(p))
        tokens = int(rng.integers(1, 33))
        wl, rwl = sp.Workload(tokens, sp.Phase.GENERATION), ref.Workload(tokens, ref.Phase.GENERATION)
        r_gg = float(rng.uniform(0, 1)) if i % 4 else 0.0
        a = sp.solve_rcg(prof, ours, wl, r_gg)
        b = ref.solve_rcg(rprof, theirs, rwl, r_gg)
        assert (a.rates.cc, a.rates.cg, a.rates.gg, a.t_fin) == (b.rates.cc, b.rates.cg, b.rates.gg, b.t_fin)
        assert a.candidates == b.candidates
        T = int(rng.integers(1, 700))
        for tm in ("literal", "rate_scaled"):
            pa = sp.solve_ng(prof, ours, T, a.rates, tm)
            pb = ref.solve_ng(rprof, theirs, T, ref.SlicingRates(b.rates.cc, b.rates.cg, b.rates.gg), tm)
            assert (pa.n_g, pa.t_fin_prompt, pa.baseline_t_fin) == (pb.n_g, pb.t_fin_prompt, pb.baseline_t_fin)
        if i % 10 == 0:
            layers = [ours] * int(rng.integers(1, 5))
            rlayers = [theirs] * len(layers)
            budget = float(rng.uniform(0, 2.5)) * ours.layer_bytes
            ga = sp.greedy_assign(prof, layers, wl, budget, n_steps=8)
            gb = ref.greedy_assign(rprof, rlayers, rwl, budget, n_steps=8)
            assert ga.per_layer_rgg == gb.per_layer_rgg and ga.bytes_used == gb.bytes_used
            assert [(s.layer_index, s.rgg, s.importance) for s in ga.trace] == \
                   [(s.layer_index, s.rgg, s.importance) for s in gb.trace]


def test_solve_ng_layer_extension_limits():
    """planner.solve_ng_layer (extension, no reference counterpart): a free host
    keeps every expert's rows on the host, a very slow host none; deterministic."""
    import copy

    from paper_2411_15715_b200 import costs

    base = costs.profile_to_dict(PROFILES[0]) if isinstance(PROFILES, list) else costs.profile_to_dict(
        next(iter(PROFILES.values())))
    layer_ = sp.LayerSpec(4096, 14336, n_gemms=3, precision=sp.Precision.FP16)
    rates = sp.SlicingRates(0.35, 0.15, 0.5)
    toks = [100, 120, 130, 140]
    fast, slow = copy.deepcopy(base), copy.deepcopy(base)
    for doc, k in ((fast, 1e-6), (slow, 1e6)):
        for g in doc["gemm"].values():
            g["cpu"]["alpha"] *= k
            g["cpu"]["beta"] *= k
    pf = sp.solve_ng_layer(costs.profile_from_dict(fast), layer_, toks, rates)
    ps = sp.solve_ng_layer(costs.profile_from_dict(slow), layer_, toks, rates)
    assert pf.n_g == (0, 0, 0, 0)
    assert ps.n_g == tuple(toks)
    again = sp.solve_ng_layer(costs.profile_from_dict(fast), layer_, toks, rates)
    assert again == pf


def test_prompt_layer_busy_matches_the_layer_plan():
    """planner.prompt_layer_busy (extension: the cost model the bench re-anchors
    the prompt profile with) reproduces solve_ng_layer's own link / host
    predictions for the plan it returns, and scales linearly in the CPU terms."""
    import copy

    from paper_2411_15715_b200 import costs

    base = costs.profile_to_dict(PROFILES[0]) if isinstance(PROFILES, list) else costs.profile_to_dict(
        next(iter(PROFILES.values())))
    layer_ = sp.LayerSpec(4096, 14336, n_gemms=3, precision=sp.Precision.FP16)
    rates = sp.SlicingRates(0.35, 0.15, 0.5)
    toks = [100, 120, 130, 140, 0, 90]
    prof = costs.profile_from_dict(base)
    plan = sp.solve_ng_layer(prof, layer_, toks, rates)
    lk, cp = sp.prompt_layer_busy(prof, layer_, toks, plan.n_g, rates)
    assert lk == plan.link_s and cp == plan.cpu_s
    half = copy.deepcopy(base)
    for g in half["gemm"].values():
        g["cpu"]["alpha"] *= 0.5
        g["cpu"]["beta"] *= 0.5
    _, cp2 = sp.prompt_layer_busy(costs.profile_from_dict(half), layer_, toks, plan.n_g, rates)
    assert abs(cp2 - 0.5 * cp) <= 1e-12 * max(1.0, cp)
