"""Pin the CPU oracle to the reference's own outputs before trusting it.

tests/golden/forward_golden.npz holds slicing_kernel.py's dense and sliced
forwards, block widths and execution tags on 48 seeded cases (made by
tests/golden/make_golden.py from the unmodified reference).  The oracle's G=2
path must reproduce them; the SwiGLU (G=3) and MoE extensions are then pinned
by reduction properties.
"""

from __future__ import annotations

import itertools
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sliced_forward as orc

NPZ = np.load(GOLDEN / "forward_golden.npz")
META = json.loads(bytes(NPZ["meta_json"]).decode())


@pytest.mark.parametrize("case", META["cases"], ids=lambda c: c["key"])
def test_oracle_matches_reference_goldens(case):
    k = case["key"]
    x, w1, w2 = NPZ[f"{k}_x"], NPZ[f"{k}_w1"], NPZ[f"{k}_w2"]
    cc, cg, _ = (float.fromhex(v) for v in case["rates"])
    assert list(orc.boundaries(w1.shape[1], cc, cg)) == case["boundaries"]
    assert list(orc.block_widths(w1.shape[1], cc, cg)) == case["widths"]
    dense = orc.dense_forward(x, w1, w2, case["act"])
    sliced = orc.sliced_forward(x, w1, w2, case["act"], cc, cg)
    # same numpy/BLAS arithmetic; allow last-ulp BLAS kernel differences across hosts
    np.testing.assert_allclose(dense, NPZ[f"{k}_dense"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sliced, NPZ[f"{k}_sliced"], rtol=0, atol=1e-12)
    tags = [list(t) for t in orc.execution_tags(w1.shape[1], cc, cg, x.shape[0], case["n_g"])]
    assert tags == case["tags"]


def test_cfg1_widths_pinned():
    assert META["cfg1_widths"] == [716, 1076, 1792]
    assert list(orc.block_widths(3584, 0.2, 0.3)) == [716, 1076, 1792]


def test_recombination_helper_pinned():
    assert float.fromhex(META["recombination_seed123_trials50"]) <= 1e-10


@pytest.mark.parametrize("act", orc.ACTIVATIONS)
def test_gated_sliced_equals_dense(act):
    rng = np.random.default_rng(5)
    for _ in range(20):
        t, m, h, n = (int(rng.integers(1, 9)), int(rng.integers(2, 40)), int(rng.integers(2, 90)),
                      int(rng.integers(2, 40)))
        x, w1, w3, w2 = (rng.uniform(-1, 1, s) for s in ((t, m), (m, h), (m, h), (h, n)))
        raw = rng.uniform(0, 1, 3)
        raw /= raw.sum()
        got = orc.sliced_forward(x, w1, w2, act, raw[0], raw[1], w3)
        ref = orc.dense_forward(x, w1, w2, act, w3)
        assert np.max(np.abs(got - ref)) <= 1e-10


def test_gated_reduces_to_plain_when_gate_branch_is_one():
    # x @ w3 == 1 for every column: a constant input feature carrying the gate
    rng = np.random.default_rng(6)
    x = np.concatenate([rng.uniform(-1, 1, (4, 7)), np.ones((4, 1))], axis=1)
    w1 = rng.uniform(-1, 1, (8, 30))
    w2 = rng.uniform(-1, 1, (30, 5))
    w3 = np.zeros((8, 30))
    w3[-1, :] = 1.0
    for act in orc.ACTIVATIONS:
        np.testing.assert_allclose(orc.dense_forward(x, w1, w2, act, w3),
                                   orc.dense_forward(x, w1, w2, act), rtol=0, atol=1e-13)


def test_block_permutation_invariance_gated():
    rng = np.random.default_rng(3)
    x, w1, w3, w2 = (rng.uniform(-1, 1, s) for s in ((5, 12), (12, 15), (12, 15), (15, 7)))
    b1, b2 = orc.boundaries(15, 0.4, 0.3)
    parts = [orc.segment_forward(x, w1, w2, "silu", lo, hi, w3) for lo, hi in ((0, b1), (b1, b2), (b2, 15))]
    totals = [sum(parts[i] for i in order) for order in itertools.permutations(range(3))]
    for tot in totals[1:]:
        assert np.max(np.abs(tot - totals[0])) <= 1e-12


def test_moe_single_expert_is_dense():
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (6, 10))
    w1, w3, w2 = rng.uniform(-1, 1, (10, 20)), rng.uniform(-1, 1, (10, 20)), rng.uniform(-1, 1, (20, 9))
    router = rng.uniform(-1, 1, (10, 1))
    got = orc.moe_forward(x, [(w1, w3, w2)], router, k=1)
    np.testing.assert_allclose(got, orc.dense_forward(x, w1, w2, "silu", w3), rtol=0, atol=1e-12)


def test_moe_routing_and_sliced_experts():
    rng = np.random.default_rng(9)
    E, k = 8, 2
    x = rng.uniform(-1, 1, (5, 16))
    experts = [(rng.uniform(-1, 1, (16, 24)), rng.uniform(-1, 1, (16, 24)), rng.uniform(-1, 1, (24, 16)))
               for _ in range(E)]
    router = rng.uniform(-1, 1, (16, E))
    ids, gates = orc.route_topk(x @ router, k)
    assert ids.shape == (5, 2) and np.allclose(gates.sum(axis=1), 1.0)
    assert np.all((x @ router)[np.arange(5), ids[:, 0]] >= (x @ router)[np.arange(5), ids[:, 1]])
    dense = orc.moe_forward(x, experts, router, k)
    rates = [tuple(rng.dirichlet(np.ones(3))[:2]) for _ in range(E)]
    sliced = orc.moe_forward(x, experts, router, k, rates=rates)
    assert np.max(np.abs(dense - sliced)) <= 1e-10


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    a = np.random.default_rng(1).standard_normal(10000) * 10
    ours = orc.bf16_round(a)
    theirs = torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)
    assert np.array_equal(ours, theirs)
