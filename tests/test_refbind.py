"""The reference-side binding (``paper_2411_15715_b200/refbind.py``, the module
INTEGRATION.md tells a maintainer to add as ``sliceplan/_b200.py``) driven
through a stand-in of the reference's operator API.

The stand-in restates ``SlicedWeights`` and ``slice_weights``
(/root/reference/pkg/src/sliceplan/slicing_kernel.py:41-80) verbatim in
behaviour: a frozen dataclass of column / row VIEWS of the caller's arrays.
``refbind.mlp_forward_sliced`` has the signature of ``slicing_kernel.py:97-124``;
the goldens it is held to were produced by the unmodified reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ast
import gc
import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sliced_forward as orc
from paper_2411_15715_b200 import refbind
from paper_2411_15715_b200.errors import ShapeMismatch, TokenCountOutOfRange

FP32_TOL = 1e-5


@dataclass(frozen=True)
class StandInRates:
    cc: float
    cg: float
    gg: float


@dataclass(frozen=True)
class StandInSlicedWeights:  # slicing_kernel.py:41-54
    w1_blocks: tuple
    w2_blocks: tuple
    rates: StandInRates
    boundaries: tuple

    @property
    def block_widths(self):
        b1, b2 = self.boundaries
        h = sum(b.shape[1] for b in self.w1_blocks)
        return (b1, b2 - b1, h - b2)


def standin_slice_weights(w1, w2, rates):  # slicing_kernel.py:57-80
    w1 = np.asarray(w1, dtype=float)
    w2 = np.asarray(w2, dtype=float)
    hidden = w1.shape[1]
    b1 = min(int(math.floor(rates.cc * hidden)), hidden)
    b2 = min(max(int(math.floor((rates.cc + rates.cg) * hidden)), b1), hidden)
    return StandInSlicedWeights((w1[:, :b1], w1[:, b1:b2], w1[:, b2:]),
                                (w2[:b1, :], w2[b1:b2, :], w2[b2:, :]), rates, (b1, b2))


def test_binding_imports_only_numpy_ctypes_and_errors():
    """Droppable into the reference package: no import of this package except
    the exception module both packages define."""
    tree = ast.parse(Path(refbind.__file__).read_text())
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods |= {a.name.split(".")[0] for a in node.names}
        elif isinstance(node, ast.ImportFrom):
            mods.add(("." * node.level) + (node.module or "") if node.level else node.module.split(".")[0])
    assert mods <= {"__future__", "ctypes", "math", "os", "threading", "weakref", "pathlib", "numpy", "scipy",
                    ".errors"}, mods


def test_argument_errors_before_any_device_work():
    """slicing_kernel.py:110-118: validation happens before the forward, so it
    raises the reference's classes even where no device exists."""
    rng = np.random.default_rng(0)
    s = standin_slice_weights(rng.uniform(-1, 1, (6, 10)), rng.uniform(-1, 1, (10, 4)),
                              StandInRates(0.2, 0.3, 0.5))
    with pytest.raises(ShapeMismatch):
        refbind.mlp_forward_sliced(np.zeros((2, 5)), s, "identity")
    with pytest.raises(ShapeMismatch):
        refbind.mlp_forward_sliced(np.zeros(6), s, "identity")
    with pytest.raises(TokenCountOutOfRange):
        refbind.mlp_forward_sliced(np.zeros((2, 6)), s, "identity", n_g=3)
    with pytest.raises(TokenCountOutOfRange):
        refbind.mlp_forward_sliced(np.zeros((2, 6)), s, "identity", n_g=-1)
    assert issubclass(ShapeMismatch, ValueError) and issubclass(TokenCountOutOfRange, ValueError)


@pytest.mark.gpu
def test_refbind_matches_reference_goldens():
    npz = np.load(GOLDEN / "forward_golden.npz")
    meta = json.loads(bytes(npz["meta_json"]).decode())
    for case in meta["cases"]:
        k = case["key"]
        x, w1, w2 = npz[f"{k}_x"], npz[f"{k}_w1"], npz[f"{k}_w2"]
        rates = StandInRates(*(float.fromhex(v) for v in case["rates"]))
        s = standin_slice_weights(w1, w2, rates)
        assert list(s.block_widths) == case["widths"]
        got = refbind.mlp_forward_sliced(x, s, case["act"], case["n_g"])
        assert got.dtype == np.float64 and got.shape == npz[f"{k}_sliced"].shape
        assert orc.max_rel_error(got, npz[f"{k}_sliced"]) <= FP32_TOL, k
        refbind.release(s)
    assert refbind.placed_count() == 0


@pytest.mark.gpu
def test_refbind_places_once_and_frees_on_gc():
    import enum

    class Activation(enum.Enum):  # slicing_kernel.py:27-30
        IDENTITY = "identity"
        SILU = "silu"
        GELU = "gelu"

    rng = np.random.default_rng(7)
    M, H, N = 96, 700, 80
    w1, w2 = rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (H, N))
    s = standin_slice_weights(w1, w2, StandInRates(0.25, 0.35, 0.4))
    base = refbind.placed_count()
    for t in (1, 3, 8):
        for act in Activation:
            x = rng.uniform(-1, 1, (t, M))
            n_g = int(rng.integers(0, t + 1))
            got = refbind.mlp_forward_sliced(x, s, act, n_g)
            ref = orc.sliced_forward(x, w1, w2, act.value, 0.25, 0.35)
            assert orc.max_rel_error(got, ref) <= FP32_TOL
    assert refbind.placed_count() == base + 3  # one placement per activation, reused across calls
    del s
    gc.collect()
    assert refbind.placed_count() == base
    # empty token batch: same shape contract as the reference
    s2 = standin_slice_weights(w1, w2, StandInRates(0.0, 0.0, 1.0))
    assert refbind.mlp_forward_sliced(np.zeros((0, M)), s2, Activation.SILU).shape == (0, N)


@pytest.mark.gpu
def test_reference_cc_executor_runs_the_cc_block_through_numpy():
    """use_reference_cc: the CC block is the reference's own fp64 numpy
    expression, run by the library's coordinator thread next to the GPU work;
    the result still matches the reference goldens, and the native CC kernels
    are back once it is switched off."""
    from paper_2411_15715_b200 import _native as nat

    npz = np.load(GOLDEN / "forward_golden.npz")
    meta = json.loads(bytes(npz["meta_json"]).decode())
    calls = []
    orig = refbind._reference_cc

    def counting(*a):
        calls.append(a[4])  # rows
        return orig(*a)

    refbind._reference_cc = counting
    try:
        refbind.use_reference_cc(True)
        n_cc = 0
        for case in meta["cases"]:
            k = case["key"]
            x, w1, w2 = npz[f"{k}_x"], npz[f"{k}_w1"], npz[f"{k}_w2"]
            s = standin_slice_weights(w1, w2, StandInRates(*(float.fromhex(v) for v in case["rates"])))
            got = refbind.mlp_forward_sliced(x, s, case["act"], case["n_g"])
            assert orc.max_rel_error(got, npz[f"{k}_sliced"]) <= FP32_TOL, k
            if s.block_widths[0] > 0 and x.shape[0] - case["n_g"] > 0:
                n_cc += 1
            refbind.release(s)
        assert len(calls) == n_cc > 0
    finally:
        refbind.use_reference_cc(False)
        refbind._reference_cc = orig
    before = len(calls)
    rng = np.random.default_rng(3)
    s = standin_slice_weights(rng.uniform(-1, 1, (32, 200)), rng.uniform(-1, 1, (200, 16)), StandInRates(0.5, 0.2, 0.3))
    refbind.mlp_forward_sliced(rng.uniform(-1, 1, (2, 32)), s, "silu")
    assert len(calls) == before  # native CC again
    assert nat.lib().sp_abi_version() >= 4
