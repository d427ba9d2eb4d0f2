"""Host-side logic of the operator API: the floor rule, the dispatch table and
the argument errors -- the reference's own test cases
(/root/reference/pkg/tests/test_slicing_kernel.py:20-50, 125-165) run against
this package.  None of these touch the GPU."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import sliced_forward as orc
from paper_2411_15715_b200 import (
    Activation,
    ShapeMismatch,
    SlicingRates,
    TokenCountOutOfRange,
    execution_tags,
    mlp_forward_reference,
    mlp_forward_sliced,
    slice_weights,
)


class TestSliceWeights:
    def test_all_cpu_takes_everything(self):
        w1, w2 = np.arange(12.0).reshape(3, 4), np.arange(8.0).reshape(4, 2)
        sliced = slice_weights(w1, w2, SlicingRates(1, 0, 0))
        assert sliced.block_widths == (4, 0, 0)
        assert np.array_equal(sliced.w1_blocks[0], w1) and np.array_equal(sliced.w2_blocks[0], w2)

    def test_widths_on_even_split(self):
        assert slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(0.5, 0.25, 0.25)).block_widths == (4, 2, 2)

    def test_floor_rule_sends_remainder_to_resident_block(self):
        s = slice_weights(np.zeros((4, 10)), np.zeros((10, 4)), SlicingRates(1 / 3, 1 / 3, 1 / 3))
        assert s.block_widths == (3, 3, 4)

    def test_config1_widths(self):
        s = slice_weights(np.zeros((2, 3584)), np.zeros((3584, 2)), SlicingRates(0.2, 0.3, 0.5))
        assert s.block_widths == (716, 1076, 1792)

    def test_block_heights_match_widths(self):
        s = slice_weights(np.zeros((6, 9)), np.zeros((9, 5)), SlicingRates(0.4, 0.4, 0.2))
        for a, b in zip(s.w1_blocks, s.w2_blocks):
            assert a.shape[1] == b.shape[0]

    def test_gated_blocks_follow_w1(self):
        s = slice_weights(np.zeros((6, 9)), np.zeros((9, 5)), SlicingRates(0.4, 0.4, 0.2), w3=np.ones((6, 9)))
        assert [b.shape for b in s.w3_blocks] == [b.shape for b in s.w1_blocks]

    def test_shape_mismatch(self):
        with pytest.raises(ShapeMismatch):
            slice_weights(np.zeros((3, 4)), np.zeros((5, 2)), SlicingRates(1, 0, 0))
        with pytest.raises(ShapeMismatch):
            slice_weights(np.zeros((3, 4)), np.zeros((4, 2)), SlicingRates(1, 0, 0), w3=np.zeros((3, 5)))

    @settings(max_examples=200, deadline=None)
    @given(h=st.integers(1, 20000), cc=st.floats(0, 1), frac=st.floats(0, 1))
    def test_floor_rule_equals_oracle(self, h, cc, frac):
        cg = (1.0 - cc) * frac
        rates = SlicingRates(cc, cg, 1.0 - cc - cg)
        s = slice_weights(np.zeros((1, h)), np.zeros((h, 1)), rates)
        assert s.boundaries == orc.boundaries(h, rates.cc, rates.cg)


class TestExecutionTags:
    def test_full_diversion_relabels_cpu_block(self):
        s = slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(1, 0, 0))
        tasks = execution_tags(s, tokens=4, n_g=4)
        assert [(t.block, t.executor, t.row_start, t.row_stop) for t in tasks] == [("cg_prime", "gpu", 0, 4)]

    def test_mixed_rates_tag_layout(self):
        s = slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(0.5, 0.25, 0.25))
        tasks = execution_tags(s, tokens=6, n_g=2)
        assert [(t.block, t.executor, t.row_start, t.row_stop) for t in tasks] == [
            ("cc", "cpu", 0, 4), ("cg_prime", "gpu", 4, 6), ("cg", "gpu", 0, 6), ("gg", "gpu", 0, 6)]

    def test_tag_range_checked(self):
        s = slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(1, 0, 0))
        with pytest.raises(TokenCountOutOfRange):
            execution_tags(s, tokens=4, n_g=5)

    @settings(max_examples=100, deadline=None)
    @given(h=st.integers(1, 64), cc=st.floats(0, 1), frac=st.floats(0, 1), t=st.integers(1, 40),
           data=st.data())
    def test_tags_equal_oracle(self, h, cc, frac, t, data):
        n_g = data.draw(st.integers(0, t))
        cg = (1.0 - cc) * frac
        rates = SlicingRates(cc, cg, 1.0 - cc - cg)
        s = slice_weights(np.zeros((1, h)), np.zeros((h, 1)), rates)
        got = [(k.block, k.executor, k.row_start, k.row_stop) for k in execution_tags(s, t, n_g)]
        assert got == orc.execution_tags(h, rates.cc, rates.cg, t, n_g)


class TestErrorsBeforeCompute:
    """Argument errors are raised before any device work (slicing_kernel.py:111-118)."""

    def test_forward_input_mismatch(self):
        s = slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(1, 0, 0))
        with pytest.raises(ShapeMismatch):
            mlp_forward_sliced(np.zeros((2, 5)), s, Activation.IDENTITY)

    def test_reference_mismatch(self):
        with pytest.raises(ShapeMismatch):
            mlp_forward_reference(np.zeros((2, 3)), np.zeros((4, 5)), np.zeros((5, 2)), Activation.IDENTITY)

    def test_ng_out_of_range(self):
        s = slice_weights(np.zeros((4, 8)), np.zeros((8, 4)), SlicingRates(1, 0, 0))
        with pytest.raises(TokenCountOutOfRange):
            mlp_forward_sliced(np.zeros((2, 4)), s, Activation.IDENTITY, n_g=3)
