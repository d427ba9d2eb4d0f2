"""Edge cases of the sliced path that the reference handles
(/root/reference/pkg/src/sliceplan/slicing_kernel.py:97-158): empty token
batches, degenerate splits, tiny dimensions, and the runtime's documented
limits (include/sliced.h "Limits"), which must fail before any work."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available
from oracle import sliced_forward as orc
from paper_2411_15715_b200 import _native as nat
from paper_2411_15715_b200 import errors

FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def ctx():
    """The device context on a GPU box, a host-only context elsewhere."""
    if gpu_available():
        nat.init(0)
        yield "gpu"
    else:
        nat.init(-1, 2)
        yield "host"
        nat.shutdown()


def test_execution_tags_for_an_empty_batch_match_the_reference():
    """tokens = 0: the reference still lists the CG and GG tasks with empty row
    ranges and no CC task (slicing_kernel.py:146-158)."""
    import paper_2411_15715_b200 as sp

    rng = np.random.default_rng(0)
    s = sp.slice_weights(rng.uniform(-1, 1, (6, 20)), rng.uniform(-1, 1, (20, 3)), sp.SlicingRates(0.25, 0.25, 0.5))
    tags = [(t.block, t.executor, t.row_start, t.row_stop) for t in sp.execution_tags(s, 0, 0)]
    assert tags == [("cg", "gpu", 0, 0), ("gg", "gpu", 0, 0)]
    assert [t[:4] for t in orc.execution_tags(20, 0.25, 0.25, 0, 0)] == tags


@pytest.mark.parametrize("N,dtype,ok", [(8192, "bf16", True), (8193, "bf16", False), (4096, "f32", True),
                                        (4097, "f32", False)])
def test_out_dim_limit_is_refused_at_creation(ctx, N, dtype, ok):
    from paper_2411_15715_b200.sliced import NativeLayer

    rng = np.random.default_rng(1)
    w1t = rng.standard_normal((64, 32)).astype(np.float32)
    w2 = rng.standard_normal((64, N)).astype(np.float32)
    if ok:
        NativeLayer(w1t, w2, 64, 64, "silu", dtype=dtype).release()  # host-only blocks: runs without a GPU
    else:
        with pytest.raises(ValueError, match="out_dim"):
            NativeLayer(w1t, w2, 64, 64, "silu", dtype=dtype)


def test_model_dim_limit_is_refused_at_creation(ctx):
    from paper_2411_15715_b200.sliced import NativeLayer

    rng = np.random.default_rng(2)
    with pytest.raises(ValueError, match="model_dim"):
        NativeLayer(rng.standard_normal((2, 16385)), rng.standard_normal((2, 8)), 2, 2, "silu", dtype="f32")


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_empty_batch_returns_an_empty_output(ctx, on_device):
    """x of shape (0, M): the reference returns zeros((0, N)); so does the
    sliced forward, on the host and on the device, without touching the GPU."""
    import torch

    import paper_2411_15715_b200 as sp

    rng = np.random.default_rng(3)
    s = sp.slice_weights(rng.uniform(-1, 1, (12, 40)), rng.uniform(-1, 1, (40, 5)), sp.SlicingRates(0.3, 0.3, 0.4))
    launches = nat.stats()["kernel_launches"]
    if on_device:
        y = sp.mlp_forward_sliced(torch.zeros((0, 12), device="cuda"), s, sp.Activation.SILU)
        assert tuple(y.shape) == (0, 5) and y.is_cuda
    else:
        y = sp.mlp_forward_sliced(np.zeros((0, 12)), s, sp.Activation.SILU)
        assert y.shape == (0, 5) and y.dtype == np.float64
    assert nat.stats()["kernel_launches"] == launches


@pytest.mark.gpu
def test_empty_moe_batch(ctx):
    from paper_2411_15715_b200.sliced import MoEDispatch, NativeLayer

    rng = np.random.default_rng(4)
    lays = [NativeLayer(rng.standard_normal((64, 32)) / 8, rng.standard_normal((64, 16)) / 8, 16, 32, "silu",
                        rng.standard_normal((64, 32)) / 8, dtype="bf16") for _ in range(4)]
    d = MoEDispatch(lays, rng.standard_normal((32, 4)), 2)
    assert d(np.zeros((0, 32), dtype=np.float32)).shape == (0, 16)
    for l in lays:
        l.release()


@pytest.mark.gpu
@pytest.mark.parametrize("M,H,N", [(1, 1, 1), (1, 7, 3), (5, 1, 2), (3, 2, 1)])
@pytest.mark.parametrize("rates", [(0.0, 0.0, 1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.5, 0.5, 0.0)])
def test_tiny_dimensions_every_block(ctx, M, H, N, rates):
    """Single hidden unit / feature / output: the floor rule leaves whole
    blocks empty, and everything still matches the oracle at fp32."""
    import paper_2411_15715_b200 as sp

    rng = np.random.default_rng(M * 100 + H * 10 + N)
    x, w1, w2 = rng.uniform(-1, 1, (3, M)), rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (H, N))
    s = sp.slice_weights(w1, w2, sp.SlicingRates(*rates))
    for act in sp.Activation:
        for n_g in (0, 2, 3):
            got = sp.mlp_forward_sliced(x, s, act, n_g)
            ref = orc.sliced_forward(x, w1, w2, act.value, rates[0], rates[1])
            assert orc.max_rel_error(got, ref) <= FP32_TOL, (act, n_g)


@pytest.mark.gpu
def test_too_many_calls_fail_before_any_work(ctx):
    from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls

    rng = np.random.default_rng(5)
    lay = NativeLayer(rng.standard_normal((64, 16)), rng.standard_normal((64, 8)), 16, 32, "silu", dtype="f32")
    launches = nat.stats()["kernel_launches"]
    with pytest.raises(ValueError, match="n_calls"):
        forward_calls([CallSpec(lay)] * 33, rng.standard_normal((2, 16)))
    with pytest.raises(errors.ShapeMismatch):
        forward_calls([CallSpec(lay, token_ids=[0, 5])], rng.standard_normal((2, 16)))
    with pytest.raises(errors.TokenCountOutOfRange):
        forward_calls([CallSpec(lay, n_g=3)], rng.standard_normal((2, 16)))
    assert nat.stats()["kernel_launches"] == launches
    lay.release()
