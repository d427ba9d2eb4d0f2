"""The C-ABI library: loads without a GPU, exports what include/sliced.h
declares, maps status codes to the reference exception classes, and its CC
host kernel (the only compute it may run without a device) matches the oracle."""

from __future__ import annotations

import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, gpu_available
from oracle import sliced_forward as orc
from paper_2411_15715_b200 import _native as nat
from paper_2411_15715_b200 import errors

HEADER = (ROOT / "include" / "sliced.h").read_text()


def declared_functions() -> set[str]:
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(sp_\w+)\s*\(", HEADER, re.M))


def test_library_loads_and_exports_every_declared_symbol():
    lib = nat.lib()
    declared = declared_functions()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(nat.LIB_PATH)], capture_output=True, text=True)
    exported = set(re.findall(r" T (sp_\w+)", out.stdout))
    assert declared <= exported
    assert set(nat.SIGNATURES) == declared


def test_abi_version_and_struct_layouts():
    assert nat.lib().sp_abi_version() == int(re.search(r"SP_ABI_VERSION (\d+)", HEADER).group(1))
    assert C.sizeof(nat.LayerDesc) == 3 * 8 + 4 * 4 + 2 * 8
    assert C.sizeof(nat.Call) == 5 * 8
    assert C.sizeof(nat.TraceRecord) == 4 * 4 + 4 * 8


def test_status_codes_map_to_reference_classes():
    codes = dict(re.findall(r"SP_(ERR_\w+|OK) = (\d+)", HEADER))
    assert int(codes["ERR_SHAPE"]) == errors.SP_ERR_SHAPE and int(codes["ERR_TOKENS"]) == errors.SP_ERR_TOKENS
    assert errors.SP_ERR_SHAPE == 1 and errors.SP_ERR_TOKENS == 2
    with pytest.raises(errors.ShapeMismatch):
        errors.raise_for(errors.SP_ERR_SHAPE, "x")
    with pytest.raises(errors.TokenCountOutOfRange):
        errors.raise_for(errors.SP_ERR_TOKENS, "x")
    with pytest.raises(ValueError):
        errors.raise_for(errors.SP_ERR_VALUE, "x")
    assert issubclass(errors.ShapeMismatch, ValueError)


def host_has_amx() -> bool:
    try:
        return "amx_bf16" in open("/proc/cpuinfo").read()
    except OSError:
        return False


@pytest.fixture(scope="module")
def host_ctx():
    if gpu_available():
        pytest.skip("host-only context is for GPU-less hosts")
    nat.init(-1, 4)
    yield
    nat.shutdown()


def test_gpu_entry_points_refuse_without_device(host_ctx):
    from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls

    rng = np.random.default_rng(0)
    lay = NativeLayer(rng.standard_normal((32, 16)), rng.standard_normal((32, 8)), 32, 32, "silu", dtype="f32")
    with pytest.raises(errors.NativeError, match="no CPU fallback"):
        forward_calls([CallSpec(lay)], rng.standard_normal((2, 16)))
    # a GG block cannot be placed without a device
    with pytest.raises(errors.NativeError):
        NativeLayer(rng.standard_normal((32, 16)), rng.standard_normal((32, 8)), 0, 0, "silu", dtype="f32")


def test_layer_create_validates_like_the_reference(host_ctx):
    from paper_2411_15715_b200.sliced import NativeLayer

    rng = np.random.default_rng(1)
    with pytest.raises(errors.ShapeMismatch):
        NativeLayer(rng.standard_normal((32, 16)), rng.standard_normal((31, 8)), 32, 32, dtype="f32")
    with pytest.raises(ValueError):
        NativeLayer(rng.standard_normal((32, 16)), rng.standard_normal((32, 8)), 20, 10, dtype="f32")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("gated", [False, True])
@pytest.mark.parametrize("act", ["identity", "silu", "gelu"])
def test_cc_host_kernel_matches_oracle(host_ctx, dtype, gated, act):
    from paper_2411_15715_b200.sliced import NativeLayer

    rng = np.random.default_rng([len(dtype), int(gated), len(act)])
    for M, H, N, T, chunk in ((64, 200, 48, 5, 64), (100, 130, 20, 1, 64), (37, 300, 33, 9, 128),
                             (100, 700, 52, 33, 128)):
        w1, w3 = rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (M, H))
        w2, x = rng.uniform(-1, 1, (H, N)), rng.uniform(-1, 1, (T, M))
        lay = NativeLayer(w1.T, w2, H, H, act, w3.T if gated else None, dtype=dtype, chunk_rows=chunk)
        got = lay.cc_forward_host(x, threads=3)
        q = orc.bf16_round if dtype == "bf16" else (lambda a: a)
        ref = orc.dense_forward(q(x), q(w1), q(w2), act, q(w3) if gated else None)
        if dtype == "bf16" and T >= 4 and host_has_amx():
            # AMX tile path: the hidden activation is rounded to bf16 (as on the GPU tensor
            # cores); fp32 vs fp64 pre-activations can land on opposite sides of a bf16
            # rounding boundary, a one-ulp (2^-8) flip of single hidden units
            ref_h = orc.dense_forward_bf16_hidden(q(x), q(w1), q(w2), act, q(w3) if gated else None)
            assert orc.max_rel_error(got, ref_h) <= 5e-4
            assert orc.max_rel_error(got, ref) <= 5e-3
            continue
        assert orc.max_rel_error(got, ref) <= 1e-5
        assert lay.block_widths == (H, 0, 0)
        assert lay.placed_bytes()["gg"] == 0 and lay.placed_bytes()["cc"] > 0


def test_moe_router_matches_oracle():
    """sp_moe_route (fp64 logits, top-k ties -> lower id, softmax over k) vs the oracle."""
    from paper_2411_15715_b200.sliced import moe_route, to_bf16_bits

    rng = np.random.default_rng(4)
    for T, M, E, k in ((1, 4096, 8, 2), (7, 64, 16, 2), (5, 32, 8, 1), (3, 48, 4, 4)):
        x = rng.standard_normal((T, M)).astype(np.float32)
        router = rng.standard_normal((M, E)).astype(np.float32)
        ids, gates = moe_route(x, router, k)
        ref_ids, ref_g = orc.route_topk(x.astype(np.float64) @ router.astype(np.float64), k)
        assert np.array_equal(ids, ref_ids)
        np.testing.assert_allclose(gates, ref_g, rtol=1e-6)
        xb = to_bf16_bits(x)
        ids_b, _ = moe_route(xb, router, k)
        ref_b, _ = orc.route_topk(orc.bf16_round(x) @ router.astype(np.float64), k)
        assert np.array_equal(ids_b, ref_b)
    # exact ties go to the lower expert id
    ids, gates = moe_route(np.ones((1, 4), np.float32), np.ones((4, 6), np.float32), 2)
    assert ids.tolist() == [[0, 1]] and np.allclose(gates, 0.5)


def test_native_bf16_cast_matches_numpy_rule():
    """sp_round_bf16 (host activation cast) == the integer RNE rule, bit for bit."""
    from paper_2411_15715_b200.sliced import to_bf16_bits

    rng = np.random.default_rng(9)
    x = (rng.standard_normal(70001) * rng.choice([1e-40, 1e-3, 1.0, 1e30], 70001)).astype(np.float32)
    x[:6] = [1.00390625, 1.01171875, -3.0e38, 0.0, np.inf, -np.inf]
    u = x.view(np.uint32).astype(np.uint64)
    ref = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(to_bf16_bits(x), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("gated", [True, False])
def test_amx_cc_kernel_on_the_gpu_box(gated):
    """The AMX tile kernel (host_cc_amx.cpp) runs every prompt-row CC block on
    the GPU box; checked directly here (the host-only fixture above skips when a
    GPU is present).  Rows >= 4 take the AMX path; a bf16 hidden activation as
    on the tensor cores.  Also through a whole forward (CC block only, host
    threads) at Mixtral-like widths."""
    from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls

    if not host_has_amx():
        pytest.skip("this host has no AMX (amx_bf16)")
    nat.init(0)
    rng = np.random.default_rng(31 + gated)
    q = orc.bf16_round
    for M, H, N, T in ((256, 640, 192, 4), (512, 1000, 256, 16), (1024, 2048, 1024, 33), (4096, 1024, 4096, 64)):
        w1, w3 = rng.uniform(-1, 1, (M, H)) / 8, rng.uniform(-1, 1, (M, H)) / 8
        w2, x = rng.uniform(-1, 1, (H, N)) / 8, rng.uniform(-1, 1, (T, M))
        lay = NativeLayer(w1.T, w2, H, H, "silu", w3.T if gated else None, dtype="bf16", chunk_rows=128)
        ref_h = orc.dense_forward_bf16_hidden(q(x), q(w1), q(w2), "silu", q(w3) if gated else None)
        ref = orc.dense_forward(q(x), q(w1), q(w2), "silu", q(w3) if gated else None)
        got = lay.cc_forward_host(x, threads=0)
        assert orc.max_rel_error(got, ref_h) <= 5e-4, (M, H, N, T)
        assert orc.max_rel_error(got, ref) <= 1e-2, (M, H, N, T)
        y = forward_calls([CallSpec(lay)], x.astype(np.float32))  # CC block on the pool inside a forward
        assert orc.max_rel_error(np.asarray(y), ref) <= 1e-2, (M, H, N, T)
        lay.release()
