"""Sliced weight store, re-slicing and checkpoint loading.

CPU tests run in a host-only context (CC / CG blocks only: no GG block without
a device); the GPU tests round-trip layers with all three blocks."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import gpu_available
from oracle import sliced_forward as orc
from paper_2411_15715_b200 import _native as nat
from paper_2411_15715_b200 import store
from paper_2411_15715_b200.schedule import SlicingRates
from paper_2411_15715_b200.sliced import NativeLayer, to_bf16_bits


@pytest.fixture(scope="module")
def host_ctx():
    if gpu_available():
        pytest.skip("host-only context is for GPU-less hosts")
    nat.init(-1, 4)
    yield
    nat.shutdown()


def _weights(rng, M, H, N):
    return (rng.uniform(-1, 1, (H, M)) / 8, rng.uniform(-1, 1, (H, M)) / 8, rng.uniform(-1, 1, (H, N)))


def test_safetensors_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    t = {"a.bf16": to_bf16_bits(rng.standard_normal((7, 5))), "b.f32": rng.standard_normal((3, 4)).astype(np.float32),
         "c.i64": np.arange(6, dtype=np.int64).reshape(2, 3)}
    p = tmp_path / "t.safetensors"
    store.save_safetensors(p, t, {"a.bf16": "BF16"})
    h = store.read_safetensors_header(p)
    assert h["a.bf16"]["dtype"] == "BF16" and h["a.bf16"]["shape"] == [7, 5]
    back = store.load_safetensors(p)
    for k in t:
        assert back[k].dtype == t[k].dtype and np.array_equal(back[k], t[k])
    assert set(store.load_safetensors(p, ["b.f32"])) == {"b.f32"}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_store_round_trip_host_blocks(host_ctx, tmp_path, dtype):
    rng = np.random.default_rng(1)
    M, H, N = 96, 300, 40
    w1t, w3t, w2 = _weights(rng, M, H, N)
    layers = {"cc_only": NativeLayer(w1t, w2, H, H, "silu", w3t, dtype=dtype, chunk_rows=64),
              "cc_cg": NativeLayer(w1t, w2, 110, H, "gelu", None, dtype=dtype)}
    p = tmp_path / "layers.spstore"
    header = store.save_store(p, layers)
    assert store.read_store_header(p) == json.loads(json.dumps(header))
    back = store.load_store(p)
    x = rng.uniform(-1, 1, (3, M))
    for name, lay in layers.items():
        b = back[name]
        assert b.meta() == lay.meta() and b.block_widths == lay.block_widths
        g0, h0 = lay.export_images()
        g1, h1 = b.export_images()
        assert np.array_equal(g0, g1) and np.array_equal(h0, h1)
        assert np.array_equal(b.cc_forward_host(x, threads=2), lay.cc_forward_host(x, threads=2))
    # images through memory too
    lay = layers["cc_cg"]
    again = NativeLayer.from_images(lay.meta(), *lay.export_images())
    assert np.array_equal(again.cc_forward_host(x, threads=2), lay.cc_forward_host(x, threads=2))


def test_store_rejects_mismatched_images(host_ctx, tmp_path):
    rng = np.random.default_rng(2)
    w1t, w3t, w2 = _weights(rng, 64, 128, 32)
    lay = NativeLayer(w1t, w2, 128, 128, "silu", w3t, dtype="f32", chunk_rows=64)
    gg, host = lay.export_images()
    with pytest.raises(Exception, match="image sizes"):
        NativeLayer.from_images(lay.meta(), gg, host[:-4096])
    with pytest.raises(ValueError, match="not a sliced store"):
        p = tmp_path / "bad"
        p.write_bytes(b"x" * 64)
        store.load_store(p)


def test_reslice_host_blocks_matches_oracle(host_ctx):
    rng = np.random.default_rng(3)
    M, H, N = 80, 257, 36
    w1t, w3t, w2 = _weights(rng, M, H, N)
    lay = NativeLayer(w1t, w2, H, H, "silu", w3t, dtype="f32", chunk_rows=64)
    x = rng.uniform(-1, 1, (2, M))
    for b1 in (0, 1, 100, 256, H):
        r = lay.reslice(b1, H)
        assert r.block_widths == (b1, H - b1, 0)
        got = r.cc_forward_host(x, threads=3)
        ref = orc.segment_forward(x, w1t.T, w2, "silu", 0, b1, w3t.T)
        assert orc.max_rel_error(got, ref) <= 1e-5 if b1 else np.all(got == 0)
    with pytest.raises(ValueError):
        lay.reslice(10, 5)


def _mixtral_checkpoint(tmp_path, rng, E=3, M=64, H=192, layer=1):
    names = store.mixtral_moe_names(layer, E)
    tensors, dtypes, ref = {}, {}, []
    gate = rng.standard_normal((E, M)).astype(np.float32)
    tensors[names["gate"]] = gate
    for e, nm in enumerate(names["experts"]):
        w1, w3, w2 = rng.uniform(-1, 1, (H, M)) / 8, rng.uniform(-1, 1, (H, M)) / 8, rng.uniform(-1, 1, (M, H))
        for k, a in (("w1", w1), ("w3", w3), ("w2", w2)):
            tensors[nm[k]] = to_bf16_bits(a)
            dtypes[nm[k]] = "BF16"
        ref.append(tuple(orc.bf16_round(a) for a in (w1, w3, w2)))
    # two shards + index, as HF writes them
    keys = list(tensors)
    shards = {"model-00001-of-00002.safetensors": keys[: len(keys) // 2],
              "model-00002-of-00002.safetensors": keys[len(keys) // 2:]}
    for f, ks in shards.items():
        store.save_safetensors(tmp_path / f, {k: tensors[k] for k in ks}, {k: dtypes[k] for k in ks if k in dtypes})
    (tmp_path / "model.safetensors.index.json").write_text(
        json.dumps({"metadata": {}, "weight_map": {k: f for f, ks in shards.items() for k in ks}}))
    return gate, ref


def test_load_mixtral_layer_from_sharded_safetensors(host_ctx, tmp_path):
    rng = np.random.default_rng(4)
    gate, ref = _mixtral_checkpoint(tmp_path, rng)
    experts, router = store.load_mixtral_moe(tmp_path, 1, 3, SlicingRates(1.0, 0.0, 0.0), chunk_rows=64)
    assert router.shape == (64, 3) and np.array_equal(router, gate.T.astype(np.float64))
    x = rng.uniform(-1, 1, (5, 64))
    for ffn, (w1, w3, w2) in zip(experts, ref):
        assert ffn.block_widths == (192, 0, 0)
        got = ffn.layer.cc_forward_host(x, threads=2)
        want = orc.dense_forward(orc.bf16_round(x), w1.T, w2.T, "silu", w3.T)
        assert orc.max_rel_error(got, want) <= 5e-3  # AMX path rounds the hidden activation to bf16


# ---------------------------------------------------------------------------
# GPU: all three blocks


@pytest.mark.gpu
def test_store_round_trip_all_blocks(tmp_path):
    import torch

    from paper_2411_15715_b200.sliced import CallSpec, SlicedFFN, forward_calls

    nat.init(0)
    rng = np.random.default_rng(5)
    M, H = 512, 1664
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (M, H)))
    ffn = SlicedFFN(w1t, w2t, SlicingRates(0.25, 0.3, 0.45), w3t=w3t, dtype="bf16")  # auto chunk_rows
    p = tmp_path / "e.spstore"
    store.save_store(p, {"e0": ffn.layer})
    back = store.load_store(p)["e0"]
    assert back.block_widths == ffn.block_widths
    for T in (1, 3, 40):
        x = torch.from_numpy(rng.standard_normal((T, M)).astype(np.float32)).cuda().to(torch.bfloat16)
        a = forward_calls([CallSpec(ffn.layer)], x).float().cpu()
        b = forward_calls([CallSpec(back)], x).float().cpu()
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_reslice_all_blocks():
    import torch

    from paper_2411_15715_b200.sliced import CallSpec, SlicedFFN, forward_calls

    nat.init(0)
    rng = np.random.default_rng(6)
    M, H = 512, 1664
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (M, H)))
    r0 = SlicingRates(0.2, 0.3, 0.5)
    ffn = SlicedFFN(w1t, w2t, r0, w3t=w3t, dtype="bf16", chunk_rows=128)
    x = torch.from_numpy(rng.standard_normal((2, M)).astype(np.float32)).cuda().to(torch.bfloat16)
    q = orc.bf16_round
    ref = orc.dense_forward(q(x.float().cpu().numpy()), q(w1t.T), q(w2t.T), "silu", q(w3t.T))
    for r in (SlicingRates(0.0, 0.0, 1.0), SlicingRates(0.5, 0.5, 0.0), SlicingRates(0.1, 0.6, 0.3)):
        moved = ffn.reslice(r)
        got = forward_calls([CallSpec(moved.layer)], x).float().cpu().numpy()
        assert orc.max_rel_error(got, ref) <= 1e-2, r
        back = moved.reslice(r0)  # and back: identical placement, identical output bits
        assert torch.equal(forward_calls([CallSpec(back.layer)], x), forward_calls([CallSpec(ffn.layer)], x))
