"""GPU parity: the sliced path (GG/CG on the B200 through libsliced, CC on host
threads) against the CPU oracle and the reference goldens.

Tolerances (north star): fp32 max relative error <= 1e-5, bf16 <= 1e-2, with
max relative error = max|got - ref| / max|ref| and the reference fed the
bf16-rounded inputs a bf16 kernel sees.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sliced_forward as orc

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 1e-2


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def sp():
    import paper_2411_15715_b200 as sp
    from paper_2411_15715_b200 import _native

    _native.init(0)
    return sp


def _golden():
    npz = np.load(GOLDEN / "forward_golden.npz")
    return npz, json.loads(bytes(npz["meta_json"]).decode())


def test_reference_goldens_fp32(sp):
    npz, meta = _golden()
    for case in meta["cases"]:
        k = case["key"]
        x, w1, w2 = npz[f"{k}_x"], npz[f"{k}_w1"], npz[f"{k}_w2"]
        rates = sp.SlicingRates(*(float.fromhex(v) for v in case["rates"]))
        act = sp.Activation(case["act"])
        sliced = sp.slice_weights(w1, w2, rates)
        assert list(sliced.block_widths) == case["widths"]
        got = sp.mlp_forward_sliced(x, sliced, act, case["n_g"])
        assert got.dtype == np.float64 and got.shape == npz[f"{k}_sliced"].shape
        assert orc.max_rel_error(got, npz[f"{k}_sliced"]) <= FP32_TOL, k
        dense = sp.mlp_forward_reference(x, w1, w2, act)
        assert orc.max_rel_error(dense, npz[f"{k}_dense"]) <= FP32_TOL, k


def test_recombination_sweep_matches_reference_bound(sp):
    # the reference's own sweep (slicing_kernel.py:161-190), GPU sliced vs GPU dense
    assert sp.max_recombination_error(seed=123, trials=20) <= 1e-4


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("gated", [False, True])
def test_random_shapes_all_splits(sp, dtype, tol, gated):
    rng = np.random.default_rng(2024 + gated + (dtype == "bf16") * 7)
    q = orc.bf16_round if dtype == "bf16" else (lambda a: a)
    for trial in range(12):
        T = int(rng.choice([1, 2, 3, 5, 8, 9, 17]))
        M = int(rng.integers(2, 300))
        H = int(rng.integers(2, 900))
        N = int(rng.integers(2, 300))
        x, w1, w3, w2 = (q(rng.uniform(-1, 1, s)) for s in ((T, M), (M, H), (M, H), (H, N)))
        raw = rng.dirichlet(np.ones(3)) if trial % 4 else np.eye(3)[trial // 4 % 3]
        rates = sp.SlicingRates(raw[0], raw[1], 1.0 - raw[0] - raw[1])
        act = list(sp.Activation)[trial % 3]
        n_g = int(rng.integers(0, T + 1))
        sliced = sp.slice_weights(w1, w2, rates, w3 if gated else None, dtype=dtype, chunk_rows=64)
        got = sp.mlp_forward_sliced(x, sliced, act, n_g)
        ref = orc.sliced_forward(x, w1, w2, act.value, rates.cc, rates.cg, w3 if gated else None)
        assert orc.max_rel_error(got, ref) <= tol, (trial, T, M, H, N, sliced.block_widths, n_g)


def test_many_chunks_exercise_ring_reuse(sp):
    # 1000 hidden rows in 64-row chunks: 16 chunks through a 3-slot ring
    rng = np.random.default_rng(7)
    T, M, H, N = 4, 96, 1000, 80
    x, w1, w3, w2 = (rng.uniform(-1, 1, s) for s in ((T, M), (M, H), (M, H), (H, N)))
    for cc, cg in ((0.0, 1.0), (0.3, 0.6), (0.5, 0.2)):
        rates = sp.SlicingRates(cc, cg, 1.0 - cc - cg)
        sliced = sp.slice_weights(w1, w2, rates, w3, chunk_rows=64)
        for n_g in (0, 2, T):
            got = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU, n_g)
            ref = orc.dense_forward(x, w1, w2, "silu", w3)
            assert orc.max_rel_error(got, ref) <= FP32_TOL


def test_long_stream_deep_ring(sp):
    # >= 32 chunks in one call switch the staging ring to 6 slots; a following
    # short call goes back to 3 -- slot reuse is tracked per slot either way
    rng = np.random.default_rng(8)
    T, M, N = 3, 64, 48
    for H, n_g in ((2400, 0), (2400, T), (300, 1)):
        x, w1, w3, w2 = (rng.uniform(-1, 1, s) for s in ((T, M), (M, H), (M, H), (H, N)))
        sliced = sp.slice_weights(w1, w2, sp.SlicingRates(0.2, 0.8, 0.0), w3, chunk_rows=64)
        got = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU, n_g)
        ref = orc.dense_forward(x, w1, w2, "silu", w3)
        assert orc.max_rel_error(got, ref) <= FP32_TOL, (H, n_g)


def test_diversion_does_not_change_results(sp):
    rng = np.random.default_rng(11)
    x, w1, w2 = rng.uniform(-1, 1, (6, 40)), rng.uniform(-1, 1, (40, 90)), rng.uniform(-1, 1, (90, 30))
    sliced = sp.slice_weights(w1, w2, sp.SlicingRates(1, 0, 0))
    outs = [sp.mlp_forward_sliced(x, sliced, sp.Activation.GELU, n_g=g) for g in range(7)]
    for o in outs[1:]:
        assert np.max(np.abs(o - outs[0])) <= 1e-5


def test_deterministic_repeat(sp):
    rng = np.random.default_rng(12)
    x, w1, w3, w2 = (rng.uniform(-1, 1, s) for s in ((3, 128), (128, 700), (128, 700), (700, 64)))
    sliced = sp.slice_weights(w1, w2, sp.SlicingRates(0.2, 0.3, 0.5), w3, dtype="bf16", chunk_rows=128)
    a = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU)
    b = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU)
    assert np.array_equal(a, b)


def test_device_io_matches_host_io(sp, torch):
    from paper_2411_15715_b200.sliced import SlicedFFN

    rng = np.random.default_rng(13)
    M, H, N = 256, 1536, 256
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (N, H)))
    ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(0.25, 0.25, 0.5), w3t=w3t, dtype="bf16", chunk_rows=256)
    x = torch.randn(5, M, device="cuda", dtype=torch.bfloat16)
    y_dev = ffn(x)
    torch.cuda.synchronize()
    y_host = ffn(x.cpu().float().numpy())
    assert y_dev.dtype == torch.bfloat16 and y_dev.is_cuda
    ref = orc.dense_forward(orc.bf16_round(x.float().cpu().numpy()), orc.bf16_round(w1t.T),
                            orc.bf16_round(w2t.T), "silu", orc.bf16_round(w3t.T))
    assert orc.max_rel_error(y_dev.float().cpu().numpy(), ref) <= BF16_TOL
    # 5 tokens take the tensor-core path (bf16 hidden activations): bf16 bound
    assert orc.max_rel_error(y_host, ref) <= BF16_TOL
    # same arithmetic either way: device and host I/O differ only by the bf16 output cast
    assert orc.max_rel_error(y_dev.float().cpu().numpy(), y_host) <= 4e-3


def test_moe_top2_matches_oracle(sp, torch):
    from paper_2411_15715_b200.sliced import SlicedFFN, SlicedMoE

    rng = np.random.default_rng(14)
    E, M, H = 8, 128, 448
    experts_w = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((H, M), (H, M), (M, H)))
                 for _ in range(E)]
    rates = [sp.SlicingRates(*(lambda r: (r[0], r[1], 1 - r[0] - r[1]))(rng.dirichlet(np.ones(3))))
             for _ in range(E)]
    experts = [SlicedFFN(w1t, w2t, r, w3t=w3t, dtype="f32", chunk_rows=64)
               for (w1t, w3t, w2t), r in zip(experts_w, rates)]
    router = rng.standard_normal((M, E))
    moe = SlicedMoE(experts, router, top_k=2)
    for T in (1, 4, 11):
        x = rng.standard_normal((T, M))
        got = moe(x)
        ref = orc.moe_forward(x, [(w1t.T, w3t.T, w2t.T) for (w1t, w3t, w2t) in experts_w], router, 2)
        assert orc.max_rel_error(got, ref) <= FP32_TOL
        xd = torch.from_numpy(x.astype(np.float32)).cuda()
        got_d = moe(xd).cpu().numpy()
        assert orc.max_rel_error(got_d, ref) <= FP32_TOL


@pytest.mark.slow
def test_full_size_mixtral_expert_bf16(sp, torch):
    """One Mixtral-8x7B expert (4096 x 14336, SwiGLU, bf16) at config-2 style
    rates: GPU sliced vs fp64 oracle on the same bf16 values."""
    from paper_2411_15715_b200.sliced import SlicedFFN

    M, H = 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    w1t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(torch.bfloat16)
    w3t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(torch.bfloat16)
    w2t = (torch.randn(M, H, device="cuda", generator=g) / 120).to(torch.bfloat16)
    x = torch.randn(2, M, device="cuda", generator=g).to(torch.bfloat16)
    ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(0.15, 0.2, 0.65), w3t=w3t, dtype="bf16")
    y = ffn(x).float().cpu().numpy()
    f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    ref = orc.dense_forward(f(x), f(w1t).T, f(w2t).T, "silu", f(w3t).T)
    assert orc.max_rel_error(y, ref) <= BF16_TOL
    # output rounding to bf16 dominates; the fp32 accumulation itself is much tighter
    assert orc.max_rel_error(y, ref) <= 5e-3


@pytest.mark.parametrize("gated", [True, False])
@pytest.mark.parametrize("T", [16, 64, 200, 300])
def test_prefill_tensor_core_path(sp, torch, gated, T):
    """T >= 16 bf16 tokens go through the tcgen05 GEMM pair (up + fused SwiGLU,
    down accumulate); CG chunks, the n_g diverted rows and the CC host rows
    included."""
    from paper_2411_15715_b200.sliced import SlicedFFN

    rng = np.random.default_rng(100 + T + gated)
    M, H = 512, 1664
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (M, H)))
    q = orc.bf16_round
    for cc, cg, ng in ((0.0, 0.0, 0), (0.25, 0.25, 0), (0.25, 0.25, T // 2), (0.5, 0.0, T)):
        ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(cc, cg, 1.0 - cc - cg), w3t=w3t if gated else None,
                        activation="silu", dtype="bf16", chunk_rows=256)
        x = torch.from_numpy(rng.standard_normal((T, M)).astype(np.float32)).cuda().to(torch.bfloat16)
        y = ffn(x, n_g=ng).float().cpu().numpy()
        ref = orc.dense_forward(q(x.float().cpu().numpy()), q(w1t.T), q(w2t.T), "silu", q(w3t.T) if gated else None)
        assert orc.max_rel_error(y, ref) <= BF16_TOL, (cc, cg, ng)


@pytest.mark.parametrize("M,H,T", [(1024, 3000, 300), (768, 1100, 256), (4096, 14336, 512)])
def test_prefill_cta_pair_up_gemm(sp, torch, M, H, T):
    """256-token tiles run the up GEMM on CTA pairs (gemm_up_pair_kernel:
    tcgen05 cta_group::2, M = 256 across two SMs, each loading half the x
    tile): split-K z partials (resident, few tiles), an odd row-tile count
    (the last pair's second CTA is past the rows), and a whole Mixtral expert
    at T = 512 with the direct SwiGLU epilogue."""
    from paper_2411_15715_b200.sliced import SlicedFFN

    rng = np.random.default_rng(M + H + T)
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (M, H)))
    ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(0.0, 0.0, 1.0), w3t=w3t, activation="silu", dtype="bf16")
    x = torch.from_numpy(rng.standard_normal((T, M)).astype(np.float32)).cuda().to(torch.bfloat16)
    y0 = ffn(x)
    assert torch.equal(y0, ffn(x))
    q = orc.bf16_round
    rows = slice(None) if T <= 300 else slice(0, T, 7)  # fp64 oracle on a token subset at full size
    xs = q(x.float().cpu().numpy())[rows]
    ref = orc.dense_forward(xs, q(w1t.T), q(w2t.T), "silu", q(w3t.T))
    assert orc.max_rel_error(y0.float().cpu().numpy()[rows], ref) <= BF16_TOL


def test_prefill_moe_tensor_core_path(sp, torch):
    from paper_2411_15715_b200.sliced import SlicedFFN, SlicedMoE

    rng = np.random.default_rng(321)
    E, M, H, T = 8, 256, 768, 96
    ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((H, M), (H, M), (M, H))) for _ in range(E)]
    experts = [SlicedFFN(w1t, w2t, sp.SlicingRates(0.2, 0.3, 0.5), w3t=w3t, dtype="bf16", chunk_rows=128)
               for w1t, w3t, w2t in ws]
    router = rng.standard_normal((M, E))
    x = rng.standard_normal((T, M)).astype(np.float32)
    xq = orc.bf16_round(x)
    got = SlicedMoE(experts, router, 2)(torch.from_numpy(x).cuda().to(torch.bfloat16)).float().cpu().numpy()
    q = orc.bf16_round
    ref = orc.moe_forward(xq, [(q(a.T), q(b.T), q(c.T)) for a, b, c in ws], router, 2)
    assert orc.max_rel_error(got, ref) <= BF16_TOL


@pytest.mark.parametrize("T", [1, 24])
def test_back_to_back_device_forwards(sp, torch, T):
    """Consecutive device-I/O forwards return before their GPU work (and the
    finalize that reads the CC partial from pinned staging) has run: every
    output must still be its own input's."""
    from paper_2411_15715_b200.sliced import SlicedFFN

    rng = np.random.default_rng(77 + T)
    M, H = 512, 1536
    w1t, w3t, w2t = (rng.standard_normal(s).astype(np.float32) / 16 for s in ((H, M), (H, M), (M, H)))
    ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(0.3, 0.3, 0.4), w3t=w3t, dtype="bf16", chunk_rows=128)
    xs = [torch.from_numpy(rng.standard_normal((T, M)).astype(np.float32)).cuda().to(torch.bfloat16) for _ in range(8)]
    ys = [ffn(x) for x in xs]  # no synchronisation in between
    torch.cuda.synchronize()
    q = orc.bf16_round
    for x, y in zip(xs, ys):
        ref = orc.dense_forward(q(x.float().cpu().numpy()), q(w1t.T), q(w2t.T), "silu", q(w3t.T))
        assert orc.max_rel_error(y.float().cpu().numpy(), ref) <= BF16_TOL


def test_grouped_gg_launch_with_many_experts(sp, torch):
    """Eight experts with 3 tokens each in one grouped GG launch (a short prompt
    or a big decode batch), 4608 GG rows each: 8 x 4608 / 148 SMs would put 249
    rows in a CTA, more than its shared memory holds at a 4-token tile -- the
    group must spread them over more CTAs.  Reference: torch fp32 on the GPU."""
    from paper_2411_15715_b200.sliced import CallSpec, SlicedFFN, forward_calls

    E, M, H, T = 8, 4096, 4608, 16
    g = torch.Generator(device="cuda").manual_seed(55)
    ws = [tuple((torch.randn(*s, device="cuda", generator=g) / 32).to(torch.bfloat16) for s in ((H, M), (H, M), (M, H)))
          for _ in range(E)]
    experts = [SlicedFFN(w1t.cpu(), w2t.cpu(), sp.SlicingRates(0.0, 0.0, 1.0), w3t=w3t.cpu(), dtype="bf16")
               for w1t, w3t, w2t in ws]
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    ids = [torch.tensor([(2 * i) % T, (2 * i + 1) % T, (2 * i + 5) % T], dtype=torch.int32) for i in range(E)]
    y = forward_calls([CallSpec(e.layer, i.numpy()) for e, i in zip(experts, ids)], x).float()
    ref = torch.zeros(T, M, device="cuda")
    xf = x.float()
    for (w1t, w3t, w2t), i in zip(ws, ids):
        xi = xf[i.long().cuda()]
        h = torch.nn.functional.silu(xi @ w1t.float().t()) * (xi @ w3t.float().t())
        ref.index_add_(0, i.long().cuda(), h @ w2t.float().t())
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    assert err <= BF16_TOL, err
    for e in experts:
        e.layer.release()


_CC_BATCH_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2411_15715_b200 import _native
_native.init(0)
import paper_2411_15715_b200 as sp
from paper_2411_15715_b200.sliced import SlicedFFN, SlicedMoE
rng = np.random.default_rng(5)
E, M, H = 4, 256, 1000
ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((H, M), (H, M), (M, H))) for _ in range(E)]
experts = [SlicedFFN(a, c, sp.SlicingRates(0.4, 0.3, 0.3), w3t=b, dtype="bf16", chunk_rows=128) for a, b, c in ws]
moe = SlicedMoE(experts, rng.standard_normal((M, E)), 2)
ys = [moe(rng.standard_normal((T, M))) for T in (1, 2, 3)]
sys.stdout.buffer.write(b"".join(np.ascontiguousarray(y, dtype=np.float32).tobytes() for y in ys))
"""


def test_cc_batch_pass_is_bit_identical_to_per_expert_passes(tmp_path):
    """cc_forward_batch (one pool pass for every active expert's CC block) must
    give the same bits as one cc_forward per expert (SP_CC_BATCH=0)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    repo = str(Path(__file__).resolve().parents[1])
    script = tmp_path / "probe.py"
    script.write_text(_CC_BATCH_PROBE)
    outs = []
    for v in ("0", "1"):
        env = dict(os.environ, SP_CC_BATCH=v)
        r = subprocess.run([sys.executable, str(script), repo], env=env, capture_output=True, timeout=300)
        assert r.returncode == 0, r.stderr.decode()[-2000:]
        outs.append(r.stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1]
