"""GPU parity of the tensor-core prefill path (gather -> tcgen05 up GEMM with
fused SwiGLU -> down GEMM -> finalize) at 5 <= T <= 128 tokens on edge shapes:
row counts that are not multiples of the 128-row tile or the 64-row k-block,
output widths that are not multiples of the 256-column down tile, model widths
that are not multiples of 64, token counts on and off the 16/32/64/128 tiles,
split-K over many CTAs and over one, and the n_g split (CC rows streamed for the
diverted prompt rows).  Checked against the fp64 oracle on the same bf16 values
(north-star bf16 bound 1e-2, max |got - ref| / max |ref|); the forward being
matched is the reference's sliced MLP (slicing_kernel.py:97-124)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sliced_forward as orc

pytestmark = pytest.mark.gpu

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


CASES = [
    # M, H, N, T, gated, act
    (384, 900, 384, 5, True, "silu"),
    (512, 1664, 512, 16, True, "silu"),
    (512, 1664, 512, 17, True, "silu"),
    (256, 1000, 200, 33, True, "gelu"),
    (200, 700, 260, 64, False, "gelu"),
    (1024, 3000, 1024, 100, True, "silu"),
    (768, 1100, 768, 128, True, "silu"),
    (128, 130, 68, 20, True, "identity"),  # 2 row tiles, 3 down k-blocks
    (4096, 1000, 64, 24, True, "silu"),  # one 64-column down tile over a long K
    (2048, 5632, 2048, 48, True, "silu"),
]


@pytest.mark.parametrize("M,H,N,T,gated,act", CASES)
def test_resident_block_matches_oracle(sp, torch, M, H, N, T, gated, act):
    rng = np.random.default_rng(M * 7 + H + N + T)
    q = orc.bf16_round
    x, w1, w3, w2 = (q(rng.standard_normal(s) / d) for s, d in (((T, M), 1), ((M, H), 16), ((M, H), 16), ((H, N), 16)))
    sliced = sp.slice_weights(w1, w2, sp.SlicingRates(0.0, 0.0, 1.0), w3 if gated else None, dtype="bf16")
    got = sp.mlp_forward_sliced(x, sliced, sp.Activation(act))
    ref = orc.dense_forward(x, w1, w2, act, w3 if gated else None)
    err = orc.max_rel_error(got, ref)
    print(f"PARITY tc M={M} H={H} N={N} T={T} gated={gated} {act}: {err:.2e}")
    assert err <= BF16_TOL
    # fixed split-K partition, splits summed in order: bit-identical on repeat
    assert np.array_equal(got, sp.mlp_forward_sliced(x, sliced, sp.Activation(act)))


@pytest.mark.parametrize("T,n_g", [(40, 13), (128, 64), (96, 96)])
def test_split_rates_and_diverted_rows(sp, torch, T, n_g):
    """CC + CG + GG with n_g diverted prompt rows: the GG block is applied to
    every token and the CC rows [0, b1) are streamed for the last n_g tokens."""
    rng = np.random.default_rng(500 + T + n_g)
    M, H = 512, 2000
    q = orc.bf16_round
    x, w1, w3, w2 = (q(rng.standard_normal(s) / d) for s, d in (((T, M), 1), ((M, H), 16), ((M, H), 16), ((H, M), 16)))
    for rates in ((0.2, 0.3, 0.5), (0.0, 0.5, 0.5), (0.5, 0.0, 0.5)):
        sliced = sp.slice_weights(w1, w2, sp.SlicingRates(*rates), w3, dtype="bf16", chunk_rows=256)
        got = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU, n_g)
        ref = orc.sliced_forward(x, w1, w2, "silu", rates[0], rates[1], w3)
        assert orc.max_rel_error(got, ref) <= BF16_TOL, rates


@pytest.mark.slow
@pytest.mark.parametrize("T", [16, 64, 128])
def test_full_mixtral_expert(sp, torch, T):
    """A whole Mixtral-8x7B expert (4096 x 14336 SwiGLU) resident at the
    per-expert token counts of a 512-token prompt; fp64 oracle on a token subset."""
    from paper_2411_15715_b200.sliced import SlicedFFN

    M, H = 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(T)
    w1t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(torch.bfloat16)
    w3t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(torch.bfloat16)
    w2t = (torch.randn(M, H, device="cuda", generator=g) / 120).to(torch.bfloat16)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    ffn = SlicedFFN(w1t, w2t, sp.SlicingRates(0.0, 0.0, 1.0), w3t=w3t, dtype="bf16")
    y = ffn(x)
    assert torch.equal(y, ffn(x))
    rows = slice(0, T, 5)
    f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    ref = orc.dense_forward(f(x)[rows], f(w1t).T, f(w2t).T, "silu", f(w3t).T)
    err = orc.max_rel_error(y.float().cpu().numpy()[rows], ref)
    print(f"PARITY tc mixtral T={T}: {err:.2e}")
    assert err <= BF16_TOL


@pytest.mark.parametrize("n_g", [0, 70])
def test_host_io_prompt_merges_cc_on_the_host(sp, torch, n_g):
    """Host-I/O prompt calls whose output exceeds the zero-copy limit add the CC
    partials on the host to the read-back device output (SP_HOST_MERGE): a dense
    layer with CC + CG + GG blocks and the n_g split, and a top-2 MoE layer
    (gates, several calls per token) -- both against the oracle."""
    from paper_2411_15715_b200.sliced import SlicedFFN, SlicedMoE

    rng = np.random.default_rng(900 + n_g)
    q = orc.bf16_round
    T, M, H = 200, 1024, 1536
    x, w1, w3, w2 = (q(rng.standard_normal(s) / d) for s, d in (((T, M), 1), ((M, H), 16), ((M, H), 16), ((H, M), 16)))
    sliced = sp.slice_weights(w1, w2, sp.SlicingRates(0.3, 0.3, 0.4), w3, dtype="bf16", chunk_rows=256)
    got = sp.mlp_forward_sliced(x, sliced, sp.Activation.SILU, n_g)  # numpy x: host I/O, 800 KB output
    ref = orc.sliced_forward(x, w1, w2, "silu", 0.3, 0.3, w3)
    assert orc.max_rel_error(got, ref) <= BF16_TOL
    E, H2 = 4, 768
    ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((H2, M), (H2, M), (M, H2))) for _ in range(E)]
    experts = [SlicedFFN(a, c, sp.SlicingRates(0.3, 0.2, 0.5), w3t=b, dtype="bf16", chunk_rows=128) for a, b, c in ws]
    router = rng.standard_normal((M, E)).astype(np.float32).astype(np.float64)
    xm = q(rng.standard_normal((T, M)))
    got = np.asarray(SlicedMoE(experts, router, 2)(xm))
    ref = orc.moe_forward(xm, [(q(a.T), q(b.T), q(c.T)) for a, b, c in ws], router, 2)
    assert orc.max_rel_error(got, ref) <= BF16_TOL
