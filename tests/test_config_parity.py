"""GPU parity at every BASELINE.json config shape bench.py reports.

Each test builds the layer exactly as ``bench.py`` does for that config
(same shapes, dtype, router, top-k and the slicing rates ``bench.plan_rates``
derives from the committed B200 profiles under the stated budget), runs it
through the product path (sp_moe_forward / sp_forward_batch via ctypes) and
compares with the fp64 oracle (oracle/sliced_forward.py, the restatement of
/root/reference/pkg/src/sliceplan/slicing_kernel.py:97-124, pinned to the
reference's goldens in tests/test_oracle.py).

Tolerances are the north star's, written here: fp32 max relative error
<= 1e-5 and bf16 <= 1e-2 against the oracle fed the same (bf16-rounded)
weights and activations.  Full-size weights are converted to fp64 a block of
hidden units at a time (``orc.segment_forward`` per block, summed in fp64), so
the oracle never holds a whole fp64 expert of the large configs.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import ROOT  # noqa: F401  (puts the repo root on sys.path)
from oracle import sliced_forward as orc

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 1e-2
# the bench's committed profiles were fitted with 16 host threads (the 1-GPU
# pool box); plan with that count so the widths are the bench line's
PROFILE_THREADS = "16"


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    from paper_2411_15715_b200 import _native

    _native.init(0)
    return torch


def bench_plan(monkeypatch, *argv):
    """(args, rates) exactly as bench.py plans the config."""
    import bench

    monkeypatch.setenv("SP_HOST_THREADS", PROFILE_THREADS)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse(list(argv))
    rates = bench.plan_rates(args, args.batch)[0]
    return args, rates


def make_weights(torch, E, M, H, dtype, seed0=1000):
    """bench.make_experts' random-init weights (HF layout, CPU tensors)."""
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    out = []
    for e in range(E):
        g = torch.Generator(device="cuda").manual_seed(seed0 + e)
        w1t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(tdt).cpu()
        w3t = (torch.randn(H, M, device="cuda", generator=g) / 64).to(tdt).cpu()
        w2t = (torch.randn(M, H, device="cuda", generator=g) / 120).to(tdt).cpu()
        out.append((w1t, w3t, w2t))
    return out


def oracle_expert(x64, w1t, w3t, w2t, block=2048):
    """fp64 SwiGLU expert on rows x64, the hidden dimension in blocks."""
    H = w1t.shape[0]
    y = np.zeros((x64.shape[0], w2t.shape[0]))
    for lo in range(0, H, block):
        hi = min(H, lo + block)
        w1 = w1t[lo:hi].double().numpy().T
        w3 = w3t[lo:hi].double().numpy().T
        w2 = w2t[:, lo:hi].double().numpy().T
        y += orc.segment_forward(x64, w1, w2, "silu", 0, hi - lo, w3)
    return y


def oracle_moe(x64, weights, router, k, rows=None):
    """Top-k MoE (oracle routing on the fp32-held router) on the selected rows."""
    rows = np.arange(x64.shape[0]) if rows is None else np.asarray(rows)
    xs = x64[rows]
    ids, gates = orc.route_topk(xs @ router.astype(np.float32).astype(np.float64), k)
    y = np.zeros((xs.shape[0], weights[0][2].shape[0]))
    for e in np.unique(ids):
        sel, slot = np.nonzero(ids == e)
        ye = oracle_expert(xs[sel], *weights[int(e)])
        y[sel] += gates[sel, slot][:, None] * ye
    return y, ids


def place(weights, rates, dtype):
    from paper_2411_15715_b200.sliced import SlicedFFN

    return [SlicedFFN(w1t, w2t, rates, w3t=w3t, activation="silu", dtype=dtype) for w1t, w3t, w2t in weights]


def release(experts):
    for e in experts:
        e.layer.release()


def check_moe(torch, experts, weights, router, k, xs, tol, rows=None):
    """Product MoE (device I/O and host I/O) vs the oracle for each x in xs."""
    from paper_2411_15715_b200.sliced import SlicedMoE, moe_route

    moe = SlicedMoE(experts, router, k)
    dt = torch.bfloat16 if experts[0].layer.dtype == "bf16" else torch.float32
    worst = 0.0
    for x in xs:
        xd = torch.from_numpy(x.astype(np.float32)).cuda().to(dt)
        x64 = xd.float().cpu().numpy().astype(np.float64)  # the values the kernels see
        ref, ref_ids = oracle_moe(x64, weights, router, k, rows)
        ids, _ = moe_route(x64.astype(np.float32), router, k)
        sel = slice(None) if rows is None else rows
        assert np.array_equal(ids[sel], ref_ids), "product routing differs from the oracle's"
        y_dev = moe(xd).float().cpu().numpy()[sel]
        y_host = np.asarray(moe(x64.astype(np.float32)))[sel]
        for io, got in (("device", y_dev), ("host", y_host)):
            err = orc.max_rel_error(got, ref)
            worst = max(worst, err)
            print(f"PARITY T={x.shape[0]} io={io} max_rel_err={err:.3e} tol={tol:g}")
            assert err <= tol, (x.shape, err)
    return worst


# ---------------------------------------------------------------------------
# configs[0]: 1024/3584 fp32, 8 experts top-2, fixed 0.2/0.3/0.5


def test_cfg1_fp32_moe_layer(torch, monkeypatch):
    args, rates = bench_plan(monkeypatch, "--config", "cfg1")
    assert (rates.cc, rates.cg, rates.gg) == (0.2, 0.3, 0.5)
    weights = make_weights(torch, args.experts, args.model_dim, args.hidden_dim, "f32")
    experts = place(weights, rates, "f32")
    print(f"PARITY cfg1 widths={experts[0].block_widths}")
    assert experts[0].block_widths == (716, 1076, 1792)
    router = np.random.default_rng(7).standard_normal((args.model_dim, args.experts))
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal((T, args.model_dim)) for T in (1, 1, 3, 8)]
    check_moe(torch, experts, weights, router, args.top_k, xs, FP32_TOL)
    release(experts)


# ---------------------------------------------------------------------------
# configs[1]: Mixtral-8x7B layer, bf16, decode at the solver's widths


def test_cfg2_mixtral_moe_layer_at_solved_widths(torch, monkeypatch):
    args, rates = bench_plan(monkeypatch)
    weights = make_weights(torch, args.experts, args.model_dim, args.hidden_dim, "bf16")
    experts = place(weights, rates, "bf16")
    print(f"PARITY cfg2 widths={experts[0].block_widths}")
    assert experts[0].block_widths == (5386, 1781, 7169)  # BENCH_r01 config.block_widths
    router = np.random.default_rng(7).standard_normal((args.model_dim, args.experts))
    rng = np.random.default_rng(2)
    # decode steps (the headline), a 2-token and a 9-token batch (tensor-core path)
    xs = [rng.standard_normal((1, args.model_dim)) for _ in range(3)] + [
        rng.standard_normal((T, args.model_dim)) for T in (2, 9)]
    check_moe(torch, experts, weights, router, args.top_k, xs, BF16_TOL)
    release(experts)


# ---------------------------------------------------------------------------
# configs[2]: the prompt layer, T = 512 with solve_ng's token split


def test_cfg3_prompt_layer_with_solve_ng_split(torch, monkeypatch):
    import bench
    import paper_2411_15715_b200 as sp
    from paper_2411_15715_b200.sliced import SlicedMoE, moe_route

    args, rates = bench_plan(monkeypatch, "--config", "cfg3")
    p_profile, _ = bench.load_profile(bench.prompt_profile_path(args))
    spec = sp.LayerSpec(args.model_dim, args.hidden_dim, n_gemms=3, precision=sp.Precision.FP16)
    weights = make_weights(torch, args.experts, args.model_dim, args.hidden_dim, "bf16")
    experts = place(weights, rates, "bf16")
    router = np.random.default_rng(11).standard_normal((args.model_dim, args.experts))
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal((args.prompt, args.model_dim)).astype(np.float32)).cuda().to(
        torch.bfloat16)
    x64 = x.float().cpu().numpy().astype(np.float64)
    ids, _ = moe_route(x64.astype(np.float32), router, args.top_k)
    counts = np.bincount(ids.ravel(), minlength=args.experts)
    n_g = {e: sp.solve_ng(p_profile, spec, int(t), rates, transfer_model=args.transfer_model).n_g
           for e, t in enumerate(counts) if t}
    assert any(0 < n < counts[e] for e, n in n_g.items()), (n_g, counts)  # a real CPU/GPU split
    y = SlicedMoE(experts, router, args.top_k)(x, n_g=n_g).float().cpu().numpy()
    rows = np.arange(0, args.prompt, 5)  # fp64 oracle on a token subset
    ref, _ = oracle_moe(x64, weights, router, args.top_k, rows)
    err = orc.max_rel_error(y[rows], ref)
    print(f"PARITY cfg3 T={args.prompt} n_g={n_g} counts={counts.tolist()} max_rel_err={err:.3e}")
    assert err <= BF16_TOL
    release(experts)


# ---------------------------------------------------------------------------
# configs[3]: LLaMA-2-70B dense FFN 8192/28672 (ffn_block NV=4, tcgen05 at M = 8192)


@pytest.mark.parametrize("world", [1, 2])
def test_cfg4_llama70b_dense_ffn(torch, monkeypatch, world):
    from paper_2411_15715_b200.expert_parallel import column_shard
    from paper_2411_15715_b200.sliced import SlicedFFN

    args, _ = bench_plan(monkeypatch, "--config", "cfg4")
    lo, hi = column_shard(args.hidden_dim, 0, world)  # rank 0's shard (the whole layer at world 1)
    args.shard_hidden = hi - lo
    import bench

    rates = bench.plan_rates(args, 1)[0]
    (w1t, w3t, w2t), = make_weights(torch, 1, args.model_dim, hi - lo, "bf16")
    ffn = SlicedFFN(w1t, w2t, rates, w3t=w3t, activation="silu", dtype="bf16")
    assert sum(ffn.block_widths) == hi - lo and min(ffn.block_widths) > 0
    rng = np.random.default_rng(4)
    for T in (1, 2, 8, 40):  # CUDA-core GEMV tiles (T <= 2 at M = 8192), then tcgen05
        x = torch.from_numpy(rng.standard_normal((T, args.model_dim)).astype(np.float32)).cuda().to(torch.bfloat16)
        x64 = x.float().cpu().numpy().astype(np.float64)
        ref = oracle_expert(x64, w1t, w3t, w2t)
        got = ffn(x).float().cpu().numpy()
        got_h = np.asarray(ffn(x64.astype(np.float32)))
        e_d, e_h = orc.max_rel_error(got, ref), orc.max_rel_error(got_h, ref)
        print(f"PARITY cfg4 world={world} widths={ffn.block_widths} T={T} device={e_d:.3e} host={e_h:.3e}")
        assert e_d <= BF16_TOL and e_h <= BF16_TOL, T
    ffn.layer.release()


# ---------------------------------------------------------------------------
# configs[4]: PhiMoE 16x(4096/6400) and Mixtral-8x22B 8x(6144/16384), batch sweep


@pytest.mark.parametrize("moe", ["phimoe", "8x22b"])
def test_cfg5_moe_batch_sweep(torch, monkeypatch, moe):
    args, rates = bench_plan(monkeypatch, "--config", "cfg5", "--moe", moe)
    weights = make_weights(torch, args.experts, args.model_dim, args.hidden_dim, "bf16")
    experts = place(weights, rates, "bf16")
    print(f"PARITY cfg5 {moe} widths={experts[0].block_widths}")
    router = np.random.default_rng(7).standard_normal((args.model_dim, args.experts))
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal((B, args.model_dim)) for B in (1, 4, 32)]
    # B = 32: every expert active with ~8 tokens each -> the tcgen05 pair at M = 6144 / 4096
    rows = np.arange(0, 32, 3)
    check_moe(torch, experts, weights, router, args.top_k, xs[:2], BF16_TOL)
    check_moe(torch, experts, weights, router, args.top_k, xs[2:], BF16_TOL, rows=rows)
    release(experts)
