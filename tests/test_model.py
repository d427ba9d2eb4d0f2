"""Whole-model decode loop: SlicedMixtral with the
sliced MoE vs the same decoder with the MoE computed by the fp64 oracle."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sliced_forward as orc

pytestmark = pytest.mark.gpu


def test_decoder_matches_oracle_moe():
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral
    from paper_2411_15715_b200.schedule import SlicingRates
    from paper_2411_15715_b200.sliced import SlicedFFN

    nat.init(0)
    cfg = DecoderConfig(layers=3, distinct=2, model_dim=256, hidden_dim=640, experts=4, top_k=2, heads=4,
                        kv_heads=2, max_seq=32)
    rng = np.random.default_rng(0)
    weights = {}

    def factory(d):
        ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((640, 256), (640, 256), (256, 640)))
              for _ in range(cfg.experts)]
        weights[d] = [tuple(orc.bf16_round(a) for a in w) for w in ws]
        return [SlicedFFN(w1t, w2t, SlicingRates(0.25, 0.25, 0.5), w3t=w3t, chunk_rows=128) for w1t, w3t, w2t in ws]

    m = SlicedMixtral(cfg, SlicingRates(0.25, 0.25, 0.5), experts_factory=factory)

    class OracleMoE(SlicedMixtral):
        def _moe(self, d, h):
            hq = h.float().cpu().numpy().astype(np.float64)
            experts = [(w1t.T, w3t.T, w2t.T) for w1t, w3t, w2t in weights[d]]  # reference layout
            router = self.routers[d].astype(np.float32).astype(np.float64)  # as the runtime stores it
            y = orc.moe_forward(hq, experts, router, self.cfg.top_k)
            return torch.from_numpy(y.astype(np.float32)).to(h.device, h.dtype)

    ref = OracleMoE.__new__(OracleMoE)
    ref.__dict__.update(m.__dict__)
    ref.kv = m.kv.clone()
    x = (torch.randn(1, 256, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) * 0.5).to(
        torch.bfloat16)
    xa, xb = x, x
    for pos in range(4):
        xa = m.decode_step(xa, pos)
        xb = ref.decode_step(xb, pos)
    err = orc.max_rel_error(xa.float().cpu().numpy(), xb.float().cpu().numpy())
    # whole decoder (attention + bf16 residual stream over 3 layers x 4 steps); each
    # MoE call alone is held to 1e-2 in test_every_moe_call_in_the_decoder_matches_the_oracle
    assert err <= 3e-2, err
    m.release()


def test_every_moe_call_in_the_decoder_matches_the_oracle():
    """Inside the decode loop, every sliced MoE call (the path under test) is
    held to the north-star bf16 bound (<= 1e-2) against the fp64 oracle on
    the same input h.  The whole-decoder comparison above allows 3e-2: it also
    carries the torch attention / RMSNorm and the bf16 residual stream across
    layers, which are outside the sliced path."""
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral
    from paper_2411_15715_b200.schedule import SlicingRates
    from paper_2411_15715_b200.sliced import SlicedFFN

    nat.init(0)
    cfg = DecoderConfig(layers=3, distinct=2, model_dim=256, hidden_dim=640, experts=4, top_k=2, heads=4,
                        kv_heads=2, max_seq=32)
    rng = np.random.default_rng(5)
    weights = {}

    def factory(d):
        ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((640, 256), (640, 256), (256, 640)))
              for _ in range(cfg.experts)]
        weights[d] = [tuple(orc.bf16_round(a) for a in w) for w in ws]
        return [SlicedFFN(w1t, w2t, SlicingRates(0.25, 0.25, 0.5), w3t=w3t, chunk_rows=128) for w1t, w3t, w2t in ws]

    m = SlicedMixtral(cfg, SlicingRates(0.25, 0.25, 0.5), experts_factory=factory)
    seen = []
    inner = m._moe

    def checked(d, h, out=None):
        y = inner(d, h, out=out)
        torch.cuda.synchronize()
        hq = h.float().cpu().numpy().astype(np.float64)
        experts = [(w1t.T, w3t.T, w2t.T) for w1t, w3t, w2t in weights[d]]
        router = m.routers[d].astype(np.float32).astype(np.float64)
        ref = orc.moe_forward(hq, experts, router, cfg.top_k)
        seen.append(orc.max_rel_error(y.float().cpu().numpy(), ref))
        return y

    m._moe = checked
    x = (torch.randn(1, 256, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)) * 0.5).to(
        torch.bfloat16)
    for pos in range(4):
        x = m.decode_step(x, pos)
    assert len(seen) == 4 * cfg.layers
    assert max(seen) <= 1e-2, seen
    m.release()


def test_graph_decode_matches_eager():
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral
    from paper_2411_15715_b200.schedule import SlicingRates

    nat.init(0)
    cfg = DecoderConfig(layers=3, distinct=2, model_dim=256, hidden_dim=640, experts=4, top_k=2, heads=4,
                        kv_heads=2, max_seq=16)
    m = SlicedMixtral(cfg, SlicingRates(0.25, 0.25, 0.5))
    x = (torch.randn(1, 256, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2)) * 0.5).to(
        torch.bfloat16)
    kv0 = m.kv.clone()
    eager = [x]
    for pos in range(5):
        eager.append(m.decode_step(eager[-1], pos))
    m.kv.copy_(kv0)
    m.enable_graphs(x)
    y = x
    for pos in range(5):
        y = m.decode_step_graph(y, 0 if pos == 0 else None).clone()
        err = orc.max_rel_error(y.float().cpu().numpy(), eager[pos + 1].float().cpu().numpy())
        assert err <= 2e-2, (pos, err)
    assert int(m.pos_dev.item()) == 5
    m.release()


def test_prefill_then_decode_matches_incremental_decode():
    """Causal prefill of a short prompt == feeding it token by token through
    decode_step (same cache contents, same last hidden state)."""
    import torch

    from paper_2411_15715_b200 import _native as nat
    from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral
    from paper_2411_15715_b200.schedule import SlicingRates

    nat.init(0)
    cfg = DecoderConfig(layers=2, distinct=2, model_dim=256, hidden_dim=640, experts=4, top_k=2, heads=4,
                        kv_heads=2, max_seq=16)
    m = SlicedMixtral(cfg, SlicingRates(0.25, 0.25, 0.5))
    P = 5
    xs = (torch.randn(P, 256, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)) * 0.5).to(
        torch.bfloat16)
    inc = [m.decode_step(xs[i:i + 1], i) for i in range(P)]
    kv_inc = m.kv.clone()
    m.kv.zero_()
    pre = m.prefill(xs, token_planner=lambda t: t // 2)
    err = orc.max_rel_error(pre[-1:].float().cpu().numpy(), inc[-1].float().cpu().numpy())
    assert err <= 3e-2, err
    kerr = orc.max_rel_error(m.kv[:, :, :, :, :P].float().cpu().numpy(), kv_inc[:, :, :, :, :P].float().cpu().numpy())
    assert kerr <= 3e-2, kerr
    m.release()
