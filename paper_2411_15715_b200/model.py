"""Whole-model decode loop around the sliced MoE FFN.

The reference models one FFN/MoE layer at a time (pipeline.py:237-260 runs
the recurrence over n_l layers of FFN GEMMs only); a served model interleaves
attention with those layers.  This is the smallest faithful Mixtral-style
decoder around the path:

    x = x + o_proj(attn(rope(q_proj(rms(x))), kv_cache))     (torch: plumbing)
    x = x + moe(rms(x))                                       (libsliced: the path)

The MoE is ``sliced.moe_forward`` -- routing, GG / CG / CC blocks and the merge
in one native call per layer, ordered on the current CUDA stream -- so the
attention of layer l+1 runs on the GPU right behind layer l's merge kernel
with no host synchronisation besides the router's read of x.  The CC partial
needs no host-to-device copy (finalize_kernel reads it from pinned memory),
which is the reference's separate Y_cc transfer (pipeline.py:367-383) folded
into the merge.  Attention is PyTorch over a static KV cache (one query
token: two batched GEMVs per KV-head group and a softmax): it is outside the
sliced path and stays plain library code.

Weights are random-init (seeded) with Mixtral-8x7B shapes by default; layers
may share MoE weight sets (``distinct``) so a 32-layer stack fits the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .schedule import SlicingRates
from .sliced import CallSpec, MoEDispatch, SlicedFFN, forward_calls, moe_route


@dataclass
class DecoderConfig:
    layers: int = 32
    distinct: int = 4          # distinct MoE weight sets cycled over the layers
    model_dim: int = 4096
    hidden_dim: int = 14336
    experts: int = 8
    top_k: int = 2
    heads: int = 32
    kv_heads: int = 8
    max_seq: int = 1024
    rope_theta: float = 1e6
    eps: float = 1e-5


class SlicedMixtral:
    """Mixtral-style decoder whose MoE FFNs run the sliced CC/CG/GG path."""

    def __init__(self, cfg: DecoderConfig, rates: SlicingRates, device: int = 0, seed: int = 0,
                 dtype: str = "bf16", experts_factory=None):
        import torch

        self.torch = torch
        self.cfg = cfg
        dev = torch.device("cuda", device)
        self.device = dev
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdt = tdt
        M, hd = cfg.model_dim, cfg.model_dim // cfg.heads
        self.head_dim = hd
        g = torch.Generator(device=dev).manual_seed(seed)

        def rnd(*shape, scale):
            return (torch.randn(*shape, device=dev, generator=g) * scale).to(tdt)

        self.attn = []
        for _ in range(cfg.layers):
            self.attn.append({
                "wqkv": rnd((cfg.heads + 2 * cfg.kv_heads) * hd, M, scale=1 / math.sqrt(M)),
                "wo": rnd(M, cfg.heads * hd, scale=1 / math.sqrt(cfg.heads * hd)),
                "n1": torch.ones(M, device=dev, dtype=tdt),
                "n2": torch.ones(M, device=dev, dtype=tdt),
            })
        rng = np.random.default_rng(seed)
        make = experts_factory or (lambda d: [
            SlicedFFN(rnd(cfg.hidden_dim, M, scale=1 / 64).cpu(), rnd(M, cfg.hidden_dim, scale=1 / 120).cpu(),
                      rates, w3t=rnd(cfg.hidden_dim, M, scale=1 / 64).cpu(), activation="silu", dtype=dtype,
                      device=device)
            for _ in range(cfg.experts)])
        self.moe_sets = [make(d) for d in range(cfg.distinct)]
        self.routers = [rng.standard_normal((M, cfg.experts)) / math.sqrt(M) for _ in range(cfg.distinct)]
        self.dispatch = [MoEDispatch([e.layer for e in self.moe_sets[d]], self.routers[d], cfg.top_k)
                         for d in range(cfg.distinct)] if self.moe_sets and self.moe_sets[0] else []
        kv_shape = (cfg.layers, 2, 1, cfg.kv_heads, cfg.max_seq, hd)
        self.kv = torch.zeros(kv_shape, device=dev, dtype=tdt)
        pos = torch.arange(cfg.max_seq, device=dev, dtype=torch.float32)
        inv = cfg.rope_theta ** (-torch.arange(0, hd, 2, device=dev, dtype=torch.float32) / hd)
        ang = torch.outer(pos, inv)
        self.cos, self.sin = ang.cos(), ang.sin()

    # -- torch plumbing ------------------------------------------------------
    def _rms(self, x, w):
        torch = self.torch
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.cfg.eps)).to(x.dtype) * w

    def _rope(self, t, pos):
        # t: [B, heads, hd]; rotate pairs (even, odd) at position pos
        c, s = self.cos[pos], self.sin[pos]
        tf = t.float().view(*t.shape[:-1], -1, 2)
        a, b = tf[..., 0], tf[..., 1]
        return self.torch.stack((a * c - b * s, a * s + b * c), -1).flatten(-2).to(t.dtype)

    def _attention(self, l, h, pos):
        torch = self.torch
        cfg, hd = self.cfg, self.head_dim
        B = h.shape[0]
        qkv = h @ self.attn[l]["wqkv"].t()
        q = qkv[:, : cfg.heads * hd].view(B, cfg.heads, hd)
        k = qkv[:, cfg.heads * hd: (cfg.heads + cfg.kv_heads) * hd].view(B, cfg.kv_heads, hd)
        v = qkv[:, (cfg.heads + cfg.kv_heads) * hd:].view(B, cfg.kv_heads, hd)
        q, k = self._rope(q, pos), self._rope(k, pos)
        self.kv[l, 0, 0, :, pos] = k[0]
        self.kv[l, 1, 0, :, pos] = v[0]
        K = self.kv[l, 0, 0, :, : pos + 1]  # [kv_heads, pos+1, hd]
        V = self.kv[l, 1, 0, :, : pos + 1]
        # one query token: two batched GEMVs per KV head group (no per-length
        # plan building, which cuDNN's SDPA does for every new context length)
        qg = q.view(cfg.kv_heads, cfg.heads // cfg.kv_heads, hd)
        p = torch.softmax((qg @ K.transpose(-1, -2)).float() * (1.0 / math.sqrt(hd)), dim=-1).to(q.dtype)
        o = p @ V  # [kv_heads, group, hd]
        return o.reshape(B, cfg.heads * hd) @ self.attn[l]["wo"].t()

    # -- decode --------------------------------------------------------------
    def decode_step(self, x, pos: int):
        """One token through every layer (batch 1); x: [1, M] on the device."""
        cfg = self.cfg
        for l in range(cfg.layers):
            x = x + self._attention(l, self._rms(x, self.attn[l]["n1"]), pos)
            d = l % cfg.distinct
            h = self._rms(x, self.attn[l]["n2"])
            x = x + self._moe(d, h)
        return x

    def _moe(self, d: int, h, out=None):
        return self.dispatch[d](h, out)

    # -- prefill -----------------------------------------------------------------
    def prefill(self, x, token_planner=None):
        """The prompt x [P, M] through every layer: causal attention over the
        prompt (K / V written to cache positions [0, P)), then the sliced MoE
        with the prompt-phase token split -- ``token_planner(T_e) -> n_g`` per
        expert (e.g. the reference's solve_ng; None keeps every row on the
        host for the CC columns).  Routing uses the runtime's router, as decode
        does.  Returns the hidden states [P, M]."""
        torch = self.torch
        cfg, hd = self.cfg, self.head_dim
        P = x.shape[0]
        cos, sin = self.cos[:P][:, None, :], self.sin[:P][:, None, :]

        def rope(t):  # [P, heads, hd]
            tf = t.float().view(*t.shape[:-1], -1, 2)
            a, b = tf[..., 0], tf[..., 1]
            return torch.stack((a * cos - b * sin, a * sin + b * cos), -1).flatten(-2).to(t.dtype)

        for l in range(cfg.layers):
            h = self._rms(x, self.attn[l]["n1"])
            qkv = h @ self.attn[l]["wqkv"].t()
            q = rope(qkv[:, : cfg.heads * hd].view(P, cfg.heads, hd))
            k = rope(qkv[:, cfg.heads * hd: (cfg.heads + cfg.kv_heads) * hd].view(P, cfg.kv_heads, hd))
            v = qkv[:, (cfg.heads + cfg.kv_heads) * hd:].view(P, cfg.kv_heads, hd)
            self.kv[l, 0, 0, :, :P] = k.transpose(0, 1)
            self.kv[l, 1, 0, :, :P] = v.transpose(0, 1)
            o = torch.nn.functional.scaled_dot_product_attention(
                q.transpose(0, 1)[None], k.transpose(0, 1)[None], v.transpose(0, 1)[None], is_causal=True,
                enable_gqa=True)
            x = x + o[0].transpose(0, 1).reshape(P, cfg.heads * hd) @ self.attn[l]["wo"].t()
            h2 = self._rms(x, self.attn[l]["n2"])
            d = l % cfg.distinct
            ids, gates = moe_route(h2.float().cpu().numpy(), self.routers[d], cfg.top_k)
            calls = []
            for e, ffn in enumerate(self.moe_sets[d]):
                rows, slots = np.nonzero(ids == e)
                if rows.size:
                    ng = int(token_planner(rows.size)) if token_planner else 0
                    calls.append(CallSpec(ffn.layer, rows.astype(np.int32), gates[rows, slots].astype(np.float32),
                                          min(ng, rows.size)))
            x = x + forward_calls(calls, h2)
        return x

    # -- CUDA-graph decode ------------------------------------------------------
    # Per layer the torch part (residual add of the previous MoE output, RMSNorm,
    # QKV, RoPE, KV-cache write, attention, O-proj, RMSNorm) is ~20 small kernels
    # and host-launch bound; it is captured once per layer as a CUDA graph over
    # static buffers, with the decode position kept on the device (masked
    # attention over the whole cache, position advanced inside the last graph).
    # The sliced MoE stays a native call between replays.

    def _attention_dev(self, l, h):
        torch = self.torch
        cfg, hd = self.cfg, self.head_dim
        B = h.shape[0]
        qkv = h @ self.attn[l]["wqkv"].t()
        q = qkv[:, : cfg.heads * hd].view(B, cfg.heads, hd)
        k = qkv[:, cfg.heads * hd: (cfg.heads + cfg.kv_heads) * hd].view(B, cfg.kv_heads, hd)
        v = qkv[:, (cfg.heads + cfg.kv_heads) * hd:].view(B, cfg.kv_heads, hd)
        c = self.cos.index_select(0, self.pos_dev)  # [1, hd/2]
        s = self.sin.index_select(0, self.pos_dev)

        def rope(t):
            tf = t.float().view(*t.shape[:-1], -1, 2)
            a, b = tf[..., 0], tf[..., 1]
            return torch.stack((a * c - b * s, a * s + b * c), -1).flatten(-2).to(t.dtype)

        q, k = rope(q), rope(k)
        Kc, Vc = self.kv[l, 0, 0], self.kv[l, 1, 0]  # [kv_heads, max_seq, hd]
        Kc.index_copy_(1, self.pos_dev, k.view(cfg.kv_heads, 1, hd))
        Vc.index_copy_(1, self.pos_dev, v.view(cfg.kv_heads, 1, hd))
        qg = q.view(cfg.kv_heads, cfg.heads // cfg.kv_heads, hd)
        sc = (qg @ Kc.transpose(-1, -2)).float() * (1.0 / math.sqrt(hd))
        sc = sc.masked_fill(self.seq_idx > self.pos_dev, float("-inf"))
        o = torch.softmax(sc, dim=-1).to(q.dtype) @ Vc
        return o.reshape(B, cfg.heads * hd) @ self.attn[l]["wo"].t()

    def enable_graphs(self, x_example):
        """Capture the per-layer torch part; decode_step_graph then replays them."""
        torch = self.torch
        cfg = self.cfg
        dev = self.device
        self.pos_dev = torch.zeros(1, dtype=torch.long, device=dev)
        self.seq_idx = torch.arange(cfg.max_seq, device=dev)
        self.g_x0 = torch.zeros_like(x_example)
        self.g_mid = [torch.zeros_like(x_example) for _ in range(cfg.layers)]
        self.g_h = [torch.zeros_like(x_example) for _ in range(cfg.layers)]
        self.g_y = [torch.zeros_like(x_example) for _ in range(cfg.layers)]
        self.g_out = torch.zeros_like(x_example)

        def body(l):
            x = self.g_x0 if l == 0 else self.g_mid[l - 1] + self.g_y[l - 1]
            mid = x + self._attention_dev(l, self._rms(x, self.attn[l]["n1"]))
            self.g_mid[l].copy_(mid)
            self.g_h[l].copy_(self._rms(mid, self.attn[l]["n2"]))

        def tail():
            self.g_out.copy_(self.g_mid[-1] + self.g_y[-1])
            self.pos_dev.add_(1)

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm up the kernels off the capture
            saved = (self.kv.clone(), self.pos_dev.clone())
            for l in range(cfg.layers):
                body(l)
            self.kv.copy_(saved[0])
            self.pos_dev.copy_(saved[1])
        torch.cuda.current_stream().wait_stream(side)
        self.graphs = []
        for l in range(cfg.layers):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body(l)
            self.graphs.append(g)
        self.g_tail = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_tail):
            tail()
        torch.cuda.synchronize()

    def decode_step_graph(self, x, pos: int | None = None):
        """decode_step with the captured graphs; ``pos`` (re)sets the device position."""
        if pos is not None:
            self.pos_dev.fill_(pos)
        self.g_x0.copy_(x)
        cfg = self.cfg
        for l in range(cfg.layers):
            self.graphs[l].replay()
            self._moe(l % cfg.distinct, self.g_h[l], out=self.g_y[l])
        self.g_tail.replay()
        return self.g_out

    def release(self):
        for s in self.moe_sets:
            for e in s:
                e.layer.release()
