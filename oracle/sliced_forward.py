"""CPU ORACLE for the sliced-weight FFN path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product (``paper_2411_15715_b200``) never imports
it; its GG/CG segments run on the B200 or fail loudly.

What it restates (fp64 numpy, the reference's own arithmetic):

* ``boundaries``      -- the floor rule of slice_weights,
                         /root/reference/pkg/src/sliceplan/slicing_kernel.py:57-80
* ``activate``        -- identity / SiLU / erf-GELU, slicing_kernel.py:27-38
* ``dense_forward``   -- mlp_forward_reference, slicing_kernel.py:83-94
* ``sliced_forward``  -- mlp_forward_sliced, slicing_kernel.py:97-124
                         (fixed cc -> cg -> gg order, empty blocks skipped)
* ``execution_tags``  -- slicing_kernel.py:127-158

Extensions the reference does not pin, proven to reduce to
the reference for G=2 in tests/test_oracle.py:

* gated SwiGLU (G=3): ``act(x W1) * (x W3) @ W2`` sliced on the same columns;
* MoE top-k: softmax over the selected router logits, sum of weighted experts.

Parity is pinned: tests/golden/forward_golden.npz was produced by the reference
itself (tests/golden/make_golden.py) and tests/test_oracle.py checks this
module against every vector in it.
"""

from __future__ import annotations

import math

import numpy as np

try:  # scipy is in the image; the reference uses scipy.special.erf too
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    _erf = np.vectorize(math.erf)

ACTIVATIONS = ("identity", "silu", "gelu")


def boundaries(hidden: int, cc: float, cg: float) -> tuple[int, int]:
    """(b1, b2) with b1 = floor(cc*H), b2 = floor((cc+cg)*H), clamped."""
    b1 = min(int(math.floor(cc * hidden)), hidden)
    b2 = min(max(int(math.floor((cc + cg) * hidden)), b1), hidden)
    return b1, b2


def block_widths(hidden: int, cc: float, cg: float) -> tuple[int, int, int]:
    b1, b2 = boundaries(hidden, cc, cg)
    return b1, b2 - b1, hidden - b2


def activate(name: str, z: np.ndarray) -> np.ndarray:
    if name == "identity":
        return z
    if name == "silu":
        return z / (1.0 + np.exp(-z))
    if name == "gelu":
        return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))
    raise ValueError(f"unknown activation {name!r}")


def _hidden(x, w1, w3, act):
    h = activate(act, x @ w1)
    return h if w3 is None else h * (x @ w3)


def dense_forward(x, w1, w2, act: str, w3=None) -> np.ndarray:
    """act(x W1) [* (x W3)] @ W2, fp64."""
    x, w1, w2 = (np.asarray(a, dtype=float) for a in (x, w1, w2))
    w3 = None if w3 is None else np.asarray(w3, dtype=float)
    return _hidden(x, w1, w3, act) @ w2


def sliced_forward(x, w1, w2, act: str, cc: float, cg: float, w3=None) -> np.ndarray:
    """Sum over the (cc, cg, gg) column blocks in that order, skipping empty ones."""
    x, w1, w2 = (np.asarray(a, dtype=float) for a in (x, w1, w2))
    w3 = None if w3 is None else np.asarray(w3, dtype=float)
    hidden = w1.shape[1]
    b1, b2 = boundaries(hidden, cc, cg)
    out = np.zeros((x.shape[0], w2.shape[1]))
    for lo, hi in ((0, b1), (b1, b2), (b2, hidden)):
        if hi - lo == 0:
            continue
        part_w3 = None if w3 is None else w3[:, lo:hi]
        out = out + _hidden(x, w1[:, lo:hi], part_w3, act) @ w2[lo:hi, :]
    return out


def dense_forward_bf16_hidden(x, w1, w2, act: str, w3=None) -> np.ndarray:
    """dense_forward with the hidden activation rounded to bf16 before the down
    projection: the arithmetic of a bf16 tile / tensor-core block (the GPU
    tcgen05 GEMM pair and the host AMX CC kernel keep `a` in bf16)."""
    x, w1, w2 = (np.asarray(a, dtype=float) for a in (x, w1, w2))
    w3 = None if w3 is None else np.asarray(w3, dtype=float)
    return bf16_round(_hidden(x, w1, w3, act)) @ w2


def segment_forward(x, w1, w2, act: str, lo: int, hi: int, w3=None) -> np.ndarray:
    """One block's partial output (e.g. the CC slice alone)."""
    x, w1, w2 = (np.asarray(a, dtype=float) for a in (x, w1, w2))
    part_w3 = None if w3 is None else np.asarray(w3, dtype=float)[:, lo:hi]
    return _hidden(x, w1[:, lo:hi], part_w3, act) @ w2[lo:hi, :]


def execution_tags(hidden: int, cc: float, cg: float, tokens: int, n_g: int):
    """[(block, executor, row_start, row_stop)] as slicing_kernel.py:137-158."""
    if not 0 <= n_g <= tokens:
        raise ValueError(f"n_g must lie in [0, {tokens}], got {n_g}")
    w_cc, w_cg, w_gg = block_widths(hidden, cc, cg)
    split = tokens - n_g
    tags = []
    if w_cc:
        if split:
            tags.append(("cc", "cpu", 0, split))
        if n_g:
            tags.append(("cg_prime", "gpu", split, tokens))
    if w_cg:
        tags.append(("cg", "gpu", 0, tokens))
    if w_gg:
        tags.append(("gg", "gpu", 0, tokens))
    return tags


def route_topk(logits: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Top-k experts per token (ties -> lower id) and softmax over the k logits."""
    logits = np.asarray(logits, dtype=float)
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    picked = np.take_along_axis(logits, order, axis=1)
    e = np.exp(picked - picked.max(axis=1, keepdims=True))
    return order, e / e.sum(axis=1, keepdims=True)


def moe_forward(x, experts, router_w, k: int, act: str = "silu", rates=None) -> np.ndarray:
    """Top-k MoE layer: experts = [(w1, w3|None, w2)], rates = [(cc, cg)] or None
    (dense).  Expert outputs are accumulated token by token in ascending
    expert-rank order."""
    x = np.asarray(x, dtype=float)
    ids, gates = route_topk(x @ np.asarray(router_w, dtype=float), k)
    out = np.zeros((x.shape[0], np.asarray(experts[0][2]).shape[1]))
    for t in range(x.shape[0]):
        for slot in range(k):
            e = int(ids[t, slot])
            w1, w3, w2 = experts[e]
            if rates is None:
                y = dense_forward(x[t : t + 1], w1, w2, act, w3)
            else:
                y = sliced_forward(x[t : t + 1], w1, w2, act, rates[e][0], rates[e][1], w3)
            out[t] += gates[t, slot] * y[0]
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (for feeding the
    oracle exactly the values a bf16 kernel sees)."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def max_rel_error(got: np.ndarray, ref: np.ndarray) -> float:
    """max|got - ref| / max|ref| -- the north-star parity metric."""
    ref = np.asarray(ref, dtype=float)
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    err = float(np.max(np.abs(np.asarray(got, dtype=float) - ref))) if ref.size else 0.0
    return err / scale if scale > 0 else err
