"""Sliced-weight FFN execution on B200 -- the drop-in for slicing_kernel.py.

Reference API (/root/reference/pkg/src/sliceplan/slicing_kernel.py) and what
each name does here:

=========================  =====================================================
``slice_weights``          same floor rule and views (:57-80); additionally the
                           returned ``SlicedWeights`` places itself on first use:
                           GG block -> HBM, CG block -> pinned host (streamed),
                           CC block -> pinned host (run on host threads)
``mlp_forward_sliced``     same signature (:97-124); runs GG/CG on the GPU
                           through libsliced, CC on host threads, merges
``mlp_forward_reference``  same signature (:83-94); the dense forward, i.e. the
                           whole hidden dimension as one GG block on the GPU
``execution_tags``         same task list (:127-158); it is also the dispatch
                           table the runtime executes (cc rows on the CPU,
                           cg_prime rows on the GPU)
``max_recombination_error``same random sweep (:161-190) with the GPU sliced
                           forward against the GPU dense forward
=========================  =====================================================

Errors are the reference classes (ShapeMismatch, TokenCountOutOfRange) and
are raised before anything runs.  numpy inputs follow the reference contract
(float64 in, float64 out; arithmetic is fp32 on the device); torch CUDA
tensors stay on the device (bf16 or fp32).

Beyond the reference: ``SlicedFFN`` (a placed layer built straight from
nn.Linear-layout weights, optionally gated/SwiGLU) and ``SlicedMoE`` (top-k
experts, each with its own split) -- the Mixtral-shaped workloads of the
benchmarks.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as nat
from .errors import ShapeMismatch, TokenCountOutOfRange
from .schedule import SlicingRates

_BLOCK_NAMES = ("cc", "cg", "gg")


class Activation(enum.Enum):
    IDENTITY = "identity"
    SILU = "silu"
    GELU = "gelu"


def _act_name(activation) -> str:
    if isinstance(activation, Activation):
        return activation.value
    if isinstance(activation, str) and activation in nat.ACT_CODES:
        return activation
    raise ValueError(f"unknown activation {activation!r}")


def split_boundaries(hidden: int, rates: SlicingRates) -> tuple[int, int]:
    """b1 = floor(cc*H), b2 = floor((cc+cg)*H), clamped (slicing_kernel.py:71-74)."""
    b1 = min(int(math.floor(rates.cc * hidden)), hidden)
    b2 = min(max(int(math.floor((rates.cc + rates.cg) * hidden)), b1), hidden)
    return b1, b2


# ---------------------------------------------------------------------------
# dtype helpers (numpy has no bfloat16: bf16 travels as its uint16 bit pattern)


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float -> bfloat16 bit patterns (uint16)."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if f.size >= 4096 and nat.available():
        # native AVX-512 cast (~50x faster than the numpy form below on a prompt); not
        # torch's: its spinning OpenMP workers would steal the CC block's cores
        out = np.empty(f.shape, dtype=np.uint16)
        nat.check(nat.lib().sp_round_bf16(f.ctypes.data, out.ctypes.data, f.size))
        return out
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return u


def from_bf16_bits(u: np.ndarray) -> np.ndarray:
    return (np.asarray(u, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _dtype_code(dtype: str) -> int:
    if dtype in ("f32", "float32", "fp32"):
        return nat.SP_F32
    if dtype in ("bf16", "bfloat16"):
        return nat.SP_BF16
    raise ValueError(f"weight dtype must be 'f32' or 'bf16', got {dtype!r}")


def _host_weights(a, code: int) -> np.ndarray:
    """Contiguous host array in the storage dtype (float32 or bf16 bits)."""
    try:
        import torch

        if isinstance(a, torch.Tensor):
            t = a.detach()
            if code == nat.SP_BF16:
                return t.to("cpu", torch.bfloat16).contiguous().view(torch.int16).numpy().view(np.uint16)
            return t.to("cpu", torch.float32).contiguous().numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(a)
    if code == nat.SP_BF16:
        return a if a.dtype == np.uint16 and a.flags.c_contiguous else to_bf16_bits(a)
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------
# a placed layer


class NativeLayer:
    """One FFN instance placed by libsliced (GG in HBM, CC/CG in pinned host).

    w1t, w3t: [H, M] (the reference's w1 / w3 transposed: hidden unit h owns row
    h); w2: [H, N] (the reference's own w2 layout)."""

    def __init__(self, w1t, w2, b1: int, b2: int, activation="silu", w3t=None,
                 dtype: str = "bf16", chunk_rows: int = 0, device: int | None = None):
        code = _dtype_code(dtype)
        a1 = _host_weights(w1t, code)
        a2 = _host_weights(w2, code)
        a3 = None if w3t is None else _host_weights(w3t, code)
        if a1.ndim != 2 or a2.ndim != 2:
            raise ShapeMismatch("w1t and w2 must be 2-D matrices")
        hidden, model = a1.shape
        hidden2, out = a2.shape
        if hidden2 != hidden:
            raise ShapeMismatch(f"w1t has {hidden} rows but w2 has {hidden2}; the hidden dim must match")
        if a3 is not None and a3.shape != a1.shape:
            raise ShapeMismatch(f"w3t is {a3.shape}, expected {a1.shape}")
        nat.init(device)
        self.model_dim, self.hidden_dim, self.out_dim = int(model), int(hidden), int(out)
        self.b1, self.b2 = int(b1), int(b2)
        self.gated = a3 is not None
        self.activation = _act_name(activation)
        self.dtype = "bf16" if code == nat.SP_BF16 else "f32"
        desc = nat.LayerDesc(self.model_dim, self.hidden_dim, self.out_dim, int(self.gated),
                             nat.ACT_CODES[self.activation], code, int(chunk_rows), self.b1, self.b2)
        handle = C.c_void_p()
        nat.check(nat.lib().sp_layer_create(
            C.byref(desc), a1.ctypes.data, None if a3 is None else a3.ctypes.data, a2.ctypes.data,
            C.byref(handle)))
        self._h = handle
        cr = C.c_int32(0)  # the runtime picks chunk_rows when 0 was asked for
        nat.check(nat.lib().sp_layer_image_sizes(handle, None, None, C.byref(cr)))
        self.chunk_rows = int(cr.value)

    @classmethod
    def _adopt(cls, handle: C.c_void_p, model_dim: int, hidden_dim: int, out_dim: int, b1: int, b2: int,
               gated: bool, activation: str, dtype: str, chunk_rows: int) -> "NativeLayer":
        """Wrap a layer the runtime created (images, file, re-slice)."""
        obj = cls.__new__(cls)
        obj.model_dim, obj.hidden_dim, obj.out_dim = int(model_dim), int(hidden_dim), int(out_dim)
        obj.b1, obj.b2 = int(b1), int(b2)
        obj.gated, obj.activation, obj.dtype = bool(gated), _act_name(activation), dtype
        obj.chunk_rows = int(chunk_rows)
        obj._h = handle
        return obj

    def desc(self, b1: int | None = None, b2: int | None = None) -> "nat.LayerDesc":
        return nat.LayerDesc(self.model_dim, self.hidden_dim, self.out_dim, int(self.gated),
                             nat.ACT_CODES[self.activation], _dtype_code(self.dtype), self.chunk_rows,
                             self.b1 if b1 is None else int(b1), self.b2 if b2 is None else int(b2))

    def meta(self) -> dict:
        """Everything besides the two images that recreates this layer."""
        return {"model_dim": self.model_dim, "hidden_dim": self.hidden_dim, "out_dim": self.out_dim,
                "b1": self.b1, "b2": self.b2, "gated": self.gated, "activation": self.activation,
                "dtype": self.dtype, "chunk_rows": self.chunk_rows}

    def image_sizes(self) -> tuple[int, int]:
        gg, host = C.c_size_t(), C.c_size_t()
        nat.check(nat.lib().sp_layer_image_sizes(self.handle, C.byref(gg), C.byref(host), None))
        return gg.value, host.value

    def export_images(self) -> tuple[np.ndarray, np.ndarray]:
        """(GG image as laid out in HBM, pinned host region) as uint8 arrays."""
        gg_n, host_n = self.image_sizes()
        gg, host = np.empty(gg_n, dtype=np.uint8), np.empty(host_n, dtype=np.uint8)
        nat.check(nat.lib().sp_layer_export(self.handle, gg.ctypes.data if gg_n else None,
                                            host.ctypes.data if host_n else None))
        return gg, host

    @classmethod
    def from_images(cls, meta: dict, gg: np.ndarray, host: np.ndarray, device: int | None = None) -> "NativeLayer":
        nat.init(device)
        obj = cls._adopt(None, **meta)
        handle = C.c_void_p()
        gg = np.ascontiguousarray(gg, dtype=np.uint8)
        host = np.ascontiguousarray(host, dtype=np.uint8)
        nat.check(nat.lib().sp_layer_create_from_images(
            C.byref(obj.desc()), gg.ctypes.data if gg.size else None, gg.size,
            host.ctypes.data if host.size else None, host.size, C.byref(handle)))
        obj._h = handle
        return obj

    @classmethod
    def load_file(cls, meta: dict, path: str, gg_offset: int, gg_bytes: int, host_offset: int, host_bytes: int,
                  device: int | None = None) -> "NativeLayer":
        nat.init(device)
        obj = cls._adopt(None, **meta)
        handle = C.c_void_p()
        nat.check(nat.lib().sp_layer_load_file(C.byref(obj.desc()), str(path).encode(), int(gg_offset),
                                               int(gg_bytes), int(host_offset), int(host_bytes), C.byref(handle)))
        obj._h = handle
        return obj

    def reslice(self, b1: int, b2: int) -> "NativeLayer":
        """A new layer with boundaries (b1, b2) from this one's weights."""
        if not 0 <= b1 <= b2 <= self.hidden_dim:
            raise ValueError(f"boundaries must satisfy 0 <= b1 <= b2 <= {self.hidden_dim}, got ({b1}, {b2})")
        handle = C.c_void_p()
        nat.check(nat.lib().sp_layer_reslice(self.handle, int(b1), int(b2), C.byref(handle)))
        meta = self.meta()
        meta.update(b1=int(b1), b2=int(b2))
        return NativeLayer._adopt(handle, **meta)

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("layer was released")
        return self._h

    def placed_bytes(self) -> dict[str, int]:
        gg, cg, cc = C.c_size_t(), C.c_size_t(), C.c_size_t()
        nat.check(nat.lib().sp_layer_bytes(self.handle, C.byref(gg), C.byref(cg), C.byref(cc)))
        return {"gg": gg.value, "cg": cg.value, "cc": cc.value}

    @property
    def block_widths(self) -> tuple[int, int, int]:
        w = (C.c_int64 * 3)()
        nat.check(nat.lib().sp_layer_widths(self.handle, w))
        return int(w[0]), int(w[1]), int(w[2])

    def release(self) -> None:
        if getattr(self, "_h", None) is not None and nat._lib is not None:
            nat.lib().sp_layer_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.release()
        except Exception:
            pass

    def cc_forward_host(self, x: np.ndarray, threads: int = 0) -> np.ndarray:
        """The CC block alone on host threads (no GPU involved)."""
        xa, code = _host_activations(x, self.dtype)
        T = xa.shape[0]
        y = np.zeros((T, self.out_dim), dtype=np.float32)
        nat.check(nat.lib().sp_cc_forward_host(
            self.handle, xa.ctypes.data, code, T,
            y.ctypes.data_as(C.POINTER(C.c_float)), int(threads)))
        return y


def _host_activations(x, dtype: str) -> tuple[np.ndarray, int]:
    if dtype == "bf16":
        return to_bf16_bits(x), nat.SP_BF16
    return np.ascontiguousarray(np.asarray(x), dtype=np.float32), nat.SP_F32


def _host_input(x, dtype: str) -> tuple[np.ndarray, int, int]:
    """Host activations for a forward with SP_IO_HOST: (array, xdtype, extra flags).
    bf16 layers get f32 x plus SP_X_TO_BF16 -- the runtime rounds it while
    staging, into persistent pinned memory (no caller-side cast / allocation)."""
    a = np.asarray(x)
    if dtype == "bf16" and a.dtype != np.uint16:
        return np.ascontiguousarray(a, dtype=np.float32), nat.SP_F32, nat.SP_X_TO_BF16
    xh, code = _host_activations(a, dtype)
    return xh, code, 0


@dataclass
class CallSpec:
    """One layer application inside a batched forward (sp_call)."""

    layer: NativeLayer
    token_ids: Sequence[int] | None = None
    gates: Sequence[float] | None = None
    n_g: int = 0
    tokens: int | None = None


def forward_calls(calls: Sequence[CallSpec], x, out=None, host_threads_off: bool = False):
    """y[t] = sum over calls of gate * layer(x[t]); one sp_forward_batch.

    ``x`` is a torch CUDA tensor (device I/O, result on the device, ordered on
    the current stream), a torch CPU tensor or a numpy array (host I/O).
    """
    if not calls:
        raise ValueError("forward_calls needs at least one call")
    M, N = calls[0].layer.model_dim, calls[0].layer.out_dim
    torch = _maybe_torch()
    on_device = torch is not None and isinstance(x, torch.Tensor) and x.is_cuda
    keep = []
    arr = (nat.Call * len(calls))()
    for i, c in enumerate(calls):
        T = x.shape[0]
        if c.token_ids is not None:
            ids = np.ascontiguousarray(c.token_ids, dtype=np.int32)
            tokens = ids.shape[0]
            ids_p = ids.ctypes.data_as(C.POINTER(C.c_int32))
            keep.append(ids)
        else:
            tokens = T if c.tokens is None else int(c.tokens)
            ids_p = None
        if c.gates is not None:
            g = np.ascontiguousarray(c.gates, dtype=np.float32)
            if g.shape[0] != tokens:
                raise ShapeMismatch(f"call {i}: {g.shape[0]} gates for {tokens} tokens")
            gates_p = g.ctypes.data_as(C.POINTER(C.c_float))
            keep.append(g)
        else:
            gates_p = None
        arr[i] = nat.Call(c.layer.handle, tokens, ids_p, gates_p, int(c.n_g))
    flags = nat.SP_NO_CC_THREADS if host_threads_off else 0
    if on_device:
        if x.dim() != 2 or x.shape[1] != M:
            raise ShapeMismatch(f"input is {tuple(x.shape)} but the layer expects {M} features")
        x = x.contiguous()
        if x.dtype not in (torch.bfloat16, torch.float32):
            x = x.float()
        xcode = nat.SP_BF16 if x.dtype == torch.bfloat16 else nat.SP_F32
        if out is None:
            out = torch.empty((x.shape[0], N), dtype=x.dtype, device=x.device)
        ycode = nat.SP_BF16 if out.dtype == torch.bfloat16 else nat.SP_F32
        nat.init(x.device.index)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        nat.check(nat.lib().sp_forward_batch(arr, len(calls), x.data_ptr(), xcode, x.shape[0],
                                             out.data_ptr(), ycode, flags, C.c_void_p(stream)))
        return out
    # host I/O
    if torch is not None and isinstance(x, torch.Tensor):
        x = x.detach().float().numpy()
    xh, xcode, xflag = _host_input(x, calls[0].layer.dtype)
    if xh.ndim != 2 or xh.shape[1] != M:
        raise ShapeMismatch(f"input is {xh.shape} but the layer expects {M} features")
    y = np.empty((xh.shape[0], N), dtype=np.float32) if out is None else out
    nat.check(nat.lib().sp_forward_batch(arr, len(calls), xh.ctypes.data, xcode, xh.shape[0],
                                         y.ctypes.data, nat.SP_F32, flags | xflag | nat.SP_IO_HOST, None))
    return y


def _maybe_torch():
    try:
        import torch

        return torch
    except ImportError:  # pragma: no cover
        return None


# ---------------------------------------------------------------------------
# reference-compatible operator API


@dataclass(frozen=True)
class SlicedWeights:
    """Column blocks of w1 (and w3) and the matching row blocks of w2.

    Same fields as slicing_kernel.py:41-54; ``dtype`` / ``chunk_rows`` choose the
    placement, which happens lazily on the first forward (one NativeLayer per
    activation, cached in ``_placed``)."""

    w1_blocks: tuple[np.ndarray, np.ndarray, np.ndarray]
    w2_blocks: tuple[np.ndarray, np.ndarray, np.ndarray]
    rates: SlicingRates
    boundaries: tuple[int, int]
    w3_blocks: tuple[np.ndarray, np.ndarray, np.ndarray] | None = None
    dtype: str = "f32"
    chunk_rows: int = 0
    _placed: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def block_widths(self) -> tuple[int, int, int]:
        b1, b2 = self.boundaries
        hidden = sum(b.shape[1] for b in self.w1_blocks)
        return (b1, b2 - b1, hidden - b2)

    @property
    def model_dim(self) -> int:
        return self.w1_blocks[0].shape[0]

    def placed(self, activation, device: int | None = None) -> NativeLayer:
        act = _act_name(activation)
        # the library binds one device per process: a layer placed on one GPU is
        # never silently reused for inputs on another
        bound = nat.current_device()
        if device is not None and bound is not None and device != bound:
            raise ValueError(f"input is on cuda:{device} but this process's sliced layers live on cuda:{bound}")
        key = (act, device if device is not None else bound)
        layer = self._placed.get(key)
        if layer is None:
            w1 = np.concatenate(self.w1_blocks, axis=1)
            w2 = np.concatenate(self.w2_blocks, axis=0)
            w3 = None if self.w3_blocks is None else np.concatenate(self.w3_blocks, axis=1)
            b1, b2 = self.boundaries
            layer = NativeLayer(w1.T, w2, b1, b2, act, None if w3 is None else w3.T,
                                dtype=self.dtype, chunk_rows=self.chunk_rows, device=device)
            self._placed[(act, nat.current_device())] = layer
        return layer


def slice_weights(w1, w2, rates: SlicingRates, w3=None, *, dtype: str = "f32",
                  chunk_rows: int = 0) -> SlicedWeights:
    """Partition w1 (and w3) columns and w2 rows at floor(rate * H) boundaries;
    the rounding remainder lands in the GPU-resident block (slicing_kernel.py:57-80)."""
    w1 = np.asarray(w1, dtype=float)
    w2 = np.asarray(w2, dtype=float)
    if w1.ndim != 2 or w2.ndim != 2:
        raise ShapeMismatch("w1 and w2 must be 2-D matrices")
    hidden = w1.shape[1]
    if w2.shape[0] != hidden:
        raise ShapeMismatch(
            f"w1 has {hidden} columns but w2 has {w2.shape[0]} rows; the hidden dim must match"
        )
    w3_blocks = None
    if w3 is not None:
        w3 = np.asarray(w3, dtype=float)
        if w3.shape != w1.shape:
            raise ShapeMismatch(f"w3 is {w3.shape}, expected {w1.shape}")
    b1, b2 = split_boundaries(hidden, rates)
    if w3 is not None:
        w3_blocks = (w3[:, :b1], w3[:, b1:b2], w3[:, b2:])
    return SlicedWeights(
        w1_blocks=(w1[:, :b1], w1[:, b1:b2], w1[:, b2:]),
        w2_blocks=(w2[:b1, :], w2[b1:b2, :], w2[b2:, :]),
        rates=rates,
        boundaries=(b1, b2),
        w3_blocks=w3_blocks,
        dtype=dtype,
        chunk_rows=chunk_rows,
    )


def _as_host_or_device(x):
    torch = _maybe_torch()
    if torch is not None and isinstance(x, torch.Tensor):
        return x, x.is_cuda
    return np.asarray(x, dtype=float), False


def mlp_forward_sliced(x, sliced: SlicedWeights, activation: Activation, n_g: int = 0):
    """Forward summed over the cc/cg/gg blocks (slicing_kernel.py:97-124).

    The last ``n_g`` rows run the CC columns on the GPU (cg_prime) and the
    first ``T - n_g`` on host threads, exactly the split ``execution_tags``
    describes; the numbers do not depend on ``n_g`` beyond rounding."""
    x, on_device = _as_host_or_device(x)
    if x.ndim != 2 or x.shape[1] != sliced.model_dim:
        raise ShapeMismatch(
            f"input is {tuple(x.shape)} but the sliced weights expect {sliced.model_dim} features"
        )
    tokens = x.shape[0]
    if not 0 <= n_g <= tokens:
        raise TokenCountOutOfRange(f"n_g must lie in [0, {tokens}], got {n_g}")
    layer = sliced.placed(activation, x.device.index if on_device else None)
    y = forward_calls([CallSpec(layer, n_g=n_g)], x)
    return y if on_device else np.asarray(y, dtype=float)


def mlp_forward_reference(x, w1, w2, activation: Activation, w3=None):
    """Dense act(x W1) W2 (slicing_kernel.py:83-94): the whole hidden dimension
    placed as one GG block on the GPU."""
    x, on_device = _as_host_or_device(x)
    w1 = np.asarray(w1, dtype=float)
    w2 = np.asarray(w2, dtype=float)
    if x.ndim != 2 or x.shape[1] != w1.shape[0]:
        raise ShapeMismatch(f"input is {tuple(x.shape)} but w1 expects {w1.shape[0]} features")
    if w1.shape[1] != w2.shape[0]:
        raise ShapeMismatch("w1 columns must match w2 rows")
    sliced = slice_weights(w1, w2, SlicingRates(0.0, 0.0, 1.0), w3)
    return mlp_forward_sliced(x, sliced, activation)


@dataclass(frozen=True)
class ExecutorTask:
    """Who computes which block for which token rows (slicing_kernel.py:127-134)."""

    block: str
    executor: str
    row_start: int
    row_stop: int


def execution_tags(sliced: SlicedWeights, tokens: int, n_g: int) -> list[ExecutorTask]:
    """Dispatch table of one forward (slicing_kernel.py:137-158)."""
    if not 0 <= n_g <= tokens:
        raise TokenCountOutOfRange(f"n_g must lie in [0, {tokens}], got {n_g}")
    w_cc, w_cg, w_gg = sliced.block_widths
    kept = tokens - n_g
    tasks: list[ExecutorTask] = []
    if w_cc and kept:
        tasks.append(ExecutorTask("cc", "cpu", 0, kept))
    if w_cc and n_g:
        tasks.append(ExecutorTask("cg_prime", "gpu", kept, tokens))
    if w_cg:
        tasks.append(ExecutorTask("cg", "gpu", 0, tokens))
    if w_gg:
        tasks.append(ExecutorTask("gg", "gpu", 0, tokens))
    return tasks


def max_recombination_error(seed: int, trials: int, max_dim: int = 64, max_tokens: int = 8) -> float:
    """Worst |sliced - dense| over the reference's random sweep
    (slicing_kernel.py:161-190), both sides on the GPU."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        tokens = int(rng.integers(1, max_tokens + 1))
        m = int(rng.integers(2, max_dim + 1))
        h = int(rng.integers(2, max_dim + 1))
        out_dim = int(rng.integers(2, max_dim + 1))
        x = rng.uniform(-1.0, 1.0, size=(tokens, m))
        w1 = rng.uniform(-1.0, 1.0, size=(m, h))
        w2 = rng.uniform(-1.0, 1.0, size=(h, out_dim))
        raw = rng.uniform(0.0, 1.0, size=3)
        raw /= raw.sum()
        rates = SlicingRates(cc=raw[0], cg=raw[1], gg=1.0 - raw[0] - raw[1])
        n_g = int(rng.integers(0, tokens + 1))
        sliced = slice_weights(w1, w2, rates)
        for activation in Activation:
            ref = mlp_forward_reference(x, w1, w2, activation)
            got = mlp_forward_sliced(x, sliced, activation, n_g)
            worst = max(worst, float(np.max(np.abs(got - ref))))
    return worst


# ---------------------------------------------------------------------------
# Mixtral-shaped runtime objects


class SlicedFFN:
    """A gated (SwiGLU) or plain FFN placed by rates, from nn.Linear-layout weights.

    w1t, w3t: [H, M]; w2t: [N, H] (HF Mixtral ``w1``/``w3``/``w2``)."""

    def __init__(self, w1t, w2t, rates: SlicingRates | None = None, w3t=None,
                 activation="silu", dtype: str = "bf16", boundaries: tuple[int, int] | None = None,
                 chunk_rows: int = 0, device: int | None = None):
        hidden = int(w1t.shape[0])
        if boundaries is None:
            if rates is None:
                raise ValueError("give rates or boundaries")
            boundaries = split_boundaries(hidden, rates)
        self.rates = rates
        self.layer = NativeLayer(w1t, _transpose(w2t), boundaries[0], boundaries[1], activation, w3t,
                                 dtype=dtype, chunk_rows=chunk_rows, device=device)

    @property
    def block_widths(self) -> tuple[int, int, int]:
        return self.layer.block_widths

    @classmethod
    def from_layer(cls, layer: NativeLayer, rates: SlicingRates | None = None) -> "SlicedFFN":
        obj = cls.__new__(cls)
        obj.rates = rates
        obj.layer = layer
        return obj

    def reslice(self, rates: SlicingRates) -> "SlicedFFN":
        """Re-place under new rates (same floor rule as slice_weights)."""
        b1, b2 = split_boundaries(self.layer.hidden_dim, rates)
        return SlicedFFN.from_layer(self.layer.reslice(b1, b2), rates)

    def forward(self, x, n_g: int = 0, out=None):
        if not 0 <= n_g <= x.shape[0]:
            raise TokenCountOutOfRange(f"n_g must lie in [0, {x.shape[0]}], got {n_g}")
        return forward_calls([CallSpec(self.layer, n_g=n_g)], x, out)

    __call__ = forward


def _transpose(a):
    """[N, H] -> contiguous [H, N] (torch's multi-threaded copy for tensors)."""
    torch = _maybe_torch()
    if torch is not None and isinstance(a, torch.Tensor):
        return a.detach().t().contiguous()
    return np.ascontiguousarray(np.asarray(a).T)


def route_topk(logits: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Top-k expert ids (ties -> lower id) and the softmax over the k logits of
    precomputed logits (planning helpers; MoE layers route with ``moe_route``)."""
    logits = np.asarray(logits, dtype=np.float64)
    ids = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    top = np.take_along_axis(logits, ids, axis=1)
    e = np.exp(top - top.max(axis=1, keepdims=True))
    return ids, e / e.sum(axis=1, keepdims=True)


def moe_route(x, router_w, top_k: int) -> tuple[np.ndarray, np.ndarray]:
    """The runtime's router (libsliced sp_moe_route): fp64 logits x @ router_w
    with the router held in fp32, top-k with ties to the lower expert id,
    softmax over the k logits.  Every MoE path (sp_moe_forward, SlicedMoE.plan,
    expert_parallel.route_local) routes through this one routine, so a token
    picks the same experts whichever path runs it."""
    if getattr(x, "dtype", None) == np.uint16:  # bf16 bit patterns
        xh, code = np.ascontiguousarray(x), nat.SP_BF16
    else:
        xh, code = np.ascontiguousarray(np.asarray(x), dtype=np.float32), nat.SP_F32
    router = np.ascontiguousarray(router_w, dtype=np.float32)
    T, M = xh.shape
    ids = np.empty((T, top_k), dtype=np.int32)
    gates = np.empty((T, top_k), dtype=np.float32)
    nat.check(nat.lib().sp_moe_route(router.ctypes.data_as(C.POINTER(C.c_float)), M, router.shape[1], int(top_k),
                                     xh.ctypes.data, code, T, ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                     gates.ctypes.data_as(C.POINTER(C.c_float))))
    return ids, gates


class MoEDispatch:
    """One MoE layer's native call (sp_moe_forward) with its arguments prepared
    once: the layer-handle array, the float32 router and the bound function.
    A decode step then costs a few microseconds of Python instead of ~150
    (per-call router conversion, ctypes array building, library lookup).
    ``layers[e] is None`` marks an expert owned by another rank."""

    def __init__(self, layers: Sequence["NativeLayer | None"], router_w, top_k: int):
        self.layers = list(layers)  # keeps the handles alive
        first = next(l for l in self.layers if l is not None)
        self.N, self.dtype = first.out_dim, first.dtype
        self.E, self.k = len(self.layers), int(top_k)
        self.arr = (C.c_void_p * self.E)(*[None if l is None else l.handle.value for l in self.layers])
        self.router = np.ascontiguousarray(router_w, dtype=np.float32)
        self.rp = self.router.ctypes.data_as(C.POINTER(C.c_float))
        self.fn = nat.lib().sp_moe_forward
        self.torch = _maybe_torch()

    def __call__(self, x, out=None):
        torch = self.torch
        if torch is not None and isinstance(x, torch.Tensor) and x.is_cuda:
            if not x.is_contiguous():
                x = x.contiguous()
            if x.dtype not in (torch.bfloat16, torch.float32):
                x = x.float()
            xcode = nat.SP_BF16 if x.dtype == torch.bfloat16 else nat.SP_F32
            if out is None:
                out = torch.empty((x.shape[0], self.N), dtype=x.dtype, device=x.device)
            ycode = nat.SP_BF16 if out.dtype == torch.bfloat16 else nat.SP_F32
            stream = torch.cuda.current_stream(x.device).cuda_stream
            st = self.fn(self.arr, self.E, self.rp, self.k, x.data_ptr(), xcode, x.shape[0], out.data_ptr(), ycode,
                         0, C.c_void_p(stream))
            if st:
                nat.check(st)
            return out
        if torch is not None and isinstance(x, torch.Tensor):
            x = x.detach().float().numpy()
        xh, xcode, xflag = _host_input(x, self.dtype)
        y = np.empty((xh.shape[0], self.N), dtype=np.float32) if out is None else out
        st = self.fn(self.arr, self.E, self.rp, self.k, xh.ctypes.data, xcode, xh.shape[0], y.ctypes.data,
                     nat.SP_F32, nat.SP_IO_HOST | xflag, None)
        if st:
            nat.check(st)
        return y


def moe_forward(layers: Sequence["NativeLayer | None"], router_w, top_k: int, x, out=None):
    """One MoE FFN layer in one native call (sp_moe_forward): route in the
    runtime (the single read-back of x serves the router and the CC blocks),
    then one batched forward over the active experts.  ``layers[e] is None``
    marks an expert owned by another rank.  (Repeated calls on the same layer:
    keep a ``MoEDispatch``.)"""
    return MoEDispatch(layers, router_w, top_k)(x, out)


class SlicedMoE:
    """Top-k MoE layer over SlicedFFN experts, each with its own CC/CG/GG split.

    Routing runs on the host in fp64 (the expert ids must be host-visible to
    drive the CG streamer, SURVEY.md section 7 hard part 6); all active experts
    then go through ONE sp_forward_batch so their GG kernels, CG chunk copies
    and CC host work overlap."""

    def __init__(self, experts: Sequence[SlicedFFN], router_w, top_k: int = 2):
        self.experts = list(experts)
        self.router_w = np.ascontiguousarray(router_w, dtype=np.float32)  # [M, E], as sp_moe_route holds it
        if self.router_w.shape[1] != len(self.experts):
            raise ShapeMismatch("router_w must have one column per expert")
        self.top_k = int(top_k)

    def plan(self, x_host: np.ndarray, n_g: dict[int, int] | None = None) -> list[CallSpec]:
        ids, gates = moe_route(np.asarray(x_host, dtype=np.float32), self.router_w, self.top_k)
        calls = []
        for e in range(len(self.experts)):
            rows, slots = np.nonzero(ids == e)
            if rows.size == 0:
                continue
            order = np.argsort(rows, kind="stable")
            rows, slots = rows[order], slots[order]
            ng = min(int((n_g or {}).get(e, 0)), rows.size)
            calls.append(CallSpec(self.experts[e].layer, rows.astype(np.int32),
                                  gates[rows, slots].astype(np.float32), ng))
        return calls

    def forward(self, x, n_g: dict[int, int] | None = None, out=None):
        if not n_g:
            # routing + dispatch in the runtime: one native call per layer
            if getattr(self, "_dispatch", None) is None:
                self._dispatch = MoEDispatch([e.layer for e in self.experts], self.router_w, self.top_k)
            return self._dispatch(x, out)
        torch = _maybe_torch()
        if torch is not None and isinstance(x, torch.Tensor):
            x_host = x.detach().float().cpu().numpy()
        else:
            x_host = np.asarray(x, dtype=np.float64)
        return forward_calls(self.plan(x_host, n_g), x, out)

    __call__ = forward


def place_experts(weights: Iterable[tuple], rates: Sequence[SlicingRates], **kw) -> list[SlicedFFN]:
    """[(w1t, w3t, w2t)] + per-expert rates -> placed SlicedFFN experts."""
    return [SlicedFFN(w1t, w2t, r, w3t=w3t, **kw) for (w1t, w3t, w2t), r in zip(weights, rates)]
