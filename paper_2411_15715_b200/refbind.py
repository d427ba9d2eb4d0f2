"""Reference-side ctypes binding of libsliced.so -- the module a maintainer of
the reference would add as ``sliceplan/_b200.py`` to swap only the forward.

It replaces the body of ``mlp_forward_sliced``
(``/root/reference/pkg/src/sliceplan/slicing_kernel.py:97-124``) and keeps
everything else of the reference as is: ``slice_weights`` (``:57-80``) still
returns views, and this module places each ``SlicedWeights`` on the device
ONCE (GG block to HBM, CC/CG blocks to pinned host memory) and reuses the
placement on every later forward.  Validation and exception classes follow
``slicing_kernel.py:110-118`` / ``errors.py:24-29``: argument errors are
raised before any device work.

Self-contained on purpose: it imports nothing from this package except the
exception classes through ``from .errors import ...``, which resolves to
``sliceplan.errors`` when the file is dropped into the reference (both
modules define ``ShapeMismatch`` and ``TokenCountOutOfRange``).  The only
other dependency is numpy.  ``tests/test_refbind.py`` drives it through a
stand-in with the reference's signature.

``use_reference_cc(True)`` runs every CC block through the reference's own
CPU expression (``_activate(x @ w1_cc) @ w2_cc`` in fp64 numpy,
``slicing_kernel.py:33-38,119-123``) via the ABI's CC-executor hook
(``sp_set_cc_executor``), concurrently with the GPU's GG / CG work -- the
north star's "CC slice on host threads through the reference CPU code".  The
default is the library's native AVX-512 / AMX CC kernels.

Library location: ``$SLICED_LIB``, else ``_native/libsliced.so`` next to this
file.  Device: ``$SLICED_DEVICE`` (default 0).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading
import weakref
from pathlib import Path

import numpy as np

from .errors import ShapeMismatch, TokenCountOutOfRange

_SP_F32 = 0
_SP_IO_HOST = 1
_ACT = {"identity": 0, "silu": 1, "gelu": 2}


class _Desc(C.Structure):  # sp_layer_desc (include/sliced.h)
    _fields_ = [("model_dim", C.c_int64), ("hidden_dim", C.c_int64), ("out_dim", C.c_int64),
                ("gated", C.c_int32), ("act", C.c_int32), ("wdtype", C.c_int32),
                ("chunk_rows", C.c_int32), ("b1", C.c_int64), ("b2", C.c_int64)]


class _Call(C.Structure):  # sp_call (include/sliced.h)
    _fields_ = [("layer", C.c_void_p), ("tokens", C.c_int64),
                ("token_ids", C.POINTER(C.c_int32)), ("gates", C.POINTER(C.c_float)),
                ("n_g", C.c_int64)]


# sp_cc_fn (include/sliced.h)
_CC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_float), C.c_int64, C.c_int64,
                     C.POINTER(C.c_float), C.c_int64)

_lib = None
_lock = threading.RLock()  # a GC finalizer may run while it is held
# id(SlicedWeights) -> (weakref to it, {activation code: sp_layer_t, ...}, out_dim)
_placed: dict[int, tuple] = {}
# sp_layer_t -> (w1 cc block [M, b1], w2 cc block [b1, N], activation name): the
# reference CC executor's operands (views of the caller's arrays)
_cc_blocks: dict[int, tuple] = {}
_cc_callback = None


def _library():
    """Load the library and declare every signature BEFORE the first call
    (sp_last_error must return a C string for the error path to work)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("SLICED_LIB") or str(Path(__file__).resolve().parent / "_native" / "libsliced.so")
        if not Path(path).exists():
            raise RuntimeError(f"{path} is missing: the sliced forward has no CPU fallback")
        lib = C.CDLL(path)
        lib.sp_last_error.restype = C.c_char_p
        lib.sp_last_error.argtypes = []
        lib.sp_init.restype = C.c_int
        lib.sp_init.argtypes = [C.c_int, C.c_int]
        lib.sp_layer_create.restype = C.c_int
        lib.sp_layer_create.argtypes = [C.POINTER(_Desc), C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_void_p)]
        lib.sp_layer_destroy.restype = C.c_int
        lib.sp_layer_destroy.argtypes = [C.c_void_p]
        lib.sp_set_cc_executor.restype = C.c_int
        lib.sp_set_cc_executor.argtypes = [_CC_FN, C.c_void_p]
        lib.sp_forward_batch.restype = C.c_int
        lib.sp_forward_batch.argtypes = [C.POINTER(_Call), C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                         C.c_void_p, C.c_int, C.c_uint, C.c_void_p]
        _check(lib.sp_init(int(os.environ.get("SLICED_DEVICE", "0")), 0), lib)  # same device: no-op
        _lib = lib  # only once the device is up: a failed init is retried, never skipped
        return lib


_ERRORS = {1: ShapeMismatch, 2: TokenCountOutOfRange, 3: ValueError}


def _check(status: int, lib=None) -> None:
    if status:
        msg = (lib or _lib).sp_last_error()
        raise _ERRORS.get(status, RuntimeError)(msg.decode(errors="replace") if msg else f"status {status}")


def _act_code(activation) -> int:
    return _ACT[getattr(activation, "value", activation)]


def _destroy(handles: list) -> None:
    for h in handles:
        _cc_blocks.pop(h, None)
        if _lib is not None and h:
            _lib.sp_layer_destroy(h)


def _activate(name: str, z: np.ndarray) -> np.ndarray:
    """The reference's activation (slicing_kernel.py:33-38), fp64."""
    if name == "identity":
        return z
    if name == "silu":
        return z / (1.0 + np.exp(-z))
    from scipy.special import erf  # the reference's own erf

    return 0.5 * z * (1.0 + erf(z / math.sqrt(2.0)))


def _reference_cc(_user, layer, x_ptr, ldx, rows, y_ptr, out_dim) -> int:
    try:
        w1_cc, w2_cc, act = _cc_blocks[int(layer)]
        x = np.ctypeslib.as_array(x_ptr, shape=(rows, ldx))[:, : w1_cc.shape[0]].astype(np.float64)
        y = np.ctypeslib.as_array(y_ptr, shape=(rows, out_dim))
        y[:] = _activate(act, x @ w1_cc) @ w2_cc  # slicing_kernel.py:122-123, the CC block
        return 0
    except Exception:
        return 1


def use_reference_cc(on: bool = True) -> None:
    """Run CC blocks through the reference's fp64 numpy expression (True) or
    the library's native CC kernels (False)."""
    global _cc_callback
    lib = _library()
    with _lock:
        if on:
            cb = _CC_FN(_reference_cc)
            _check(lib.sp_set_cc_executor(cb, None))
            _cc_callback = cb  # kept alive while installed
        else:
            _check(lib.sp_set_cc_executor(C.cast(None, _CC_FN), None))
            _cc_callback = None


def place(sliced, activation):
    """Place ``sliced`` for ``activation`` once; later calls return the same
    handle.  The device copy lives until ``sliced`` is garbage collected."""
    lib = _library()
    code = _act_code(activation)
    key = id(sliced)
    with _lock:
        entry = _placed.get(key)
        if entry is not None and entry[0]() is sliced and code in entry[1]:
            return entry[1][code], entry[2]
    w1 = np.concatenate([np.asarray(b, dtype=np.float64) for b in sliced.w1_blocks], axis=1)  # [M, H]
    w2 = np.concatenate([np.asarray(b, dtype=np.float64) for b in sliced.w2_blocks], axis=0)  # [H, N]
    w1t = np.ascontiguousarray(w1.T, dtype=np.float32)  # hidden unit h owns row h
    w2 = np.ascontiguousarray(w2, dtype=np.float32)
    b1, b2 = sliced.boundaries
    desc = _Desc(w1.shape[0], w1.shape[1], w2.shape[1], 0, code, _SP_F32, 0, int(b1), int(b2))
    handle = C.c_void_p()
    _check(lib.sp_layer_create(C.byref(desc), w1t.ctypes.data, None, w2.ctypes.data, C.byref(handle)))
    with _lock:
        entry = _placed.get(key)
        if entry is None or entry[0]() is not sliced:
            handles: dict[int, int] = {}
            ref = weakref.ref(sliced)
            weakref.finalize(sliced, _release_key, key)
            entry = (ref, handles, int(w2.shape[1]))
            _placed[key] = entry
        entry[1][code] = handle.value
        act_name = next(k for k, v in _ACT.items() if v == code)
        _cc_blocks[handle.value] = (np.asarray(sliced.w1_blocks[0], dtype=np.float64),
                                    np.asarray(sliced.w2_blocks[0], dtype=np.float64), act_name)
    return handle.value, entry[2]


def _release_key(key: int) -> None:
    with _lock:
        entry = _placed.pop(key, None)
    if entry is not None:
        _destroy(list(entry[1].values()))


def release(sliced) -> None:
    """Free the device placement of ``sliced`` now (otherwise on GC)."""
    _release_key(id(sliced))


def forward(handle: int, out_dim: int, x: np.ndarray, n_g: int) -> np.ndarray:
    """One sliced forward of a placed layer on host x; returns float64 [T, N]."""
    lib = _library()
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    tokens = x32.shape[0]
    y = np.empty((tokens, out_dim), dtype=np.float32)
    if tokens == 0:
        return y.astype(np.float64)
    call = _Call(handle, tokens, None, None, int(n_g))
    _check(lib.sp_forward_batch(C.byref(call), 1, x32.ctypes.data, _SP_F32, tokens,
                                y.ctypes.data, _SP_F32, _SP_IO_HOST, None))
    return y.astype(np.float64)


def mlp_forward_sliced(x, sliced, activation, n_g: int = 0) -> np.ndarray:
    """Drop-in body of ``slicing_kernel.mlp_forward_sliced`` (``:97-124``):
    the reference's own checks (``:110-118``), then the device forward."""
    x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] != sliced.w1_blocks[0].shape[0]:
        raise ShapeMismatch(
            f"input is {x.shape} but the sliced weights expect "
            f"{sliced.w1_blocks[0].shape[0]} features"
        )
    tokens = x.shape[0]
    if not 0 <= n_g <= tokens:
        raise TokenCountOutOfRange(f"n_g must lie in [0, {tokens}], got {n_g}")
    handle, out_dim = place(sliced, activation)
    return forward(handle, out_dim, x, n_g)


def placed_count() -> int:
    """Layers currently placed by this binding (tests: placement happens once)."""
    with _lock:
        return sum(len(e[1]) for e in _placed.values())
