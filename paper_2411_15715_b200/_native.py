"""ctypes binding of libsliced.so (include/sliced.h).

ctypes.CDLL drops the GIL for the duration of every foreign call, so the CC
block's host threads and a Python caller's other threads keep running while a
forward is in flight.  There is no Python fallback: if the library is missing
or no sm_100 device is visible, the GPU entry points raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import NativeError, raise_for

LIB_PATH = Path(__file__).resolve().parent / "_native" / "libsliced.so"

SP_F32, SP_BF16 = 0, 1
SP_IO_DEVICE, SP_IO_HOST, SP_NO_CC_THREADS, SP_X_TO_BF16 = 0, 1, 2, 4
ACT_CODES = {"identity": 0, "silu": 1, "gelu": 2}
TRACE_KINDS = ("launch", "gg", "cg", "cg_prime", "copy", "cc", "merge", "route", "return", "ycc")
STREAM_NAMES = ("launch", "transfer", "gpu", "cpu")

# symbol -> (restype, argtypes); the CPU suite checks this table against include/sliced.h
_c_layer = C.c_void_p


class LayerDesc(C.Structure):
    _fields_ = [
        ("model_dim", C.c_int64),
        ("hidden_dim", C.c_int64),
        ("out_dim", C.c_int64),
        ("gated", C.c_int32),
        ("act", C.c_int32),
        ("wdtype", C.c_int32),
        ("chunk_rows", C.c_int32),
        ("b1", C.c_int64),
        ("b2", C.c_int64),
    ]


class Call(C.Structure):
    _fields_ = [
        ("layer", _c_layer),
        ("tokens", C.c_int64),
        ("token_ids", C.POINTER(C.c_int32)),
        ("gates", C.POINTER(C.c_float)),
        ("n_g", C.c_int64),
    ]


class TraceRecord(C.Structure):
    _fields_ = [
        ("index", C.c_int32),
        ("stream", C.c_int32),
        ("kind", C.c_int32),
        ("call", C.c_int32),
        ("start_s", C.c_double),
        ("end_s", C.c_double),
        ("bytes", C.c_double),
        ("dev_s", C.c_double),
    ]


# sp_cc_fn (include/sliced.h): user, layer, x [rows, ldx] f32, ldx, rows, y_cc [rows, out_dim] f32, out_dim
CC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_float), C.c_int64, C.c_int64,
                    C.POINTER(C.c_float), C.c_int64)

SIGNATURES = {
    "sp_set_cc_executor": (C.c_int, [CC_FN, C.c_void_p]),
    "sp_abi_version": (C.c_int, []),
    "sp_layer_image_sizes": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                       C.POINTER(C.c_int32)]),
    "sp_layer_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "sp_layer_create_from_images": (C.c_int, [C.POINTER(LayerDesc), C.c_void_p, C.c_size_t, C.c_void_p,
                                              C.c_size_t, C.POINTER(C.c_void_p)]),
    "sp_layer_load_file": (C.c_int, [C.POINTER(LayerDesc), C.c_char_p, C.c_uint64, C.c_size_t, C.c_uint64,
                                     C.c_size_t, C.POINTER(C.c_void_p)]),
    "sp_layer_reslice": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
    "sp_last_error": (C.c_char_p, []),
    "sp_init": (C.c_int, [C.c_int, C.c_int]),
    "sp_shutdown": (C.c_int, []),
    "sp_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sp_layer_create": (C.c_int, [C.POINTER(LayerDesc), C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(_c_layer)]),
    "sp_layer_destroy": (C.c_int, [_c_layer]),
    "sp_layer_bytes": (C.c_int, [_c_layer, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_size_t)]),
    "sp_layer_widths": (C.c_int, [_c_layer, C.POINTER(C.c_int64)]),
    "sp_forward_batch": (C.c_int, [C.POINTER(Call), C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                   C.c_void_p, C.c_int, C.c_uint, C.c_void_p]),
    "sp_cc_forward_host": (C.c_int, [_c_layer, C.c_void_p, C.c_int, C.c_int64,
                                     C.POINTER(C.c_float), C.c_int]),
    "sp_moe_route": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_int,
                               C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    "sp_moe_forward": (C.c_int, [C.POINTER(_c_layer), C.c_int, C.POINTER(C.c_float), C.c_int, C.c_void_p,
                                 C.c_int, C.c_int64, C.c_void_p, C.c_int, C.c_uint, C.c_void_p]),
    "sp_trace_enable": (C.c_int, [C.c_int]),
    "sp_trace_fetch": (C.c_int, [C.POINTER(TraceRecord), C.POINTER(C.c_int)]),
    "sp_stats": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "sp_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "sp_host_free": (C.c_int, [C.c_void_p]),
    "sp_round_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
}

_lib = None
_lock = threading.Lock()
_device: int | None = None


def lib():
    """Load libsliced.so once; raise if it was never built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2411_15715_b200._build` "
                    "(the sliced path has no CPU fallback)"
                )
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
        return _lib


def available() -> bool:
    """True when libsliced.so is built (host-side helpers need no device)."""
    return _lib is not None or LIB_PATH.exists()


def check(status: int) -> None:
    if status != 0:
        msg = lib().sp_last_error()
        raise_for(status, msg.decode(errors="replace") if msg else "")


def init(device: int | None = None, host_threads: int = 0) -> int:
    """Bind the library to a CUDA device (default: torch's current device, else 0).

    ``device=-1`` opens a host-only context (CC kernels only)."""
    global _device
    if device is None:
        device = _device if _device is not None else _default_device()
    if _device is not None and _device == device:
        return device
    threads = host_threads or int(os.environ.get("SP_HOST_THREADS", "0"))
    check(lib().sp_init(int(device), int(threads)))
    _device = device
    return device


def shutdown() -> None:
    global _device
    if _lib is not None:
        check(_lib.sp_shutdown())
    _device = None


def current_device() -> int | None:
    return _device


def _default_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0


def trace_enable(on: bool = True, gg_only: bool = False) -> None:
    """``gg_only``: device spans only around GG launches (plus host spans), so
    the traced region keeps the timing of an untraced one."""
    check(lib().sp_trace_enable((2 if gg_only else 1) if on else 0))


def trace_fetch() -> list[dict]:
    """Measured spans since trace_enable, in the reference Gantt schema
    (pipeline.py:347-364) plus ``kind`` / ``call`` / ``bytes``."""
    n = C.c_int(0)
    check(lib().sp_trace_fetch(None, C.byref(n)))
    buf = (TraceRecord * max(1, n.value))()
    check(lib().sp_trace_fetch(buf, C.byref(n)))
    return [
        {"gemm_index": r.index, "stream": STREAM_NAMES[r.stream], "start_s": r.start_s,
         "end_s": r.end_s, "kind": TRACE_KINDS[r.kind], "call": r.call, "bytes": r.bytes,
         "dev_s": r.dev_s}
        for r in buf[: n.value]
    ]


def stats() -> dict:
    launches, h2d = C.c_uint64(), C.c_uint64()
    check(lib().sp_stats(C.byref(launches), C.byref(h2d)))
    return {"kernel_launches": launches.value, "h2d_bytes": h2d.value}


_cc_keepalive = None  # the installed CFUNCTYPE object must outlive every forward that may call it


def set_cc_executor(fn) -> None:
    """Run every CC block through ``fn(layer_handle, x, y_cc) -> None`` (numpy
    views: x [rows, M'] f32 with M' >= model_dim, y_cc [rows, out_dim] f32 to
    overwrite) on the library's CC coordinator thread, concurrently with the
    forward's GPU work; ``None`` restores the native CC kernels."""
    global _cc_keepalive
    import numpy as np

    if fn is None:
        check(lib().sp_set_cc_executor(C.cast(None, CC_FN), None))
        _cc_keepalive = None
        return

    def trampoline(_user, layer, x, ldx, rows, y, out_dim):
        try:
            xa = np.ctypeslib.as_array(x, shape=(rows, ldx))
            ya = np.ctypeslib.as_array(y, shape=(rows, out_dim))
            fn(int(layer or 0), xa, ya)
            return 0
        except Exception:  # reported as SP_ERR_VALUE by the forward
            import traceback

            traceback.print_exc()
            return 1

    cb = CC_FN(trampoline)
    check(lib().sp_set_cc_executor(cb, None))
    _cc_keepalive = cb
