"""The AMX CC kernel's index arithmetic on a host without AMX: host_cc_amx.cpp
built with SP_AMX_EMULATE (software 16 x 64-byte tiles, same loops) against a
numpy restatement of the same math (bf16 x / weights / hidden activation, fp32
sums).  The real tiles are checked on the GPU box
(test_abi.py::test_amx_cc_kernel_on_the_gpu_box)."""

from __future__ import annotations

import ctypes as C
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from oracle import sliced_forward as orc

CSRC = ROOT / "paper_2411_15715_b200" / "csrc"


def _avx512() -> bool:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512vl"))


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    if not _avx512() or shutil.which("g++") is None:
        pytest.skip("needs g++ and an AVX-512 host")
    out = tmp_path_factory.mktemp("amx") / "libamx_emu.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-DSP_AMX_EMULATE", f"-I{CSRC}",
                    str(CSRC / "host_cc_amx.cpp"), str(CSRC / "host_cc.cpp"), str(ROOT / "tests" / "amx_emu" / "driver.cpp"),
                    "-o", str(out)], check=True, capture_output=True)
    lib = C.CDLL(str(out))
    lib.amx_emu_run.restype = C.c_int
    lib.amx_emu_run.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int]
    return lib


def _bits(a: np.ndarray) -> np.ndarray:
    return (orc.bf16_round(a).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _reference(x, w1t, w3t, w2, act, gated):
    """bf16 x and weights, fp32 sums, the hidden activation rounded to bf16 (as the tiles see it)."""
    xb = orc.bf16_round(x).astype(np.float64)
    z1 = xb @ orc.bf16_round(w1t).astype(np.float64).T
    a = orc.activate(act, z1)
    if gated:
        a = a * (xb @ orc.bf16_round(w3t).astype(np.float64).T)
    a = orc.bf16_round(a.astype(np.float32)).astype(np.float64)
    return a @ orc.bf16_round(w2).astype(np.float64)


@pytest.mark.parametrize("T,M,N,b1,chunk,gated,act,threads", [
    (4, 96, 80, 70, 64, 1, "silu", 3),        # partial token group, ragged b1 / N
    (16, 256, 128, 256, 64, 1, "silu", 4),
    (37, 200, 272, 301, 128, 1, "gelu", 5),   # ragged everything, several chunks
    (48, 128, 64, 33, 64, 0, "identity", 2),  # plain MLP, b1 just past a tile
    (128, 512, 544, 500, 192, 1, "silu", 8),  # a down round of 128 columns and a partial one
    (20, 1100, 96, 1100, 256, 1, "silu", 3),  # K and the hidden range over several 1024-wide chunks
])
@pytest.mark.parametrize("prepack", [0, 1])
def test_amx_kernel_emulated_matches_restatement(emu, T, M, N, b1, chunk, gated, act, threads, prepack):
    rng = np.random.default_rng(T * 7 + M)
    x = rng.uniform(-1, 1, (T, M)).astype(np.float32)
    w1t = (rng.standard_normal((b1, M)) / np.sqrt(M)).astype(np.float32)
    w3t = (rng.standard_normal((b1, M)) / np.sqrt(M)).astype(np.float32)
    w2 = (rng.standard_normal((b1, N)) / np.sqrt(b1)).astype(np.float32)
    y = np.full((T, N), np.nan, dtype=np.float32)
    acts = {"identity": 0, "silu": 1, "gelu": 2}
    b_w1, b_w3, b_w2 = (np.ascontiguousarray(_bits(a)) for a in (w1t, w3t, w2))
    st = emu.amx_emu_run(gated, acts[act], M, N, b1, chunk, b_w1.ctypes.data, b_w3.ctypes.data, b_w2.ctypes.data,
                         x.ctypes.data, T, y.ctypes.data, threads, prepack)
    assert st == 0 and np.isfinite(y).all()
    ref = _reference(x, w1t, w3t, w2, act, gated)
    assert orc.max_rel_error(y, ref) <= 2e-3, orc.max_rel_error(y, ref)


def test_amx_kernel_emulated_is_thread_count_invariant(emu):
    """Columns are split over threads, each output summed in one hidden order:
    bit-identical for any thread count, with or without the prepacked W2."""
    rng = np.random.default_rng(11)
    T, M, N, b1 = 33, 160, 200, 150
    x = rng.uniform(-1, 1, (T, M)).astype(np.float32)
    ws = [np.ascontiguousarray(_bits((rng.standard_normal(s) / 8).astype(np.float32))) for s in ((b1, M), (b1, M), (b1, N))]
    outs = []
    for th in (1, 3, 7):
        for pre in (0, 1):
            y = np.zeros((T, N), dtype=np.float32)
            emu.amx_emu_run(1, 1, M, N, b1, 64, ws[0].ctypes.data, ws[1].ctypes.data, ws[2].ctypes.data,
                            x.ctypes.data, T, y.ctypes.data, th, pre)
            outs.append(y)
    # and the prepacked W2 copy feeds the same tiles as the per-round repack
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
