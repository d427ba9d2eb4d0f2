"""Why is the grouped GG launch slower inside the decode step than alone?
Two GG-only experts (4096 x 7168 rows each, bf16 SwiGLU) in one forward,
CUDA-event span of the grouped launch: alone, with background H2D copies,
with a background host CC block, with both; L2 flushed between reps."""
import ctypes as C
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.b200_profile import BackgroundCC, BackgroundCopy  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402

nat.init(0)
M, H = 4096, 7168
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lays = [NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16") for _ in range(2)]
scratch = torch.zeros(64 << 20, device="cuda")
x = torch.randn(1, M, device="cuda").to(torch.bfloat16)
nbytes = sum(l.placed_bytes()["gg"] for l in lays)


lib = nat.lib()
lib.sp_debug_stamps.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
STAMPS = os.environ.get("SP_KSTAMPS") == "1"


def kernel_span():
    """device-side duration of the last ffn_block launch: first CTA start to last CTA end"""
    buf = (C.c_ulonglong * (4096 * 8))()
    nat.check(lib.sp_debug_stamps(buf, 4096 * 8))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8)
    a = a[a[:, 0] > 0]
    return (a[:, 6].max() - a[:, 0].min()) * 1e-9


def sample(reps=20):
    ts, ks = [], []
    for r in range(reps):
        scratch.add_(1.0)
        torch.cuda.synchronize()
        nat.trace_enable(True)
        forward_calls([CallSpec(l) for l in lays], x)
        torch.cuda.synchronize()
        sp = [s for s in nat.trace_fetch() if s["kind"] == "gg"]
        nat.trace_enable(False)
        if r >= 3:
            ts.append(sp[0]["end_s"] - sp[0]["start_s"])
            if STAMPS:
                ks.append(kernel_span())
    t = float(np.median(ts))
    if ks:
        print(f"    (in-kernel span {np.median(ks) * 1e6:.1f} us)", flush=True)
    return t, nbytes / t / 1e9


def busy_gpu():
    """a long-running kernel queue on another stream ahead of the launch"""
    return None


t, bw = sample()
print(f"alone:            {t*1e6:7.1f} us  {bw:7.0f} GB/s", flush=True)
for mb in (8, 512):
    with BackgroundCopy(torch, nbytes=mb << 20):
        t, bw = sample()
        print(f"+ H2D copies into {mb} MB: {t*1e6:7.1f} us  {bw:7.0f} GB/s", flush=True)
with BackgroundCopy(torch):
    t, bw = sample()
    print(f"+ H2D copies:     {t*1e6:7.1f} us  {bw:7.0f} GB/s", flush=True)
with BackgroundCC():
    t, bw = sample()
    print(f"+ host CC:        {t*1e6:7.1f} us  {bw:7.0f} GB/s", flush=True)
with BackgroundCopy(torch), BackgroundCC():
    t, bw = sample()
    print(f"+ both:           {t*1e6:7.1f} us  {bw:7.0f} GB/s", flush=True)
