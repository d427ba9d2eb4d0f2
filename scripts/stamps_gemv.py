"""Per-CTA phase timing of the fused block kernel (SP_KSTAMPS=1): where does a
GG launch spend its time?  Stamps: 0 entry, 1 barriers ready, 2 x staged,
3 phase-1 done, 4 a ready, 5 phase-2 done, 6 slice written."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["SP_KSTAMPS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402

nat.init(0)
lib = nat.lib()
lib.sp_debug_stamps.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
scratch = torch.zeros(64 << 20, device="cuda")
for h in [int(a) for a in sys.argv[1:]] or [1024, 7168]:
    g = torch.Generator(device="cuda").manual_seed(h)
    mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
    lay = NativeLayer(mk(h, 4096), mk(h, 4096), 0, 0, "silu", mk(h, 4096), dtype="bf16")
    x = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
    for r in range(4):
        scratch.add_(1.0)
        torch.cuda.synchronize()
        forward_calls([CallSpec(lay)], x)
        torch.cuda.synchronize()
    buf = (C.c_ulonglong * (148 * 8))()
    nat.check(lib.sp_debug_stamps(buf, 148 * 8))
    st = np.array(buf, dtype=np.float64).reshape(148, 8)[:, :7]
    t0 = st[:, 0].min()
    rel = (st - t0) / 1e3
    names = ["entry", "bars", "x", "phase1", "a", "phase2", "end"]
    print(f"H={h}: kernel span {rel[:, 6].max():.1f} us (first entry -> last end)")
    for i, n in enumerate(names):
        print(f"   {n:7s} min {rel[:, i].min():7.2f}  median {np.median(rel[:, i]):7.2f}  max {rel[:, i].max():7.2f} us")
    lay.release()
