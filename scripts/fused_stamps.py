"""Phase anatomy of expert_tc_kernel on one resident Mixtral expert (SP_KSTAMPS=1):
per-CTA %globaltimer stamps, percentiles over CTAs relative to the earliest start.
  0 producer start   1 last up unit issued   2 first down unit issued (its `a` ready)
  3 last up MMA commit   4 up owner published ready   5 last down MMA commit
  6 down partials stored   7 epilogue end   8 first down partial stored
  9 first fix-up's waits done   10 first fix-up done   11 epilogue reaches the
  first down segment   12 its accumulator is complete"""
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
M, H = 4096, int(os.environ.get("SP_H", 14336))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lay = NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16")
scratch = torch.zeros(64 << 20, device="cuda")
G = torch.cuda.get_device_properties(0).multi_processor_count
names = ["start", "lastU_issued", "firstD_issued", "lastU_mma", "U_ready", "lastD_mma", "D_part", "end",
         "D1_part", "fix1_waited", "fix1_done", "epi_U_done", "D1_tfull"]
for T in [int(t) for t in os.environ.get("SP_PREFILL_T", "16 64 128").split()]:
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    rows = []
    for r in range(5):
        scratch.sum()
        torch.cuda.synchronize()
        forward_calls([CallSpec(lay)], x)
        buf = (C.c_ulonglong * (4096 * 8))()
        nat.check(lib.sp_debug_stamps(buf, 4096 * 8))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 16)[:G].astype(np.int64)
        if r >= 2:
            rows.append(a)
    a = rows[-1]
    nz = np.nonzero(a[:, 0])[0]
    if nz.size != G:
        print(f"  warning: {nz.size} of {G} CTAs stamped; first unstamped {np.setdiff1d(np.arange(G), nz)[:8]}")
    a = a[nz]
    t0 = a[:, 0].min()
    print(f"T={T}: kernel span {(a[:, 7].max() - t0) / 1e3:.1f} us")
    for k, nm in enumerate(names):
        v = a[:, k]
        v = v[v > 0]
        if v.size == 0:
            continue
        d = (v - t0) / 1e3
        print(f"  {k:2d} {nm:14s} min {d.min():7.1f}  p10 {np.percentile(d, 10):7.1f}  med {np.median(d):7.1f}"
              f"  p90 {np.percentile(d, 90):7.1f}  max {d.max():7.1f} us  (n={v.size})")
    late = np.argsort(a[:, 7])[-6:]
    print("  (cta ids below index the stamped rows)")
    print("  latest CTAs (stamps - t0, us):")
    for c in late:
        print(f"   cta {c:3d}: " + " ".join(f"{(v - t0) / 1e3:6.1f}" if v > 0 else "   -  " for v in a[c, :13]))
