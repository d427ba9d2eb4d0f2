"""Is the grouped GG launch's tail systematic per SM?  Two GG-only Mixtral
experts (2 x 7168 rows) in one launch, SP_KSTAMPS=1: per launch, each CTA's end
time relative to the launch's median end, keyed by %smid; the per-SM means of
two independent halves of the launches are correlated (systematic if high)."""
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
M, H = 4096, 7168
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lays = [NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16") for _ in range(2)]
scratch = torch.zeros(64 << 20, device="cuda")
x = torch.randn(1, M, device="cuda").to(torch.bfloat16)
G = torch.cuda.get_device_properties(0).multi_processor_count
rel = {h: [] for h in (0, 1)}
relb = {h: [] for h in (0, 1)}
maps = []
spans, meds = [], []
N = int(os.environ.get("REPS", "60"))
for r in range(N + 3):
    scratch.sum()
    torch.cuda.synchronize()
    forward_calls([CallSpec(l) for l in lays], x)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (4096 * 8))()
    nat.check(lib.sp_debug_stamps(buf, 4096 * 8))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8)[:G].astype(np.int64)
    if r < 3:
        continue
    end = (a[:, 6] - a[:, 0].min()) / 1e3
    med = np.median(end)
    spans.append(end.max())
    meds.append(med)
    v = np.full(G, np.nan)
    v[a[:, 7]] = end - med
    rel[r % 2].append(v)
    relb[r % 2].append(end - med)
    maps.append(a[:, 7].copy())
h0, h1 = np.nanmean(rel[0], axis=0), np.nanmean(rel[1], axis=0)
ok = ~np.isnan(h0) & ~np.isnan(h1)
print(f"launch span median {np.median(spans):.1f} us, CTA end median {np.median(meds):.1f} us")
print(f"per-SM end - median: std {np.nanstd(np.concatenate(rel[0] + rel[1])):.2f} us per launch, "
      f"std of per-SM means {np.nanstd((h0 + h1) / 2):.2f} us")
print(f"split-half correlation of per-SM lateness: {np.corrcoef(h0[ok], h1[ok])[0, 1]:.3f}")
b0, b1 = np.mean(relb[0], axis=0), np.mean(relb[1], axis=0)
print(f"split-half correlation of per-blockIdx lateness: {np.corrcoef(b0, b1)[0, 1]:.3f}")
m = np.array(maps)
print(f"blockIdx -> SM mapping identical across launches: {bool((m == m[0]).all())} "
      f"({(m == m[0]).all(axis=1).mean():.2f} of launches match the first); first 16: {m[0][:16].tolist()}")
late = np.argsort((h0 + h1) / 2)[-10:]
print("latest SMs (mean lateness us):", ", ".join(f"{s}:{(h0[s] + h1[s]) / 2:.1f}" for s in late))
early = np.argsort((h0 + h1) / 2)[:10]
print("earliest SMs:", ", ".join(f"{s}:{(h0[s] + h1[s]) / 2:.1f}" for s in early))
