"""Sliced weight store costs for one Mixtral expert (4096 x 14336 SwiGLU, bf16):
place from row-major weights, save the images, load them back (host image read
straight into pinned memory), re-slice to new rates."""
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200 import store  # noqa: E402
from paper_2411_15715_b200.schedule import SlicingRates  # noqa: E402
from paper_2411_15715_b200.sliced import SlicedFFN  # noqa: E402

nat.init(0)
M, H = 4096, 14336
g = torch.Generator().manual_seed(0)
w1t, w3t, w2t = ((torch.randn(*s, generator=g) / 64).to(torch.bfloat16) for s in ((H, M), (H, M), (M, H)))
nbytes = 3 * M * H * 2
t = time.perf_counter()
ffn = SlicedFFN(w1t, w2t, SlicingRates(0.35, 0.15, 0.5), w3t=w3t, dtype="bf16")
print(f"place from weights: {(time.perf_counter() - t) * 1e3:7.1f} ms  ({nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s)")
d = tempfile.mkdtemp(dir=os.environ.get("STORE_DIR", "/tmp"))
p = Path(d) / "expert.spstore"
t = time.perf_counter()
store.save_store(p, {"e0": ffn.layer})
dt = time.perf_counter() - t
print(f"save images:        {dt * 1e3:7.1f} ms  ({p.stat().st_size / dt / 1e9:.1f} GB/s, {p.stat().st_size / 1e6:.0f} MB file)")
for rep in range(3):
    t = time.perf_counter()
    lay = store.load_store(p)["e0"]
    dt = time.perf_counter() - t
    print(f"load images:        {dt * 1e3:7.1f} ms  ({p.stat().st_size / dt / 1e9:.1f} GB/s, page cache warm)")
    lay.release()
for r in (SlicingRates(0.3, 0.2, 0.5), SlicingRates(0.0, 0.0, 1.0), SlicingRates(0.5, 0.5, 0.0)):
    t = time.perf_counter()
    moved = ffn.reslice(r)
    dt = time.perf_counter() - t
    print(f"reslice -> {r.cc:.2f}/{r.cg:.2f}/{r.gg:.2f}: {dt * 1e3:7.1f} ms  ({nbytes / dt / 1e9:.1f} GB/s)")
    moved.layer.release()
os.remove(p)
