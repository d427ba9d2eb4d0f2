"""Prefill GG-block throughput through the tcgen05 path: one Mixtral expert
(4096 x 14336 SwiGLU, bf16) fully in HBM, T tokens; TFLOP/s and weight GB/s."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402

nat.init(0)
root = Path(__file__).resolve().parents[1]
peaks = json.loads((root / "MEASURED_PEAKS.json").read_text()) if (root / "MEASURED_PEAKS.json").exists() else {}
M = 4096
H = int(sys.argv[1]) if len(sys.argv) > 1 else 14336
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lay = NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16")
nbytes = lay.placed_bytes()["gg"]
scratch = torch.zeros(64 << 20, device="cuda")
import os
for T in [int(t) for t in os.environ.get("SP_PREFILL_T", "16 64 128 256 512").split()]:
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    ts, ds = [], []
    for r in range(6):
        scratch.sum()  # L2 flush by reading: a write would leave dirty lines whose write-back competes
        torch.cuda.synchronize()
        nat.trace_enable(True)
        forward_calls([CallSpec(lay)], x)
        sp = [s for s in nat.trace_fetch() if s["kind"] == "gg"]
        nat.trace_enable(False)
        if r >= 2:
            ts.append(sp[0]["end_s"] - sp[0]["start_s"])
            ds.append(sp[0].get("dev_s", 0.0))
    t = float(np.median(ts))
    d = float(np.median(ds))
    flops = 2.0 * T * 3 * M * H
    print(f"H={H} T={T}: {t*1e6:8.1f} us  {flops/t/1e12:7.1f} TFLOP/s ({flops/t/1e12/peaks.get('bf16_tflops', 1669):.3f} of bf16 peak)"
          f"  weights {nbytes/t/1e9:7.0f} GB/s ({nbytes/t/1e9/peaks.get('hbm_gbs', 6550):.3f} of HBM)"
          + (f"  | device span {d*1e6:6.1f} us ({nbytes/d/1e9/peaks.get('hbm_gbs', 6550):.3f} of HBM)" if d > 0 else ""),
          flush=True)
