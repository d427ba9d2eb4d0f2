"""GG-block GEMV micro-benchmark: achieved HBM GB/s of the up+down kernel pair.

Usage: python scripts/bench_gemv.py [--T 1] [--hidden 7168 14336] [--reps 10]
Tunables come from the environment (SP_WPR, SP_CTAS_PER_SM) so a shell loop
can sweep them in separate processes.  L2 is flushed before every rep.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, nargs="+", default=[1])
    ap.add_argument("--hidden", type=int, nargs="+", default=[7168, 14336])
    ap.add_argument("--model", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--gated", type=int, default=1)
    args = ap.parse_args()
    nat.init(0)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650
    scratch = torch.zeros(64 << 20, device="cuda")
    tag = f"WPR={os.environ.get('SP_WPR', 'auto')} CTAS={os.environ.get('SP_CTAS_PER_SM', '2')}"
    for h in args.hidden:
        g = torch.Generator(device="cuda").manual_seed(h)
        tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
        mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(tdt).cpu()  # noqa: E731
        w1t, w3t, w2t = mk(h, args.model), mk(h, args.model), mk(args.model, h)
        lay = NativeLayer(w1t, w2t.t().contiguous(), 0, 0, "silu", w3t if args.gated else None, dtype=args.dtype)
        nbytes = lay.placed_bytes()["gg"]
        for T in args.T:
            x = torch.randn(T, args.model, device="cuda").to(tdt)
            times = []
            for r in range(args.reps + 2):
                scratch.add_(1.0)
                torch.cuda.synchronize()
                nat.trace_enable(True)
                forward_calls([CallSpec(lay)], x)
                sp = [s for s in nat.trace_fetch() if s["kind"] == "gg"]
                nat.trace_enable(False)
                if r >= 2:
                    times.append(sp[0]["end_s"] - sp[0]["start_s"])
            t = float(np.median(times))
            print(f"{tag} H={h} T={T} bytes={nbytes/1e6:.1f}MB  median {t*1e6:.1f} us  "
                  f"{nbytes/t/1e9:.0f} GB/s  frac={nbytes/t/1e9/peak:.3f}  best {nbytes/min(times)/1e9:.0f} GB/s",
                  flush=True)
        lay.release()


if __name__ == "__main__":
    main()
