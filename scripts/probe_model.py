"""Where does a whole-model decode step go?  Trace the sliced MoE spans of one
32-layer step and time the attention part alone."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral  # noqa: E402

sys.argv = ["bench.py"]
args = bench.parse()
nat.init(0)
rates, _, _, _ = bench.plan_rates(args, 1)
cfg = DecoderConfig(layers=8, distinct=2, max_seq=600)
m = SlicedMixtral(cfg, rates)
x = (torch.randn(1, 4096, device="cuda") * 0.5).to(torch.bfloat16)
for p in range(3):
    x = m.decode_step(x, 512 + p)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    x = m.decode_step(x, 520 + rep)
    torch.cuda.synchronize()
    print(f"step wall {1e3 * (time.perf_counter() - t0):.1f} ms for {cfg.layers} layers", flush=True)
# attention only
torch.cuda.synchronize()
t0 = time.perf_counter()
for l in range(cfg.layers):
    x = x + m._attention(l, m._rms(x, m.attn[l]["n1"]), 530)
torch.cuda.synchronize()
print(f"attention only: {1e3 * (time.perf_counter() - t0) / cfg.layers:.3f} ms/layer", flush=True)
# MoE only
torch.cuda.synchronize()
t0 = time.perf_counter()
for l in range(cfg.layers):
    x = x + m._moe(l % cfg.distinct, m._rms(x, m.attn[l]["n2"]))
torch.cuda.synchronize()
print(f"moe only: {1e3 * (time.perf_counter() - t0) / cfg.layers:.3f} ms/layer", flush=True)
nat.trace_enable(True)
x = m.decode_step(x, 540)
torch.cuda.synchronize()
spans = nat.trace_fetch()
nat.trace_enable(False)
Path("gpurun_out/timeline_model.json").write_text(json.dumps(spans))
m.release()
