"""Attention part of the decoder alone: wall vs CUDA time, kernel list (torch profiler)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15715_b200.model import DecoderConfig, SlicedMixtral  # noqa: E402
from paper_2411_15715_b200.schedule import SlicingRates  # noqa: E402

cfg = DecoderConfig(layers=8, distinct=1, experts=1, hidden_dim=256, max_seq=600)
m = SlicedMixtral(cfg, SlicingRates(0.0, 0.0, 1.0), experts_factory=lambda d: [])
x = (torch.randn(1, 4096, device="cuda") * 0.5).to(torch.bfloat16)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for l in range(cfg.layers):
        x = x + m._attention(l, m._rms(x, m.attn[l]["n1"]), 530)
    torch.cuda.synchronize()
    print(f"attention only: {1e3 * (time.perf_counter() - t0) / cfg.layers:.3f} ms/layer", flush=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for l in range(cfg.layers):
        x = x + m._attention(l, m._rms(x, m.attn[l]["n1"]), 530)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
