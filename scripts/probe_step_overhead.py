"""Decode-step host overhead: time inside the native MoE call vs outside it."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.expert_parallel import ExpertParallelMoE  # noqa: E402

sys.argv = ["bench.py"]
args = bench.parse()
nat.init(0)
rates, _, _, _ = bench.plan_rates(args, 1)
experts = bench.make_experts(args, rates, range(8), torch.device("cuda", 0))
rng = np.random.default_rng(7)
moe = ExpertParallelMoE(experts, rng.standard_normal((4096, 8)), 2, 8, out_dim=4096)
xs = [torch.from_numpy(rng.standard_normal((1, 4096)).astype(np.float32)).cuda().to(torch.bfloat16) for _ in range(64)]
for i in range(10):
    moe(xs[i % 64])
torch.cuda.synchronize()
d = moe._dispatch
inside, outside = [], []
t_prev = time.perf_counter()
for i in range(200):
    t0 = time.perf_counter()
    y = d(xs[i % 64])
    t1 = time.perf_counter()
    inside.append(t1 - t0)
    outside.append(t0 - t_prev)
    t_prev = t1
torch.cuda.synchronize()
print(f"dispatch call: median {1e6 * np.median(inside):.1f} us; between calls: median {1e6 * np.median(outside[1:]):.1f} us")
for traced in (False, True):
    nat.trace_enable(traced)
    inside, outside = [], []
    t_prev = time.perf_counter()
    for i in range(200):
        t0 = time.perf_counter()
        y = d(xs[i % 64])
        t1 = time.perf_counter()
        inside.append(t1 - t0)
        outside.append(t0 - t_prev)
        t_prev = t1
    torch.cuda.synchronize()
    if traced:
        spans = nat.trace_fetch()
        rets = sorted((s["call"], s["end_s"]) for s in spans if s["kind"] == "return")
        routes = {s["call"]: s["start_s"] for s in spans if s["kind"] == "route" and s["bytes"] > 0}
        gaps = [routes[c + 1] - e for c, e in rets if c + 1 in routes]
        print(f"trace gap return->route: median {1e6 * np.median(gaps):.1f} us")
    nat.trace_enable(False)
    print(f"traced={traced}: call median {1e6 * np.median(inside):.1f} us; between calls median {1e6 * np.median(outside[1:]):.1f} us")
inside2 = []
t_prev = time.perf_counter()
for i in range(200):
    t0 = time.perf_counter()
    y = moe(xs[i % 64])
    inside2.append(time.perf_counter() - t0)
print(f"ExpertParallelMoE call: median {1e6 * np.median(inside2):.1f} us")
