"""Pinned host -> HBM copy rate: one stream of back-to-back chunks vs two
alternating streams vs one large copy (decides the CG streamer's copy layout)."""
import sys
import torch

tot = 160 << 20
host = torch.empty(tot, dtype=torch.uint8).pin_memory()
dev = torch.empty(tot, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(chunk, nstreams, reps=5):
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for s in streams[:nstreams]:
            s.wait_event(a)
        evs = []
        for i, off in enumerate(range(0, tot, chunk)):
            s = streams[i % nstreams]
            with torch.cuda.stream(s):
                dev[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
        for s in streams[:nstreams]:
            e = torch.cuda.Event()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        b.record()
        torch.cuda.synchronize()
        best = max(best, tot / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


for chunk_mb in (2, 4, 8, 16, 32, 160):
    for ns in (1, 2, 3):
        if chunk_mb == 160 and ns > 1:
            continue
        print(f"chunk {chunk_mb:4d} MB  streams {ns}: {run(chunk_mb << 20, ns):6.2f} GB/s", flush=True)
