"""Host CC-block micro-benchmark: effective weight GB/s of the AVX-512 CC kernel
vs threads, next to a numpy read-bandwidth probe of the same host."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import NativeLayer  # noqa: E402


def main():
    dev = -1 if "--host-only" in sys.argv else 0
    nat.init(dev)
    rng = np.random.default_rng(0)
    M = N = 4096
    big = np.ones(1 << 28, dtype=np.float32)  # 1 GiB
    for _ in range(2):
        big.sum()
    t = time.perf_counter()
    for _ in range(3):
        big.sum()
    print(f"numpy sum read: {3 * big.nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s (1 thread)")
    flush = np.zeros(64 << 20)
    quick = "--quick" in sys.argv
    for H in ((6144,) if quick else (2048, 6144)):
        w1t = rng.standard_normal((H, M), dtype=np.float32)
        w2 = rng.standard_normal((H, N), dtype=np.float32)
        lay = NativeLayer(w1t, w2, H, H, "silu", w1t, dtype="bf16")
        nbytes = lay.placed_bytes()["cc"]
        x = rng.standard_normal((1, M))
        for th in ([8, os.cpu_count()] if quick else [1, 4, 8, 12, 15, 16, os.cpu_count()]):
            ts = []
            for r in range(6):
                flush += 1
                t0 = time.perf_counter()
                lay.cc_forward_host(x, threads=th)
                ts.append(time.perf_counter() - t0)
            dt = float(np.median(ts[1:]))
            print(f"CC H={H} bytes={nbytes/1e6:.0f}MB threads={th}: {dt*1e3:.2f} ms  {nbytes/dt/1e9:.1f} GB/s", flush=True)
        lay.release()


if __name__ == "__main__":
    main()
