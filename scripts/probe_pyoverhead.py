"""Per-call Python-side costs around the native MoE call (decode step overhead)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

x = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)


def bench(name, fn, n=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:40s} {1e6 * (time.perf_counter() - t) / n:7.2f} us", flush=True)


bench("torch.empty((1,4096), bf16, cuda)", lambda: torch.empty((1, 4096), dtype=torch.bfloat16, device=x.device))
bench("torch.cuda.current_stream(dev)", lambda: torch.cuda.current_stream(x.device))
bench("current_stream().cuda_stream", lambda: torch.cuda.current_stream(x.device).cuda_stream)
bench("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
bench("x.is_cuda/is_contiguous/dtype", lambda: (x.is_cuda, x.is_contiguous(), x.dtype == torch.bfloat16))
bench("x.data_ptr()", lambda: x.data_ptr())
bench("C.c_void_p(123)", lambda: C.c_void_p(123))
lib = C.CDLL(None)
bench("ctypes call (getpid)", lambda: lib.getpid())
bench("time.perf_counter", time.perf_counter)
