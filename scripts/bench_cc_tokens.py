"""CC host kernel vs token count (AMX tile path vs AVX-512 with SP_AMX=0): ms, weight GB/s, TFLOP/s.
Env: TH threads, HH hidden rows, TS token counts."""
import numpy as np, sys, time, os  # noqa: E401
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15715_b200 import _native as nat
from paper_2411_15715_b200.sliced import NativeLayer
nat.init(-1, int(os.environ.get("TH", "8")))
rng = np.random.default_rng(0)
M, H, N = 4096, int(os.environ.get("HH", "4742")), 4096
w = (rng.standard_normal((H, M), dtype=np.float32) / 64)
lay = NativeLayer(w, w, H, H, 'silu', w, dtype='bf16')
for T in [int(t) for t in os.environ.get("TS", "16,32,48,64").split(",")]:
    x = rng.standard_normal((T, M))
    lay.cc_forward_host(x, threads=0)
    t0 = time.perf_counter(); 
    for _ in range(3): lay.cc_forward_host(x, threads=0)
    dt = (time.perf_counter()-t0)/3
    print(f"T={T}: {dt*1e3:.2f} ms  {lay.placed_bytes()['cc']/dt/1e9:.1f} GB/s  {2*T*3*M*H/dt/1e12:.2f} TFLOP/s", flush=True)
