"""AMX CC kernel: median / best of REPS calls at each token count in TS (one 4096 x 4742 SwiGLU CC block, 16 host threads)."""
import numpy as np, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15715_b200 import _native as nat
from paper_2411_15715_b200.sliced import NativeLayer
nat.init(-1, 16)
rng = np.random.default_rng(0)
M, H, N = 4096, 4742, 4096
w = (rng.standard_normal((H, M), dtype=np.float32) / 64)
lay = NativeLayer(w, w, H, H, 'silu', w, dtype='bf16')
for T in [int(t) for t in os.environ.get("TS", "16,64,128").split(",")]:
    x = rng.standard_normal((T, M))
    for _ in range(2): lay.cc_forward_host(x, threads=0)
    ts = []
    for _ in range(int(os.environ.get("REPS", "10"))):
        t0 = time.perf_counter(); lay.cc_forward_host(x, threads=0); ts.append(time.perf_counter() - t0)
    dt = float(np.median(ts)); best = min(ts)
    print(f"T={T}: median {dt*1e3:.2f} ms (best {best*1e3:.2f})  {2*T*3*M*H/dt/1e12:.2f} TFLOP/s median", flush=True)
