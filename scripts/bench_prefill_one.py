"""One GG-block prefill forward (Mixtral expert, H hidden rows in HBM, T tokens) for ncu launch lists."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402

nat.init(0)
M = 4096
H = int(sys.argv[1]) if len(sys.argv) > 1 else 14336
Ts = [int(t) for t in (sys.argv[2] if len(sys.argv) > 2 else "128,512").split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lay = NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16")
for T in Ts:
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    for _ in range(2):
        forward_calls([CallSpec(lay)], x)
    torch.cuda.synchronize()
