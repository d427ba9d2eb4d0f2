"""One grouped GG launch as in a decode step (2 Mixtral experts, 7168 GG rows
each, bf16 SwiGLU, T = 1) -- the launch the bench's roofline is about, for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15715_b200 import _native as nat  # noqa: E402
from paper_2411_15715_b200.sliced import CallSpec, NativeLayer, forward_calls  # noqa: E402

nat.init(0)
M, H = 4096, 7168
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) / 64).to(torch.bfloat16).cpu()  # noqa: E731
lays = [NativeLayer(mk(H, M), mk(H, M), 0, 0, "silu", mk(H, M), dtype="bf16") for _ in range(2)]
x = torch.randn(1, M, device="cuda").to(torch.bfloat16)
for _ in range(3):
    forward_calls([CallSpec(l) for l in lays], x)
torch.cuda.synchronize()
