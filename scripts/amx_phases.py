"""AMX CC kernel phase times (SP_AMX_PROF=1 lines of scripts/bench_amx.py on stdin):
median pack / up / down per token count, and the kernel's TFLOP/s over the three
phases (the call's allocations and x conversion excluded)."""
import re
import sys
from collections import defaultdict

import numpy as np

M, H, N = 4096, 4742, 4096
ph = defaultdict(list)
for line in sys.stdin:
    m = re.match(r"amx T=(\d+): pack (\d+) us\s+up (\d+) us\s+down (\d+) us", line.strip())
    if m:
        T, a, b, c = map(int, m.groups())
        ph[T].append((a, b, c))
for T in sorted(ph):
    a = np.array(ph[T][2:] or ph[T], dtype=float)
    pk, up, dn = np.median(a, axis=0)
    fl_up, fl_dn = 2 * T * M * H * 2, 2 * T * H * N
    print(f"T={T}: pack {pk:6.0f}  up {up:6.0f} us ({fl_up / up / 1e6:5.2f} TFLOP/s)  down {dn:6.0f} us "
          f"({fl_dn / dn / 1e6:5.2f} TFLOP/s)  kernel {(fl_up + fl_dn) / (pk + up + dn) / 1e6:5.2f} TFLOP/s")
