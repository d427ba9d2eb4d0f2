"""Render a bench.py --trace-out timeline (reference Gantt schema, pipeline.py:347-364)
as an SVG Gantt chart: one lane per stream (host launch, copy engine, GPU, host CC threads).
usage: python scripts/timeline_svg.py trace.json out.svg [first_call] [n_calls]"""
import json
import sys

recs = json.load(open(sys.argv[1]))
first = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = int(sys.argv[4]) if len(sys.argv) > 4 else 2
recs = [r for r in recs if first <= r["call"] < first + n]
t0 = min(r["start_s"] for r in recs)
t1 = max(r["end_s"] for r in recs)
lanes = [("launch", "host enqueue"), ("transfer", "copy engine (CG / CC chunks)"), ("gpu", "GPU (GG, chunk kernels, merge)"),
         ("cpu", "host CC threads")]
colors = {"launch": "#999999", "copy": "#4c78a8", "gg": "#e45756", "cg": "#f58518", "cg_prime": "#b279a2",
          "merge": "#54a24b", "cc": "#72b7b2"}
W, LH, X0 = 1400, 46, 230
scale = (W - X0 - 20) / (t1 - t0)
out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{LH * len(lanes) + 70}" font-family="sans-serif" font-size="12">']
out.append(f'<text x="10" y="18">{sys.argv[1].split("/")[-1]}: calls {first}..{first + n - 1}, {1e3 * (t1 - t0):.2f} ms</text>')
for i, (lane, label) in enumerate(lanes):
    y = 30 + i * LH
    out.append(f'<text x="10" y="{y + 24}">{label}</text>')
    out.append(f'<line x1="{X0}" y1="{y + LH - 4}" x2="{W - 20}" y2="{y + LH - 4}" stroke="#ddd"/>')
    for r in recs:
        if r["stream"] != lane:
            continue
        x = X0 + (r["start_s"] - t0) * scale
        w = max(0.8, (r["end_s"] - r["start_s"]) * scale)
        c = colors.get(r["kind"], "#333")
        tip = f'{r["kind"]} call {r["call"]}: {1e6 * (r["end_s"] - r["start_s"]):.1f} us, {r["bytes"] / 1e6:.1f} MB'
        out.append(f'<rect x="{x:.1f}" y="{y + 6}" width="{w:.1f}" height="{LH - 14}" fill="{c}" stroke="white" stroke-width="0.5"><title>{tip}</title></rect>')
ticks = 10
for k in range(ticks + 1):
    x = X0 + k * (W - X0 - 20) / ticks
    out.append(f'<text x="{x:.0f}" y="{30 + len(lanes) * LH + 16}" text-anchor="middle">{1e3 * k * (t1 - t0) / ticks:.2f} ms</text>')
legend = " ".join(f'<tspan fill="{c}">&#9632; {k}</tspan>' for k, c in colors.items())
out.append(f'<text x="{X0}" y="{30 + len(lanes) * LH + 34}">{legend}</text>')
out.append("</svg>")
open(sys.argv[2], "w").write("\n".join(out))
