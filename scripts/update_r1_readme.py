"""Rewrite the numbers in profiles/r1/README.md's headline and per-config tables
from the bench_*.json lines next to it (run after copying a fresh
scripts/gpu_all_configs.sh run into profiles/r1/)."""
import json
import re
from pathlib import Path

R1 = Path(__file__).resolve().parents[1] / "profiles" / "r1"
g = lambda n: json.loads((R1 / f"{n}.json").read_text())  # noqa: E731
v = lambda n: g(n)["value"]  # noqa: E731
e = lambda n: g(n)["e2e"]["value"]  # noqa: E731
b = lambda n: g(n)["link"]["step_bound_with_cc_frac"]  # noqa: E731


def fr(n):
    r = g(n)["roofline"]
    return r["frac"], r["frac_device_span"]


s = (R1 / "README.md").read_text()
c2, ref = g("bench_cfg2"), g("bench_reference")
r2 = c2["roofline"]
heads = {
    "| value (x in HBM) |": f"| value (x in HBM) | **{v('bench_cfg2'):.1f} tokens/s** ({c2['ms_per_step']:.2f} ms/step) |",
    "| e2e (host x/y through the public API) |": f"| e2e (host x/y through the public API) | **{e('bench_cfg2'):.1f} tokens/s** |",
    "| reference arm (fp64 numpy sliced forward, 16 threads, `bench_reference.json`) |":
        f"| reference arm (fp64 numpy sliced forward, 16 threads, `bench_reference.json`) | {ref['value']:.1f} tokens/s on the "
        f"same box (e2e speed-up {e('bench_cfg2') / ref['value']:.1f}x; the arm itself ranges 39-58 across boxes) |",
    "| step bound max(GG/HBM, CG/link, CC/host rate) ÷ step |":
        f"| step bound max(GG/HBM, CG/link, CC/host rate) ÷ step | {b('bench_cfg2'):.2f} (north-star roofline "
        f"max(GG/HBM, CG/link): {c2['link']['step_roofline_frac']:.2f}) |",
    "| GG ffn_block launch, in-kernel %globaltimer span |":
        f"| GG ffn_block launch, in-kernel %globaltimer span | {r2['device_span_us']:.1f} µs → "
        f"{r2['achieved_device_span'] / 1000:.2f} TB/s = **{r2['frac_device_span']:.2f}** of measured HBM |",
    "| same launch, CUDA-event span |": f"| same launch, CUDA-event span | {r2['mean_launch_us']:.0f} µs → {r2['frac']:.2f} (see \"event spans\" below) |",
}


def row(fname, label, val, e2, bound, gg):
    return f"| `{fname}` | {label} | {val} | {e2} | {bound} | {gg} |"


def series(prefix, xs, f, fmt):
    return " / ".join(fmt.format(f(f"{prefix}{x}")) for x in xs)


rows = {
    "| `bench_cfg1.json`": row("bench_cfg1.json", "1024/3584 fp32, 8 experts top-2, fixed 0.2/0.3/0.5", f"{v('bench_cfg1'):.0f}",
                               f"{e('bench_cfg1'):.0f}", f"{b('bench_cfg1'):.2f}",
                               f"{fr('bench_cfg1')[0]:.2f} / {fr('bench_cfg1')[1]:.2f} (22 MB launch, latency bound)"),
    "| `bench_cfg2.json`": row("bench_cfg2.json", "Mixtral-8x7B layer, decode b1", f"**{v('bench_cfg2'):.0f}**",
                               f"**{e('bench_cfg2'):.0f}**", f"{b('bench_cfg2'):.2f}",
                               f"{fr('bench_cfg2')[0]:.2f} / {fr('bench_cfg2')[1]:.2f}"),
    "| `bench_cfg3.json`": row("bench_cfg3.json", "32-layer Mixtral stack, 512-token prompt with `solve_ng` split",
                               f"**{v('bench_cfg3'):.0f} prefill** ({g('bench_cfg3')['decode_tokens_per_s']:.0f} decode)",
                               f"{e('bench_cfg3'):.0f}", "link bound", "—"),
    "| `bench_cfg3_layerplan.json`": row("bench_cfg3_layerplan.json",
                                         "same, token split from the layer-level extension planner (not the reference's)",
                                         f"{v('bench_cfg3_layerplan'):.0f} prefill", f"{e('bench_cfg3_layerplan'):.0f}",
                                         "link ≈ host", "—"),
    "| `bench_cfg4.json`": row("bench_cfg4.json", "LLaMA-2-70B dense FFN (1-GPU shard = whole layer)", f"{v('bench_cfg4'):.0f}",
                               f"{e('bench_cfg4'):.0f}", f"{b('bench_cfg4'):.2f}",
                               f"{fr('bench_cfg4')[0]:.2f} / {fr('bench_cfg4')[1]:.2f}"),
    "| `bench_cfg5_8x22b": row("bench_cfg5_8x22b_b{1,4,16,32}.json", "Mixtral-8x22B, batch 1/4/16/32",
                               series("bench_cfg5_8x22b_b", (1, 4, 16, 32), v, "{:.0f}"),
                               series("bench_cfg5_8x22b_b", (1, 4, 16, 32), e, "{:.0f}"),
                               series("bench_cfg5_8x22b_b", (1, 4, 16, 32), b, "{:.2f}"), "—"),
    "| `bench_cfg5_phimoe": row("bench_cfg5_phimoe_b{1,8,32}.json", "PhiMoE 16 experts, batch 1/8/32",
                                series("bench_cfg5_phimoe_b", (1, 8, 32), v, "{:.0f}"),
                                series("bench_cfg5_phimoe_b", (1, 8, 32), e, "{:.0f}"),
                                series("bench_cfg5_phimoe_b", (1, 8, 32), b, "{:.2f}"), "—"),
    "| `bench_model_decode.json`": row("bench_model_decode.json",
                                       "32-layer decoder (attention + KV cache + sliced MoE): 512-token prefill, then decode with CUDA graphs",
                                       f"{v('bench_model_decode'):.1f} decode ({g('bench_model_decode')['prefill_tokens_per_s']:.0f} prefill)",
                                       f"{e('bench_model_decode'):.1f}", "—", "—"),
}
out = []
for line in s.splitlines():
    for k, nl in {**heads, **rows}.items():
        if line.startswith(k):
            line = nl
    out.append(line)
s = "\n".join(out) + "\n"
a = g("bench_cfg2_all_gg")
s = re.sub(r"\(`--budget-frac 1.0`, rates 0/0/1, `bench_cfg2_all_gg.json`\): \*\*\d+ tokens/s\*\*\n\(e2e \d+\)",
           f"(`--budget-frac 1.0`, rates 0/0/1, `bench_cfg2_all_gg.json`): **{a['value']:.0f} tokens/s**\n(e2e {a['e2e']['value']:.0f})", s)
(R1 / "README.md").write_text(s)
print("updated")
