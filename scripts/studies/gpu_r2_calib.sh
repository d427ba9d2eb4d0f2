#!/bin/bash
# Round-2: refbind GPU tests, then the default bench (per-box calibration on)
# alternating with --calibrate 0 on the same box.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_refbind.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2_refbind.log 2>&1; echo "refbind rc=$?"; tail -3 gpurun_out/r2_refbind.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_cal1_$i.json 2> gpurun_out/r2_cal1_$i.err; echo "cal1 rc=$?"
  timeout 600 python bench.py --no-cpu-baseline --calibrate 0 > gpurun_out/r2_cal0_$i.json 2> gpurun_out/r2_cal0_$i.err; echo "cal0 rc=$?"
done
python - <<'PY'
import json
for n in ["cal1_1","cal0_1","cal1_2","cal0_2"]:
    try:
        d=json.loads([l for l in open(f"gpurun_out/r2_{n}.json") if l.startswith("{")][0])
    except Exception as e:
        print(n, "ERR", e); continue
    m=d["model_vs_measured"]; c=d.get("calibration") or {}
    print(n, "value %.1f e2e %.1f ms %.3f full %.3f pred %.3f meas/pred %.3f frac %.3f dev %.3f k_cpu %s k_link %s rates %s" % (
        d["value"], d["e2e"]["value"], d["ms_per_step"], m["step_full_trace_s"]*1e3, m["t_fin_pred_s"]*1e3,
        m["meas_over_pred"], d["roofline"]["frac"], d["roofline"]["frac_device_span"], c.get("k_cpu"), c.get("k_link"),
        d["split"]["rates"]))
PY
