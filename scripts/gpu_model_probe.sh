#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/probe_model.py > gpurun_out/probe_model.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_model.json >> gpurun_out/probe_model.log 2>&1
echo done
