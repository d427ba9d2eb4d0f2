#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/probe_gg.py > gpurun_out/probe_gg.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ffn_block -c 12 --csv --log-file gpurun_out/probe_gg_ncu.csv python scripts/probe_gg.py > /dev/null 2>&1
echo done
