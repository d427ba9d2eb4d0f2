#!/bin/bash
mkdir -p gpurun_out
SP_KSTAMPS=1 timeout 300 python scripts/probe_gg.py > gpurun_out/probe_gg.log 2>&1
echo done
