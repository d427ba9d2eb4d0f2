#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 > gpurun_out/bench_cfg3.log 2>&1
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 --token-plan layer > gpurun_out/bench_cfg3_layerplan.log 2>&1
echo done
