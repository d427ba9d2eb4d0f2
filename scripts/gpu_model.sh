#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_model.py tests/test_store.py -x -q -m gpu > gpurun_out/gpu_tests_model.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests_model.log
timeout 900 python bench.py --config model --layers 32 --distinct-layers 4 --prompt 512 --steps 16 --warmup 3 > gpurun_out/bench_model.log 2>&1
echo done
