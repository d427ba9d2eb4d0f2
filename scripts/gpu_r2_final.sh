#!/bin/bash
# Round-2 evidence on one box: the GPU test suite, the default bench (twice) and
# the reference arm, the ncu launch list of the bench command, one ncu --set
# full capture of the grouped GG launch (scripts/gg_group_one.py), and every
# BASELINE config.
mkdir -p gpurun_out/final/cfg
F=gpurun_out/final
timeout 1500 python -m pytest tests -q -m gpu -s -p no:cacheprovider > $F/gputest.log 2>&1; echo "tests rc=$?" >> $F/gputest.log; grep -E "passed|failed|rc=" $F/gputest.log | tail -3
for i in 1 2; do timeout 600 python bench.py > $F/bench_cfg2_$i.json 2> $F/bench_cfg2_$i.err; done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $F/bench_reference.json 2> $F/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $F/ncu_launches_bench_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --calibrate 0 > /dev/null 2>&1
python scripts/ncu_launch_table.py $F/ncu_launches_bench_cfg2.csv --summary > $F/ncu_launches_bench_cfg2_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_block_kernel -s 2 -c 1 -o $F/ncu_full_gg python scripts/gg_group_one.py > $F/ncu_full_gg.log 2>&1
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $F/cfg/$name.log 2>&1; grep '^{' $F/cfg/$name.log | tail -1 > $F/cfg/$name.json; }
run bench_cfg1 --config cfg1 --steps 100 --warmup 5
run bench_cfg4 --config cfg4 --steps 30 --no-cpu-baseline
for b in 1 4 16 32; do run bench_cfg5_8x22b_b$b --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline; done
for b in 1 8 32; do run bench_cfg5_phimoe_b$b --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline; done
run bench_cfg3 --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 128
run bench_cfg3_layerplan --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 128 --token-plan layer
run bench_cfg2_all_gg --budget-frac 1.0 --steps 200 --warmup 10 --no-cpu-baseline
echo done
