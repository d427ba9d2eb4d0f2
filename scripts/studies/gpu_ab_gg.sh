#!/bin/bash
# GG placement A/B (SP_GG_LAST 1 = after the last copy is queued, 2 = behind the last chunk kernel),
# fixed rates (no per-box re-solve), cfg4 and cfg2, alternating on one box
bash scripts/gpu_ab.sh SP_GG_LAST "1 2" "--config cfg4 --steps 60 --calibrate 0" 5
mv gpurun_out/ab_SP_GG_LAST.log gpurun_out/ab_gg_cfg4.log
bash scripts/gpu_ab.sh SP_GG_LAST "1 2" "--steps 100 --calibrate 0" 5
mv gpurun_out/ab_SP_GG_LAST.log gpurun_out/ab_gg_cfg2.log
