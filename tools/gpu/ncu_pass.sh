#!/bin/bash
# ncu part of tools/measure_round.sh plus the evidence lines (tests / smoke / bench already run with tools/gpu/final.sh)
set -x
TAG=${1:-r02}
E="--steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 python bench.py --config 1 $E > gpurun_out/ev_cfg1_$TAG.json 2>&1; echo ev_cfg1=$?
timeout 900 python bench.py --config 2 --mode fused $E --no-e2e > gpurun_out/ev_cfg2_fused_$TAG.json 2>&1; echo ev_cfg2=$?
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 6000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
$P > gpurun_out/plain_prof_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_qres -s 10 -c 1 -o gpurun_out/prof_fwd_$TAG $P > gpurun_out/ncu_fwd_$TAG.log 2>&1; echo ncu_fwd=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_step -s 10 -c 1 -o gpurun_out/prof_bwd_$TAG $P > gpurun_out/ncu_bwd_$TAG.log 2>&1; echo ncu_bwd=$?
timeout 900 python bench.py --config 4 --shots 4 --nt 400 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev_cfg4grid_$TAG.json 2>&1; echo ev_cfg4=$?
P4="python tools/profile_step.py --config 4 --shots 4 --nt 12 --reps 1"
$P4 > gpurun_out/plain_prof4_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:fwd_qres -s 4 -c 1 -o gpurun_out/prof_fwd_cfg4_$TAG $P4 > gpurun_out/ncu_fwd4_$TAG.log 2>&1; echo ncu_fwd4=$?
timeout 900 ncu --set full --clock-control none -k regex:bwd_step -s 4 -c 1 -o gpurun_out/prof_bwd_cfg4_$TAG $P4 > gpurun_out/ncu_bwd4_$TAG.log 2>&1; echo ncu_bwd4=$?
