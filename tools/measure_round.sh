#!/bin/bash
# One measurement pass on the GPU box: tests, bench, ncu launch list of the bench command, full captures.
set -x
TAG=${1:-r01}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_exit=$?
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$?
tail -1 gpurun_out/bench_$TAG.json
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 4200 --csv \
      --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
P="python tools/profile_step.py --config 1 --reps 1"
$P > gpurun_out/plain_prof_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bwd_step -s 1000 -c 2 -o gpurun_out/prof_bwd_$TAG $P > gpurun_out/ncu_bwd_$TAG.log 2>&1; echo ncu_bwd=$?
ncu --set full --clock-control none --import-source on -k regex:fwd_step -s 1000 -c 2 -o gpurun_out/prof_fwd_$TAG $P > gpurun_out/ncu_fwd_$TAG.log 2>&1; echo ncu_fwd=$?
