set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err; echo bench=$?
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
timeout 300 $P > gpurun_out/c3_plain.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_qres -s 10 -c 1 -o gpurun_out/c3_fwd $P > gpurun_out/c3_ncu_fwd.log 2>&1; echo ncu_fwd=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_step -s 10 -c 1 -o gpurun_out/c3_bwd $P > gpurun_out/c3_ncu_bwd.log 2>&1; echo ncu_bwd=$?
