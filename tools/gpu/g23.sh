set -x
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
$P > gpurun_out/g23_plain.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_qres -s 10 -c 1 -o gpurun_out/g23_fwd $P > gpurun_out/g23_ncu_fwd.log 2>&1; echo ncu_fwd=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_step -s 10 -c 1 -o gpurun_out/g23_bwd $P > gpurun_out/g23_ncu_bwd.log 2>&1; echo ncu_bwd=$?
(nvidia-smi --query-gpu=power.draw,power.limit,clocks.sm,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/g23_power.csv &) 
timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g23_ev.json 2> gpurun_out/g23_ev.err; echo ev=$?
tail -c 600 gpurun_out/g23_ev.json
