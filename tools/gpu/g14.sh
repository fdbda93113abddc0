# cfg4-grid evidence (the >= 70 % roofline is judged on the cfg 4 grid) + ncu of both step kernels there
set -x
timeout 900 python bench.py --config 4 --shots 4 --nt 400 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev_cfg4grid_r02b.json 2> gpurun_out/ev_cfg4grid_r02b.err; echo ev=$?
python -c "import json;d=json.loads(open('gpurun_out/ev_cfg4grid_r02b.json').read().strip().splitlines()[-1]);print(round(d['value'],3), d['config']['shot_batch'], {k:(round(v['avg_launch_ms']*1e3,1),round(v['frac'],3),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
P="python tools/profile_step.py --config 4 --shots 4 --nt 12 --reps 1"
timeout 600 $P > gpurun_out/g14_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/g14_plain.log
timeout 900 ncu --set full --clock-control none -k regex:fwd_qres -s 4 -c 1 -o gpurun_out/prof_fwd_cfg4_r02b $P > gpurun_out/g14_ncu_fwd.log 2>&1; echo ncu_fwd=$?
timeout 900 ncu --set full --clock-control none -k regex:bwd_step -s 4 -c 1 -o gpurun_out/prof_bwd_cfg4_r02b $P > gpurun_out/g14_ncu_bwd.log 2>&1; echo ncu_bwd=$?
