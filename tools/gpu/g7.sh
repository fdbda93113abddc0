# resident-q forward, paired arithmetic + block barrier: timing and ncu
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident_q or cfg0" > gpurun_out/g7_t.log 2>&1; echo t=$?
tail -2 gpurun_out/g7_t.log
timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g7_c3.json 2> gpurun_out/g7_c3.err; echo c3=$?
python -c "import json;d=json.loads(open('gpurun_out/g7_c3.json').read().strip().splitlines()[-1]);print('c3', round(d['value'],3), {k:(round(v['avg_launch_ms']*1e3,1),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
timeout 300 $P > gpurun_out/g7_plain.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_qres -s 10 -c 1 -o gpurun_out/g7_fwd $P > gpurun_out/g7_ncu_fwd.log 2>&1; echo ncu_fwd=$?
