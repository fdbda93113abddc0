set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "resident_q or edge" > gpurun_out/g44_parity.log 2>&1; tail -3 gpurun_out/g44_parity.log
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g44_$1.json 2> gpurun_out/g44_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g44_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g44_$1.err
}
C3="--config 3 --shots 16 --nt 400"
ev split "$C3"
ev nosplit "$C3" HV_QRES_SPLIT=0
ev split_b "$C3"
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
timeout 900 ncu --set full --clock-control none -k regex:fwd_qres -s 20 -c 2 -o gpurun_out/g44_fwd $P > gpurun_out/g44_ncu.log 2>&1; echo ncu=$?
timeout 1200 python -m pytest tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/g44_golden.log 2>&1; tail -3 gpurun_out/g44_golden.log
