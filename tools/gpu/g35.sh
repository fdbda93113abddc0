set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/g35_parity.log 2>&1; tail -3 gpurun_out/g35_parity.log
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g35_$1.json 2> gpurun_out/g35_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g35_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g35_$1.err
}
ev c3 "--config 3 --shots 16 --nt 400"
ev c1 "--config 1"
ev c2f "--config 2 --mode fused"
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_step -s 10 -c 1 -o gpurun_out/g35_bwd $P > gpurun_out/g35_ncu_bwd.log 2>&1; echo ncu_bwd=$?
timeout 1200 python -m pytest tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/g35_golden.log 2>&1; tail -3 gpurun_out/g35_golden.log
