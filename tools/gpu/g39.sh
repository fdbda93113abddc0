set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "t2 or forward_only or resident or edge or duplicate" > gpurun_out/g39_parity.log 2>&1; tail -3 gpurun_out/g39_parity.log
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/g39_golden.log 2>&1; tail -3 gpurun_out/g39_golden.log
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g39_$1.json 2> gpurun_out/g39_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g39_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],4), d['ms_per_step'], {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g39_$1.err
}
ev m3 "--config 3 --mode misfit"
ev m3b "--config 3 --mode misfit"
ev m1 "--config 1 --mode misfit"
ev c3 "--config 3 --shots 16 --nt 400"
