set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "t2 or forward_only or resident or edge or duplicate" > gpurun_out/g40_parity.log 2>&1; tail -3 gpurun_out/g40_parity.log
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g40_$1.json 2> gpurun_out/g40_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g40_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],4), d['ms_per_step'], {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g40_$1.err
}
ev m3 "--config 3 --mode misfit"
