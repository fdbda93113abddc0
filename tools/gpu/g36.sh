set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "duplicate or edge or ragged or cfg0 or resident" > gpurun_out/g36_parity.log 2>&1; tail -3 gpurun_out/g36_parity.log
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g36_$1.json 2> gpurun_out/g36_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g36_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g36_$1.err
}
ev c3 "--config 3 --shots 16 --nt 400"
ev c1 "--config 1"
ev c3b "--config 3 --shots 16 --nt 400"
