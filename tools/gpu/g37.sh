set -x
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g37_$1.json 2> gpurun_out/g37_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g37_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g37_$1.err
}
C3="--config 3 --shots 16 --nt 400"
for q in 6 4 5 3; do ev q$q "$C3" HV_QFG=$q; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "duplicate" > gpurun_out/g37_dup.log 2>&1; tail -2 gpurun_out/g37_dup.log
