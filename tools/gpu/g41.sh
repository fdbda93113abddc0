set -x
ev() { # tag args [env]
  env $3 timeout 600 python bench.py $2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g41_$1.json 2> gpurun_out/g41_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g41_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],4), d['ms_per_step'], {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g41_$1.err
}
C2="--config 2 --mode fused"
ev f_base "$C2"
ev f_t2 "$C2" "HV_T2=1 HV_T2B=0"
ev f_t2b "$C2" "HV_T2=1 HV_T2B=1"
