set -x
run() { # lib tag [env]
  env $3 HV_LIB=$PWD/paper_2507_10804_b200/$1.so timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/g32_$2.json 2> gpurun_out/g32_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/g32_$2.json').read().strip().splitlines()[-1]);print('$2', round(d['value'],4), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks'])" || tail -3 gpurun_out/g32_$2.err
}
run libhv base
run libhv t2rz4 HV_T2=1
run libhv_rz2 t2rz2 HV_T2=1
run libhv base2
