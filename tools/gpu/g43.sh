set -x
ev() { # lib tag args
  HV_LIB=$PWD/paper_2507_10804_b200/$1.so timeout 300 python bench.py $3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g43_$1_$2.json 2> gpurun_out/g43_$1_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/g43_$1_$2.json').read().strip().splitlines()[-1]);print('$1 $2', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g43_$1_$2.err
}
for L in libhv libhv_sp2 libhv_sp3; do
ev $L c1 "--config 1"
ev $L c3 "--config 3 --shots 16 --nt 400"
done
