set -x
ev() { # lib tag args
  HV_LIB=$PWD/paper_2507_10804_b200/$1.so timeout 300 python bench.py $3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g33_$1_$2.json 2> gpurun_out/g33_$1_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/g33_$1_$2.json').read().strip().splitlines()[-1]);print('$1 $2', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g33_$1_$2.err
}
for L in libhv libhv_fg3 libhv_fg4; do
ev $L c3 "--config 3 --shots 16 --nt 400"
ev $L c1 "--config 1"
done
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
for L in libhv_fg3 libhv_fg4; do
HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 900 ncu --set full --clock-control none -k regex:bwd_step -s 10 -c 1 -o gpurun_out/g33_bwd_$L $P > gpurun_out/g33_ncu_$L.log 2>&1; echo ncu_$L=$?
done
