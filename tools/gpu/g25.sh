set -x
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
HV_LIB=$PWD/paper_2507_10804_b200/libhv_rz4.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_qres|bwd_step" -s 20 -c 2 -o gpurun_out/g25_rz4 $P > gpurun_out/g25_ncu.log 2>&1; echo ncu=$?
run() {
  HV_LIB=$PWD/paper_2507_10804_b200/$1.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/g25_$1_$2.json 2> gpurun_out/g25_$1_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/g25_$1_$2.json').read().strip().splitlines()[-1]);print('$1 $2', round(d['value'],4), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks'])"
}
run libhv a
run libhv_rz4 a
run libhv b
run libhv_rz4 b
