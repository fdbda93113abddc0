# L2 policies: backward lambda^{j+2} evict_first (v1), resident-q background halo evict_last (v2)
set -x
for L in libhv libhv_v1 libhv_v2; do
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g17_$L.json 2> gpurun_out/g17_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/g17_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
  P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qres|bwd_step" -s 20 -c 2 $P > gpurun_out/g17_ncu_$L.log 2>&1
  grep -E "qres_kernel|bwd_step_kernel|duration|dram__bytes" gpurun_out/g17_ncu_$L.log | head -8
done
HV_LIB=$PWD/paper_2507_10804_b200/libhv.so timeout 300 python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g17_c1.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/g17_c1.json').read().strip().splitlines()[-1]);print('c1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
