# T = 2 kernels with tile-fastest grid order: parity + per-level timings + ncu L2 hit rate
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "t2_kernels" > gpurun_out/g9_t2.log 2>&1; echo t2=$?
tail -2 gpurun_out/g9_t2.log
run() {
  HV_LIB=$2 HV_T2=$3 timeout 300 python bench.py --config $4 $5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g9_$1.json 2> gpurun_out/g9_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g9_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:(round(v['avg_launch_ms']*1e3,1),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
}
L0=$PWD/paper_2507_10804_b200/libhv.so
L1=$PWD/paper_2507_10804_b200/libhv_oz24.so
run c3_t2_56 $L0 1 3 "--shots 16 --nt 400"
run c3_t2_24 $L1 1 3 "--shots 16 --nt 400"
run c1_t2_56 $L0 1 1 ""
run c1_t2_24 $L1 1 1 ""
P="python tools/profile_step.py --config 3 --shots 16 --nt 20 --reps 1"
HV_T2=1 timeout 300 $P > gpurun_out/g9_plain.log 2>&1; echo plain=$?
HV_T2=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:_t2_ -s 2 -c 4 $P > gpurun_out/g9_ncu.log 2>&1; echo ncu=$?
grep -E "t2_kernel|duration|dram__bytes|hit_rate|issue_active" gpurun_out/g9_ncu.log | head -30
