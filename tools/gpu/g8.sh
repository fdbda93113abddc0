# T = 2 kernels with NSTAGE items of lead: parity (both tile sizes) and per-level timings
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "t2_kernels" > gpurun_out/g8_t2.log 2>&1; echo t2=$?
tail -2 gpurun_out/g8_t2.log
HV_LIB=$PWD/paper_2507_10804_b200/libhv_oz24.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "t2_kernels" > gpurun_out/g8_t2_oz24.log 2>&1; echo t2oz24=$?
tail -2 gpurun_out/g8_t2_oz24.log
run() {
  HV_LIB=$2 HV_T2=$3 timeout 300 python bench.py --config $4 $5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g8_$1.json 2> gpurun_out/g8_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g8_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:(round(v['avg_launch_ms']*1e3,1),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
}
L0=$PWD/paper_2507_10804_b200/libhv.so
L1=$PWD/paper_2507_10804_b200/libhv_oz24.so
run c3_single $L0 0 3 "--shots 16 --nt 400"
run c3_t2_56 $L0 1 3 "--shots 16 --nt 400"
run c3_t2_24 $L1 1 3 "--shots 16 --nt 400"
run c1_t2_56 $L0 1 1 ""
run c1_t2_24 $L1 1 1 ""
