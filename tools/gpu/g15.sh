# resident-q forward: stages x resident fields trade-off (cfg3 16 shots nt 400, cfg4 grid)
set -x
for L in libhv libhv_q28 libhv_q44; do
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g15_$L.json 2> gpurun_out/g15_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/g15_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
done
HV_LIB=$PWD/paper_2507_10804_b200/libhv_q28.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_q" > gpurun_out/g15_t.log 2>&1; echo t=$?; tail -2 gpurun_out/g15_t.log
