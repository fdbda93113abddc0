set -x
for L in libhv libhv_go32; do
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g22_$L.json 2> gpurun_out/g22_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/g22_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
done
HV_LIB=$PWD/paper_2507_10804_b200/libhv_go32.so timeout 300 python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g22_c1.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/g22_c1.json').read().strip().splitlines()[-1]);print('c1 go32', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
