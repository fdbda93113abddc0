# compile-time knob sweep at cfg 3 (16 shots, nt 400)
set -x
for L in libhv libhv_bfg1 libhv_bfg3 libhv_tz16 libhv_ns4; do
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g19_$L.json 2> gpurun_out/g19_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/g19_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})" || tail -3 gpurun_out/g19_$L.err
done
