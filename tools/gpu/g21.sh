# resident-q forward with thread-block clusters (background once per tile): parity + timing + DRAM bytes
set -x
HV_QRES_CLUSTER=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_q" > gpurun_out/g21_t.log 2>&1; echo t=$?; tail -3 gpurun_out/g21_t.log
HV_QRES_CLUSTER=1 timeout 900 python -m pytest tests/test_gpu_golden.py -q -x -k "cfg3" > gpurun_out/g21_g.log 2>&1; echo g=$?; tail -3 gpurun_out/g21_g.log
for C in 0 1; do
  HV_QRES_CLUSTER=$C timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g21_$C.json 2> gpurun_out/g21_$C.err
  python -c "import json;d=json.loads(open('gpurun_out/g21_$C.json').read().strip().splitlines()[-1]);print('cluster $C', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})" || tail -5 gpurun_out/g21_$C.err
  P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
  HV_QRES_CLUSTER=$C timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:qres -s 10 -c 1 $P > gpurun_out/g21_ncu_$C.log 2>&1
  grep -E "duration|dram__bytes|inst_executed" gpurun_out/g21_ncu_$C.log | head -4
done
