# resident-q forward grid order: tiles fastest (0) vs field group fastest (1)
set -x
for O in 0 1; do
  HV_QRES_ORDER=$O timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g18_$O.json 2> gpurun_out/g18_$O.err
  python -c "import json;d=json.loads(open('gpurun_out/g18_$O.json').read().strip().splitlines()[-1]);print('order $O', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
  P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
  HV_QRES_ORDER=$O timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:qres -s 10 -c 1 $P > gpurun_out/g18_ncu_$O.log 2>&1
  grep -E "duration|dram__bytes|hit_rate" gpurun_out/g18_ncu_$O.log | head -4
  HV_QRES_ORDER=$O timeout 600 python bench.py --config 4 --shots 4 --nt 200 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g18_c4_$O.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/g18_c4_$O.json').read().strip().splitlines()[-1]);print('c4 order $O', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_q or cfg0" > gpurun_out/g18_t.log 2>&1; echo t=$?; tail -1 gpurun_out/g18_t.log
