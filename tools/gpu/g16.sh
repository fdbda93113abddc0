# backward: s^j loaded with an L2 evict_last policy (read by every field group's CTA): timing + DRAM bytes
set -x
for L in libhv libhv_sjl; do
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g16_$L.json 2> gpurun_out/g16_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/g16_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
  P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
  HV_LIB=$PWD/paper_2507_10804_b200/$L.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:bwd_step -s 10 -c 2 $P > gpurun_out/g16_ncu_$L.log 2>&1
  grep -E "duration|dram__bytes|hit_rate" gpurun_out/g16_ncu_$L.log | head -8
done
