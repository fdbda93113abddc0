set -x
ev() { # tag args [env]
  env $3 timeout 300 python bench.py $2 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g31_$1.json 2> gpurun_out/g31_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/g31_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g31_$1.err
}
C3="--config 3 --shots 16 --nt 400"
ev o0 "$C3" HV_QRES_ORDER=0
ev o2 "$C3" HV_QRES_ORDER=2
ev o3 "$C3" HV_QRES_ORDER=3
ev o0b "$C3" HV_QRES_ORDER=0
ev o2b "$C3" HV_QRES_ORDER=2
P="python tools/profile_step.py --config 3 --shots 16 --nt 40 --reps 1"
for o in 2 3; do
HV_QRES_ORDER=$o timeout 900 ncu --set full --clock-control none -k regex:fwd_qres -s 10 -c 1 -o gpurun_out/g31_fwd_o$o $P > gpurun_out/g31_ncu_o$o.log 2>&1; echo ncu_o$o=$?
done
