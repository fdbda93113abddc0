# T = 2 forward + adjoint: parity vs single-step, timings, ncu of both T = 2 kernels on cfg3
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "t2_kernels" > gpurun_out/g4_t2.log 2>&1; echo t2=$?
tail -25 gpurun_out/g4_t2.log
for T in 0 1; do
HV_T2=$T timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g4_c3_t$T.json 2> gpurun_out/g4_c3_t$T.err; echo c3_t$T=$?
python -c "import json;d=json.loads(open('gpurun_out/g4_c3_t$T.json').read().strip().splitlines()[-1]);print('T2=$T', d['value'], {k:(v['avg_launch_ms'],v['frac']) for k,v in d['roofline']['kernels'].items()})"
done
P="python tools/profile_step.py --config 3 --shots 16 --nt 20 --reps 1"
HV_T2=1 timeout 300 $P > gpurun_out/g4_plain.log 2>&1; echo plain=$?
cat gpurun_out/g4_plain.log
HV_T2=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_t2 -s 3 -c 1 -o gpurun_out/g4_fwd_t2 $P > gpurun_out/g4_ncu_fwd.log 2>&1; echo ncu_fwd=$?
HV_T2=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_t2 -s 3 -c 1 -o gpurun_out/g4_bwd_t2 $P > gpurun_out/g4_ncu_bwd.log 2>&1; echo ncu_bwd=$?
