# T = 2 forward: bitwise test vs single-step, then per-level timing on cfg3 (16 shots, nt 400) and cfg1
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "t2_forward" > gpurun_out/g3_t2.log 2>&1; echo t2=$?
tail -15 gpurun_out/g3_t2.log
for T in 0 1; do
HV_T2=$T timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g3_c3_t$T.json 2> gpurun_out/g3_c3_t$T.err; echo c3_t$T=$?
python -c "import json;d=json.loads(open('gpurun_out/g3_c3_t$T.json').read().strip().splitlines()[-1]);print('T2=$T', d['value'], {k:(v['avg_launch_ms'],v['frac']) for k,v in d['roofline']['kernels'].items()})"
HV_T2=$T timeout 300 python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g3_c1_t$T.json 2> gpurun_out/g3_c1_t$T.err; echo c1_t$T=$?
python -c "import json;d=json.loads(open('gpurun_out/g3_c1_t$T.json').read().strip().splitlines()[-1]);print('T2=$T', d['value'], {k:(v['avg_launch_ms'],v['frac']) for k,v in d['roofline']['kernels'].items()})"
done
tail -3 gpurun_out/g3_c3_t1.err
