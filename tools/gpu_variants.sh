# activity tracking: parity first, then timings with and without (dev tool)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ptr.log 2>&1; echo ptr=$?; tail -15 gpurun_out/ptr.log
echo "== track"; python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1
echo "== notrack"; HV_TRACK=0 python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1
echo "== track cfg2"; timeout 600 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernels'])"
