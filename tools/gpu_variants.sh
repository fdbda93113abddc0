# runtime unit order: cfg1 (Q 28 MB, group-shot-tile), cfg3 and the cfg4 grid (tile-major) (dev tool)
python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
timeout 900 python bench.py --config 4 --shots 4 --nt 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernels'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
