# backward w through TMA (dev tool)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1; done
python tools/tune.py --config 1 --shots 2 --S 16 --FG 0 --reps 2 2>&1 | tail -1
