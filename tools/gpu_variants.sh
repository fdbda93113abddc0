# s^j through TMA in the backward (dev tool)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for st in full checkpoint boundary; do echo "== $st"; python tools/tune.py --config 1 --S 16 --FG 0 --store $st --reps 2 2>&1 | tail -1; done
echo "== 2 shots"; python tools/tune.py --config 1 --shots 2 --S 16 --FG 0 --reps 2 2>&1 | tail -1
