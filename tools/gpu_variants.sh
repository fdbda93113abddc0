# FG auto model: per-rank shot counts of the 2/4/8-GPU runs (dev tool)
for sh in 2 4 8; do
echo "== shots $sh FG16"; python tools/tune.py --config 1 --shots $sh --S 16 --FG 16 --reps 2 2>&1 | tail -1
echo "== shots $sh auto"; python tools/tune.py --config 1 --shots $sh --S 16 --FG 0 --reps 2 2>&1 | tail -1
done
echo "== 16 auto"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
