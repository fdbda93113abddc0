# persistent backward vs previous commit (dev tool)
for sh in 16 2; do
echo "== prev shots $sh"; HV_LIB=build/libhv_prev.so python tools/tune.py --config 1 --shots $sh --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== pers shots $sh"; python tools/tune.py --config 1 --shots $sh --S 16 --FG 0 --reps 2 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
