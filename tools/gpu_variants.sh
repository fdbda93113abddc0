# backward paired arithmetic A/B (dev tool)
echo "== bp1"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== bp0"; HV_LIB=build/libhv_bp0.so python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== bp1"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== bp0"; HV_LIB=build/libhv_bp0.so python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
