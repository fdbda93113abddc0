# tile height 16 (128-thread CTAs) vs 32 (dev tool)
echo "== tz32"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== tz16"; HV_LIB=build/libhv_tz16.so python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
HV_LIB=build/libhv_tz16.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg0 or ragged" 2>&1 | tail -2
