# tile height 64 (512-thread CTAs, 1 per SM) vs 32 (dev tool)
echo "== tz32"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== tz64"; HV_LIB=build/libhv_tz64.so python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== tz64 2 shots"; HV_LIB=build/libhv_tz64.so python tools/tune.py --config 1 --shots 2 --S 16 --FG 0 --reps 2 2>&1 | tail -1
HV_LIB=build/libhv_tz64.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg0 or ragged" 2>&1 | tail -2
