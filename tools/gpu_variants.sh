# A/B timing of launch/kernel variants on cfg 1 (dev tool): bash tools/gpu_variants.sh
for v in split1 split4; do echo "== $v"; HV_LIB=build/libhv_$v.so python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1; done
echo "== split2"; python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
