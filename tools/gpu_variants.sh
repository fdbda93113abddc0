# A/B timing of launch/kernel variants on cfg 1 (dev tool): bash tools/gpu_variants.sh
for v in 1 3; do echo "== bwd FG $v"; HV_LIB=build/libhv_bfg$v.so python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1; done
echo "== default"; python tools/tune.py --config 1 --S 16 --FG 16 --reps 2 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
