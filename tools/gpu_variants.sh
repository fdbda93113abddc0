# A/B timing of launch/kernel variants on cfg 1 (dev tool): bash tools/gpu_variants.sh
python tools/tune.py --config 1 --S 16 --FG 11,16,11,16,12,14 --reps 2 2>&1 | tail -6
