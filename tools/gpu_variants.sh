# storage modes on cfg 1 (dev tool)
for st in full checkpoint boundary; do echo "== $st"; python tools/tune.py --config 1 --S 16 --FG 0 --store $st --reps 2 2>&1 | tail -1; done
