# resident-q vs one-wave forward on cfg 2 (Q = 16 MB) (dev tool)
for q in 0 1; do echo "== cfg2 qres $q"; HV_QRES=$q python tools/tune.py --config 2 --shots 22 --S 22 --FG 0 --reps 1 2>&1 | tail -1; done
for q in 0 1; do echo "== cfg2 qres $q qfg 8"; HV_QRES=$q HV_QFG=8 python tools/tune.py --config 2 --shots 22 --S 22 --FG 0 --reps 1 2>&1 | tail -1; done
