# unit order on cfg3 (Q = 66 MB) and cfg2 (dev tool)
for o in gst gts; do echo "== cfg3 $o"; HV_UNIT_ORDER=$o python tools/tune.py --config 3 --shots 16 --S 16 --FG 0 --reps 1 2>&1 | tail -1; done
for o in gst gts; do echo "== cfg2 $o"; HV_UNIT_ORDER=$o python tools/tune.py --config 2 --shots 22 --S 22 --FG 0 --reps 1 2>&1 | tail -1; done
