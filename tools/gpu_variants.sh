# backward fields per CTA at small per-rank shot counts (dev tool)
for sh in 2 4; do
echo "== default shots $sh"; python tools/tune.py --config 1 --shots $sh --S 16 --FG 0 --reps 2 2>&1 | tail -1
for v in 3 4; do echo "== bfg$v shots $sh"; HV_LIB=build/libhv_bfg$v.so python tools/tune.py --config 1 --shots $sh --S 16 --FG 0 --reps 2 2>&1 | tail -1; done
done
