# backward stages 4 vs 3 with the s^j stage (dev tool)
for i in 1 2; do
echo "== ns3"; python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
echo "== ns4"; HV_LIB=build/libhv_ns4.so python tools/tune.py --config 1 --S 16 --FG 0 --reps 2 2>&1 | tail -1
done
