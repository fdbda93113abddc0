for v in "$@"; do
  echo "== $v"; HV_LIB=build/libhv_$v.so timeout 300 python tools/tune.py --config 1 --S 16 --FG 4,6 --reps 2 2>&1 | tail -2
done
