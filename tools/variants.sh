# usage: bash tools/variants.sh "FG list" tag1 tag2 ...
FGS=$1; shift
for v in "$@"; do
  echo "== $v"; HV_LIB=build/libhv_$v.so timeout 300 python tools/tune.py --config 1 --S 16 --FG $FGS --reps 2 2>&1 | tail -3
done
