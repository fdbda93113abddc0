# q_k L2 policy in the tile-major order (cfg3: Q = 66 MB; cfg4 grid: 3.3 GB) (dev tool)
for v in q0 cur q2; do
  L=build/libhv_$v.so; [ $v = cur ] && L=paper_2507_10804_b200/libhv.so
  echo "== $v cfg3"; HV_LIB=$L python tools/tune.py --config 3 --shots 16 --S 16 --FG 0 --reps 1 2>&1 | tail -1
  echo "== $v cfg4"; HV_LIB=$L timeout 900 python bench.py --config 4 --shots 4 --nt 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k: round(v['avg_launch_ms'],3) for k,v in d['roofline']['kernels'].items()})"
done
