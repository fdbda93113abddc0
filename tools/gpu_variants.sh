# shot-block size of the forward unit order (dev tool)
for b in 1 2 4 8 16; do echo "== cfg1 sblk $b"; HV_SBLK=$b python tools/tune.py --config 1 --S 16 --FG 0 --reps 1 2>&1 | tail -1; done
for b in 1 4 7 16; do echo "== cfg3 sblk $b"; HV_SBLK=$b python tools/tune.py --config 3 --shots 16 --S 16 --FG 0 --reps 1 2>&1 | tail -1; done
for b in 1 2 4; do echo "== cfg4 sblk $b"; HV_SBLK=$b timeout 900 python bench.py --config 4 --shots 4 --nt 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k: round(v['avg_launch_ms'],3) for k,v in d['roofline']['kernels'].items()})"; done
