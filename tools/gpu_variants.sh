# resident-q forward: Born fields per CTA (dev tool)
for f in 4 6 8 11; do echo "== cfg3 qfg $f"; HV_QFG=$f python tools/tune.py --config 3 --shots 16 --S 16 --FG 0 --reps 1 2>&1 | tail -1; done
for f in 4 6 8; do echo "== cfg4 qfg $f"; HV_QFG=$f timeout 900 python bench.py --config 4 --shots 4 --nt 200 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k: round(v['avg_launch_ms'],3) for k,v in d['roofline']['kernels'].items()})"; done
