# evidence lines with the resident-q forward (dev tool)
timeout 900 python bench.py --config 4 --shots 4 --nt 400 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4q.json 2>/dev/null; tail -1 gpurun_out/bench_cfg4q.json
timeout 1200 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3q.json 2>/dev/null; tail -1 gpurun_out/bench_cfg3q.json
