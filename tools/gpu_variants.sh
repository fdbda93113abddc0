# planner fix check: cfg2 bench line + whole GPU suite (dev tool)
timeout 600 python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2b.json 2> gpurun_out/bench_cfg2b.err; echo cfg2=$?; tail -1 gpurun_out/bench_cfg2b.json
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; echo pt=$?; tail -3 gpurun_out/pt.log
