set -x
TAG=${1:-r02g}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_exit=$?
tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$?
tail -c 600 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; echo ref_exit=$?
tail -c 400 gpurun_out/ref_$TAG.json
timeout 900 python bench.py --config 3 --mode misfit --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev_cfg3_misfit_$TAG.json 2>&1; echo ev_misfit=$?
tail -c 300 gpurun_out/ev_cfg3_misfit_$TAG.json
