# new API + dist tests, full gpu suite minus golden, short cfg3 bench with the new bench.py
set -x
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_dist.py -x -q > gpurun_out/g2_api.log 2>&1; echo api=$?
tail -15 gpurun_out/g2_api.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_golden.py -k "not golden" > gpurun_out/g2_gpu.log 2>&1; echo gpu=$?
tail -5 gpurun_out/g2_gpu.log
timeout 900 python bench.py --steps 2 --warmup 1 --cpu-nt 60 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo bench=$?
tail -c 3000 gpurun_out/g2_bench.json
tail -5 gpurun_out/g2_bench.err
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 1 --config 0 --no-cpu-baseline > gpurun_out/g2_bench2.json 2> gpurun_out/g2_bench2.err; echo bench2=$?
tail -5 gpurun_out/g2_bench2.err
