# difference-form Laplacian for the background only: accuracy + speed + full GPU tests
set -x
python tools/gpu/dbg_cfg2b.py > gpurun_out/g20_dbg.log 2>&1; cat gpurun_out/g20_dbg.log
python tools/gpu/dbg_cfg2.py > gpurun_out/g20_dbg2.log 2>&1; cat gpurun_out/g20_dbg2.log
timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g20_c3.json 2> gpurun_out/g20_c3.err
python -c "import json;d=json.loads(open('gpurun_out/g20_c3.json').read().strip().splitlines()[-1]);print('c3', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
timeout 300 python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g20_c1.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/g20_c1.json').read().strip().splitlines()[-1]);print('c1', round(d['value'],3), {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g20_gpu.log 2>&1; echo gpu=$?; tail -4 gpurun_out/g20_gpu.log
