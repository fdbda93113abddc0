set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g12_gpu.log 2>&1; echo gpu=$?
tail -8 gpurun_out/g12_gpu.log
timeout 300 python bench.py --config 3 --shots 16 --nt 400 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g12_c3.json 2> gpurun_out/g12_c3.err; echo c3=$?
python -c "import json;d=json.loads(open('gpurun_out/g12_c3.json').read().strip().splitlines()[-1]);print('c3', round(d['value'],3), {k:(round(v['avg_launch_ms']*1e3,1),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
timeout 300 python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g12_c1.json 2> gpurun_out/g12_c1.err; echo c1=$?
python -c "import json;d=json.loads(open('gpurun_out/g12_c1.json').read().strip().splitlines()[-1]);print('c1', round(d['value'],3), {k:(round(v['avg_launch_ms']*1e3,1),round(v['batched_frac'],3)) for k,v in d['roofline']['kernels'].items()})"
